B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for v in "-DHUSKY_ENC_IT=4 -DHUSKY_ENC_MINB=1" "-DHUSKY_ENC_IT=4 -DHUSKY_ENC_MINB=6" "-DHUSKY_ENC_IT=4 -DHUSKY_ENC_MINB=8" "-DHUSKY_ENC_IT=2 -DHUSKY_ENC_MINB=8" "-DHUSKY_ENC_IT=8 -DHUSKY_ENC_MINB=4"; do
  HUSKY_NVCC_DEFS="$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG="$v" python tools/lab_sort.py $c | sed 's/stages.*encode.: \([0-9.]*\).*/encode \1/'; done
done
