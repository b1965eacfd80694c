B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for v in 4 5 6; do
  HUSKY_NVCC_DEFS="-DHUSKY_GATHER_MINB=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG="minb$v" python tools/lab_sort.py $c | sed 's/stages.*gather.: \([0-9.]*\).*/gather \1/'; done
done
