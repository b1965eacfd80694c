# onesweep pass kernel at 2 / 3 CTAs per SM (HUSKY_RADIX_MINB)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for rep in 1 2; do for v in 2 3; do
  HUSKY_NVCC_DEFS="-DHUSKY_RADIX_MINB=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG=minb$v timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*gather.: \([0-9.]*\).*/radix \1 gather \2/'; done
done; done 2>&1 | tee gpurun_out/lab_minb.txt
python -c "$B" > /dev/null 2>&1
