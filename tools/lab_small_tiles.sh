# small inputs: onesweep keys per thread (tile = 512 x items) on C1 (1e5 strings)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for it in 12 4 2 1; do
  HUSKY_NVCC_DEFS="-DHUSKY_RADIX_ITEMS=$it" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C1; do TAG="items$it" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*/radix \1/'; done
done 2>&1 | tee gpurun_out/lab_small_tiles.txt
python -c "$B" > /dev/null 2>&1
