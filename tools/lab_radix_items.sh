# onesweep keys per thread (tile = 512 x items): HUSKY_RADIX_ITEMS 8 .. 16
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for it in 14; do
  HUSKY_NVCC_DEFS="-DHUSKY_RADIX_ITEMS=$it" python -c "$B" > /dev/null 2>&1 || echo build failed
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py -x -q -k "not multi" > gpurun_out/pytest_it$it.log 2>&1; echo pytest$it=$?; tail -1 gpurun_out/pytest_it$it.log
done
for rep in 1 2; do for it in 12 14 16; do
  HUSKY_NVCC_DEFS="-DHUSKY_RADIX_ITEMS=$it" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG=items$it timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*gather.: \([0-9.]*\).*/radix \1 gather \2/'; done
done; done 2>&1 | tee gpurun_out/lab_items.txt
python -c "$B" > /dev/null 2>&1
