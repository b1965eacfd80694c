# A/B of the device-planned passes' digit width (HUSKY_SLOT_BITS 9 vs 8) on C2..C4, parity subset on the 9-bit build
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
HUSKY_NVCC_DEFS="-DHUSKY_SLOT_BITS=9" python -c "$B" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py tests/test_gpu_next.py -x -q -k "not multi" > gpurun_out/pytest_slot.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_slot.log
for rep in 1 2; do for v in 9 8; do
  HUSKY_NVCC_DEFS="-DHUSKY_SLOT_BITS=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3 C4; do TAG="bits$v" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*/radix \1/'; done
done; done 2>&1 | tee gpurun_out/lab_slot_bits.txt
python -c "$B" > /dev/null 2>&1
