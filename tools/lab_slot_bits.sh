# A/B of the device-planned passes' digit width (HUSKY_SLOT_BITS 9 vs 8) on C2..C4,
# after a quick parity subset on the default (9-bit) build.
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
python -c "$B" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py tests/test_gpu_next.py -x -q > gpurun_out/pytest_slot.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_slot.log
for v in "-DHUSKY_SLOT_BITS=9" "-DHUSKY_SLOT_BITS=8"; do
  HUSKY_NVCC_DEFS="$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3 C4; do TAG="$v" python tools/lab_sort.py $c; done
done 2>&1 | tee gpurun_out/lab_slot_bits.txt
python -c "$B" > /dev/null 2>&1
