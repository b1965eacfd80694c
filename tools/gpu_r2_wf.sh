timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_large.py -x -q 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for lib in default lab/wf0/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  for c in "30 3 C5" "27 3 C5" "23 5 C2" "23 5 C3"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
done
