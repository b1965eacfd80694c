timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_fuzz.py -x -q -k "encode or A1 or coder or english or offsets or slab or C5 or fuzz or empty or edge" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for rep in 1 2; do for lib in default lab/encold/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  for c in "30 2 C5" "23 5 C2" "23 5 C3"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
done; done
