timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "C5 or slab or gather or ragged" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for rep in 1 2; do for lib in default lab/g0/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  for c in "30 2 C5" "23 3 C2"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
done; done
