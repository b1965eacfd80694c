timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for rep in 1 2; do for lib in default lab/t0/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  for c in "30 2 C5" "23 3 C2" "17 5 C1"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
done; done
