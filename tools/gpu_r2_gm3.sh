for lib in default lab/gm3/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  for c in "30 2 C5" "27 3 C5" "23 3 C2"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
done
