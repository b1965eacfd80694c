for lib in default lab/i11/ lab/i13/ lab/rb4w6/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  timeout 300 python tools/c5_probe.py 30 2 C5 2>&1 | tail -1
  timeout 300 python tools/c5_probe.py 23 3 C2 2>&1 | tail -1
done
