for lib in default lab/g3m5/ lab/g2m6/ lab/g3m4/ lab/g5/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  timeout 300 python tools/c5_probe.py 30 2 C5 2>&1 | tail -1
  timeout 300 python tools/c5_probe.py 23 3 C2 2>&1 | tail -1
done
