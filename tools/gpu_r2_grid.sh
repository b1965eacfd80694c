for rep in 1 2; do
for lib in default lab/w6/ lab/w8/ lab/w10/; do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  timeout 300 python tools/c5_probe.py 30 2 C5 2>&1 | tail -1
  timeout 300 python tools/c5_probe.py 23 3 C2 2>&1 | tail -1
  timeout 300 python tools/c5_probe.py 17 3 C1 2>&1 | tail -1
done; done
