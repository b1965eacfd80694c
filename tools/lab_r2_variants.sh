# A/B of lab builds (lab/<name>/libhusky.so) on C5 2^30 and C2
for lib in default $(ls -d lab/*/ 2>/dev/null); do
  if [ "$lib" = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/${lib}libhusky.so; fi
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1
done
