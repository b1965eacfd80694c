export HUSKY_LIB=$PWD/lab/timing/libhusky.so
for c in "C5 28" "C2"; do echo "== $c"; timeout 300 python tools/tile_timing.py $c; done 2>&1 | tee gpurun_out/ttiming_r2.txt
