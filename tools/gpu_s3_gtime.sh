# per-tile phases of the main gather and the radix pass at C5 (lab build with -DHUSKY_TIMING)
export HUSKY_LIB=$PWD/lab/timing/libhusky.so
timeout 600 python tools/gather_timing.py C5 1073741824 2>&1 | tail -8
timeout 600 python tools/tile_timing.py C5 30 2>&1 | tail -10
