# A/B on one box: lab/base/libhusky.so (HEAD before the change) vs the working tree's
# libhusky.so, C5 2^30 and C2, alternating
for v in base new base new; do
  if [ $v = base ]; then export HUSKY_LIB=$PWD/lab/base/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:v for k,v in d.items() if k in ('ms','ms_min','stages','verify')})" 2>&1 | cut -c1-900
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1 | cut -c1-400
  timeout 300 python tools/c5_probe.py 100000 5 C1 2>&1 | tail -1 | cut -c1-500
done 2>&1 | tee gpurun_out/s3_ab.txt
