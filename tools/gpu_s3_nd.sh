# histogram kernel: digits above a re-packed key's width counted once per thread (new) vs HEAD (lab/head)
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', [round(x,2) for x in d['ms']], d['stages'].get('hist_scan'), d['verify'])"
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C2', [round(x,3) for x in d['ms']], d['stages'].get('hist_scan'), d['verify'])"
done 2>&1 | tee gpurun_out/s3_nd.txt
