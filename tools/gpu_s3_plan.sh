# the hist kernel's plan (last CTA) with one warp per digit: parity suites, then A/B vs lab/head at C1 / 3e5 / C2 / C5
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py tests/test_gpu_keysort.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  for n in 1000 100000 300000; do timeout 300 python tools/c5_probe.py $n 9 C1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n'], [round(x,4) for x in d['ms']], d['stages'].get('hist_scan'), d['verify'])"; done
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C2', [round(x,3) for x in d['ms']], d['stages'].get('hist_scan'), d['verify'])"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', [round(x,2) for x in d['ms']], d['stages'].get('hist_scan'), d['verify'])"
done 2>&1 | tee gpurun_out/s3_plan.txt
