# gather stage word swizzle (bank conflicts): A/B vs lab/head (HEAD build) at C5 2^30 / 2^27, C2, C3; parity + fuzz tests
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', [round(x,2) for x in d['ms']], d['stages'].get('gather'), d['verify'])"
  timeout 300 python tools/c5_probe.py 27 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5/8', [round(x,3) for x in d['ms']], d['stages'].get('gather'), d['verify'])"
  for c in C2 C3 C4; do timeout 300 python tools/c5_probe.py 23 5 $c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', [round(x,3) for x in d['ms']], d['stages'].get('gather'), d['verify'])"; done
done 2>&1 | tee gpurun_out/s3_swz.txt
unset HUSKY_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_large.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
