# R20 in-run finish: its tests, the parity + fuzz suites with the finish forced at every size, the large test
# (rule mode), then A/B vs lab/head at C5 2^30 / 2^27
timeout 900 python -m pytest tests/test_gpu_finish.py -x -q -p no:cacheprovider 2>&1 | tail -3
HUSKY_FINISH=2 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', [round(x,2) for x in d['ms']], d['stages'].get('radix_pass'), d['outcome']['radix_passes'], d['outcome']['n_runs'], d['verify'])"
  timeout 300 python tools/c5_probe.py 27 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5/8', [round(x,3) for x in d['ms']], d['stages'].get('radix_pass'), d['outcome']['radix_passes'], d['verify'])"
done 2>&1 | tee gpurun_out/s3_finish.txt
