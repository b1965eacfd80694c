# partial key sort (R19) for UNICODE codes: the parity + fuzz suites, then A/B vs lab/head at C3 (1e7) and C2 / C5
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 10000000 5 C3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3', [round(x,3) for x in d['ms']], d['stages'], d['outcome']['radix_passes'], d['outcome']['n_runs'], d['verify'])"
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C2', [round(x,3) for x in d['ms']], d['verify'])"
done 2>&1 | tee gpurun_out/s3_uskip.txt
