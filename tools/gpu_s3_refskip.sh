# refinement partial sort (C4): parity + fuzz suites, then A/B vs lab/head3 (HEAD) at C5 / D1 / C4 / C2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py tests/test_gpu_large.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head3/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', [round(x,2) for x in d['ms']], d['stages'].get('radix_pass'), d['outcome']['refine_rounds'], d['verify'])"
  for c in D1 C4 C2; do timeout 300 python tools/c5_probe.py 10000000 5 $c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', [round(x,3) for x in d['ms']], d['stages'].get('fix_small'), d['stages'].get('fix_medium'), d['stages'].get('gather'), d['verify'])"; done
done 2>&1 | tee gpurun_out/s3_refskip.txt
