# large inputs launch only the planned pass slots (host reads the plan): tests above 2^26, A/B vs lab/base at C5 2^30 / 2^26
timeout 1200 python -m pytest tests/test_gpu_large.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in base new base new; do
  if [ $v = base ]; then export HUSKY_LIB=$PWD/lab/base/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print([round(x,2) for x in d['ms']], d['stages'].get('radix_pass'), d['outcome']['radix_passes'], d['verify'])"
  timeout 300 python tools/c5_probe.py 26 5 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print([round(x,3) for x in d['ms']], d['stages'].get('radix_pass'), d['verify'])"
done 2>&1 | tee gpurun_out/s3_slots.txt
