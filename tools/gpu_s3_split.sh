# radix ranking: peer masks of all items first, then the counter chain (lab/split*, HUSKY_RANK_SPLIT=1) vs HEAD
for v in default split split_b4 split_b6 default split; do
  if [ $v = default ]; then unset HUSKY_LIB; else export HUSKY_LIB=$PWD/lab/$v/libhusky.so; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print([round(x,2) for x in d['ms']], d['stages'].get('radix_pass'), d['verify'])"
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print([round(x,3) for x in d['ms']], d['stages'].get('radix_pass'), d['verify'])"
done 2>&1 | tee gpurun_out/s3_split.txt
