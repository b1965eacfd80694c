# R20 finish (batched staging loads): its tests, forced-finish parity, then A/B vs lab/head and a per-launch list at 2^27
timeout 900 python -m pytest tests/test_gpu_finish.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch
import paper_2012_00866_b200 as h, workloads.gpu as G
u,o=G.c5_device(1<<27)
for _ in range(2): h.sort(0,u,o)
torch.cuda.synchronize()
h.husky_profile_reset(); h.husky_profile_enable(1); h.sort(0,u,o); torch.cuda.synchronize(); h.husky_profile_enable(False)
for st,el,ms in h.husky_profile_launches(): print(f"{st:14s} {el:10d} {ms:8.3f} ms")
PY
for v in head new head new; do
  if [ $v = head ]; then export HUSKY_LIB=$PWD/lab/head/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  timeout 300 python tools/c5_probe.py 30 3 C5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', [round(x,2) for x in d['ms']], d['stages'].get('radix_pass'), d['outcome']['radix_passes'], d['verify'])"
done 2>&1 | tee gpurun_out/s3_finish2.txt
