timeout 300 python tools/c5_probe.py 100000 5 C1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print([round(x,4) for x in d['ms']], d['stages'], d['outcome'])"
timeout 300 python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, numpy as np
import paper_2012_00866_b200 as h, workloads as W
w=W.make("C1",100000); u=torch.from_numpy(w.units).cuda(); o=torch.from_numpy(w.offsets).cuda()
for _ in range(3): h.sort(0,u,o)
torch.cuda.synchronize()
h.husky_profile_reset(); h.husky_profile_enable(1); h.sort(0,u,o); torch.cuda.synchronize(); h.husky_profile_enable(False)
for st,el,ms in h.husky_profile_launches(): print(f"{st:14s} {el:10d} {ms*1000:8.1f} us")
PY
