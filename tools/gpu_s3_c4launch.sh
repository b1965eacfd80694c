timeout 300 python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, numpy as np
import paper_2012_00866_b200 as h, workloads as W
for cfg in ("C4", "C3", "C2"):
    w=W.make(cfg, 10_000_000); uu = w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units
    u=torch.from_numpy(np.concatenate([uu, np.zeros(16, uu.dtype)])).cuda(); o=torch.from_numpy(w.offsets).cuda()
    for _ in range(3): h.sort(w.coder,u,o)
    torch.cuda.synchronize()
    h.husky_profile_reset(); h.husky_profile_enable(1); h.sort(w.coder,u,o); torch.cuda.synchronize(); h.husky_profile_enable(False)
    print("==", cfg)
    for st,el,ms in h.husky_profile_launches(): print(f"{st:14s} {el:10d} {ms*1000:8.1f} us")
PY
