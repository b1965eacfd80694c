"""Time husky_encode (no fused histograms) on a config; compare with the sort's encode stage."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W

w = W.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
u = torch.from_numpy(w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units).cuda()
o = torch.from_numpy(w.offsets).cuda()
codes = torch.empty(w.n, dtype=torch.int64, device="cuda")
for _ in range(3):
    h.husky_encode(w.coder, u, o, codes, want_perfect=False)
torch.cuda.synchronize()
h.husky_profile_reset(); h.husky_profile_enable(True)
for _ in range(10):
    h.husky_encode(w.coder, u, o, codes, want_perfect=False)
torch.cuda.synchronize()
p = h.husky_profile_read(); h.husky_profile_enable(False)
print("encode (no hist) us/launch", p["encode"]["ms"] / p["encode"]["launches"] * 1e3)
for _ in range(2):
    h.sort(w.coder, u, o)
h.husky_profile_reset(); h.husky_profile_enable(True)
for _ in range(5):
    h.sort(w.coder, u, o)
torch.cuda.synchronize()
p = h.husky_profile_read(); h.husky_profile_enable(False)
print("encode (hist + packed) us/launch", p["encode"]["ms"] / p["encode"]["launches"] * 1e3)
