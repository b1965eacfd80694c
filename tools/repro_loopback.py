"""Repro helper: one loopback sample sort (used while debugging on the GPU box)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W

name, n, world = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
w = W.make(name, n)
u = torch.from_numpy(w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units).cuda()
o = torch.from_numpy(w.offsets).cuda()
tot = w.units.size
ws = torch.empty(h.husky_sort_multi_loopback_workspace(w.coder, world, w.n, tot), dtype=torch.uint8, device="cuda")
perm = torch.empty(w.n, dtype=torch.int32, device="cuda")
su = torch.empty(tot + 8, dtype=u.dtype, device="cuda")
so = torch.empty(w.n + 1, dtype=torch.int64, device="cuda")
print(h.husky_sort_multi_loopback(w.coder, world, u, o, perm, su, so, ws))
