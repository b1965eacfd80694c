"""Phase cycles of k_fix_staged (lab build with -DHUSKY_FIX_TIMING; HUSKY_LIB)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_00866_b200 as h  # noqa: E402
import workloads as W  # noqa: E402

w = W.make("D1", int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23)
u = torch.from_numpy(w.units).cuda()
o = torch.from_numpy(w.offsets).cuda()
perm, su, so, outc = h.sort(w.coder, u, o)
torch.cuda.synchronize()
buf = np.zeros((1024, 4), dtype=np.uint64)
h._lib.husky_debug_fix_phases(buf.ctypes.data_as(ctypes.c_void_p))
b = buf[:148].astype(np.float64)
tot = b.sum(axis=1)
print("runs", outc["runs_by_class"], "per-CTA Mcycles total (mean)", tot.mean() / 1e6)
for i, nm in enumerate(["stage+arrays", "keys", "sort", "scan+write"]):
    print(f"{nm:14s} {b[:, i].mean() / 1e6:8.3f} Mcycles  {100 * b[:, i].sum() / tot.sum():5.1f}%")
