"""Per-tile phase timing of the main gather (lab build with -DHUSKY_TIMING, loaded via HUSKY_LIB).

  python tools/gather_timing.py [C2|C5] [n]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_00866_b200 as h  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else W.FULL_N[cfg]
if cfg == "C5":
    import workloads.gpu as G
    u, o = G.c5_device(n)
    coder = 0
else:
    w = W.make(cfg, n)
    u = torch.from_numpy(w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units).cuda()
    o = torch.from_numpy(w.offsets).cuda()
    coder = w.coder
for _ in range(3):
    h.sort(coder, u, o)
torch.cuda.synchronize()
lib = h._lib
lib.husky_debug_gather_times.restype = ctypes.c_int
buf = np.zeros((16384, 8), dtype=np.uint64)
k = lib.husky_debug_gather_times(buf.ctypes.data_as(ctypes.c_void_p), 16384)
t = buf[:k].astype(np.int64)
t = t[t[:, 5] > 0]
names = ["loads+scan", "stage window", "lookback+sync", "check+runs", "writes"]
for i, nm in enumerate(names):
    d = t[:, i + 1] - t[:, i]
    print(f"{nm:16s} median {np.median(d)/1e3:7.2f} us  p90 {np.percentile(d,90)/1e3:7.2f}  mean {d.mean()/1e3:7.2f}")
tot = t[:, 5] - t[:, 0]
print(f"{'tile total':16s} median {np.median(tot)/1e3:7.2f} us  mean {tot.mean()/1e3:7.2f}  tiles {len(t)}")
