"""Reference points on the box: torch.sort (CUB radix) of the 1e7 C2 codes, and a
device copy of the same byte volume as one onesweep pass."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_00866_b200 as h
import workloads as W

w = W.make("C2")
du = torch.from_numpy(w.units).cuda(); do = torch.from_numpy(w.offsets).cuda()
codes = torch.empty(w.n, dtype=torch.int64, device="cuda")
h.husky_encode(w.coder, du, do, codes)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, k=8):
    ts = []
    for i in range(k):
        flush.fill_(i); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3
print("torch.sort stable int64 (values+int64 idx) 1e7: %.1f us" % t(lambda: torch.sort(codes, stable=True)))
idx = torch.arange(w.n, dtype=torch.int32, device="cuda")
x = torch.empty(w.n * 12 // 4, dtype=torch.int32, device="cuda"); y = torch.empty_like(x)
print("copy 120 MB (one pass volume read+write 240 MB): %.1f us" % t(lambda: y.copy_(x)))
