"""Large-n parity by the oracle's linear uniqueness verifier: husky_sort on the
GPU, then oracle.verify (bijection + strictly increasing adjacent pairs == the
oracle's unique order) and the sorted units/offsets against a host gather."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2012_00866_b200 as h
import workloads as W

name, n = sys.argv[1], int(sys.argv[2])
t0 = time.time()
w = W.make(name, n)
print(f"generated {name} n={w.n} units={w.units.size} in {time.time()-t0:.1f}s", flush=True)
u = torch.from_numpy(w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units).cuda()
o = torch.from_numpy(w.offsets).cuda()
perm, su, so, outc = h.sort(w.coder, u, o)
torch.cuda.synchronize()
ts = []
for i in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); h.sort(w.coder, u, o); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("outcome", outc, "ms", ts, "Mstr/s", w.n / (min(ts) * 1e-3) / 1e6, flush=True)
p = perm.cpu().numpy().view(np.uint32)
t0 = time.time()
r = oracle.verify(w.coder, w.units, w.offsets, p)
print("verify", r, f"{time.time()-t0:.1f}s", flush=True)
assert r == 0
lens = (w.offsets[1:] - w.offsets[:-1])[p]
so_ref = np.zeros(w.n + 1, np.int64); np.cumsum(lens, out=so_ref[1:])
assert np.array_equal(so.cpu().numpy(), so_ref)
print("sorted offsets ok")
