"""Median husky_sort time on a config, profiler off (env variants are set by the caller)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_00866_b200 as h
import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = W.make(name)
u = w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units
du = torch.from_numpy(np.ascontiguousarray(u)).cuda(); do = torch.from_numpy(w.offsets).cuda()
n, total = w.n, w.units.size
ws = torch.empty(h.husky_sort_workspace(w.coder, n, total), dtype=torch.uint8, device="cuda")
perm = torch.empty(n, dtype=torch.int32, device="cuda")
su = torch.empty(total + 8, dtype=du.dtype, device="cuda"); so = torch.empty(n + 1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(13):
    flush.fill_(i); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); h.husky_sort(w.coder, du, do, perm, su, so, ws); b.record(); torch.cuda.synchronize()
    if i >= 3: ts.append(a.elapsed_time(b))
h.husky_profile_reset(); h.husky_profile_enable(True)
for i in range(5):
    flush.fill_(i); h.husky_sort(w.coder, du, do, perm, su, so, ws)
torch.cuda.synchronize(); h.husky_profile_enable(False)
prof = h.husky_profile_read()
st = {k: round(v["ms"] / 5 * 1e3, 1) for k, v in prof.items() if v["launches"]}
print(f"{name} {os.environ.get('TAG','')}: median {np.median(ts)*1e3:.1f} us  min {min(ts)*1e3:.1f}  stages(us) {st}", flush=True)
