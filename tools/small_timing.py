"""Phase times of the cluster small-input kernel (lab build -DHUSKY_SMALL_TIMING, HUSKY_LIB)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_00866_b200 as h  # noqa: E402
import workloads as W  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
w = W.make("C1", n)
u = torch.from_numpy(w.units).cuda(); o = torch.from_numpy(w.offsets).cuda()
for _ in range(3):
    h.sort(0, u, o)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); h.sort(0, u, o); b.record(); torch.cuda.synchronize()
buf = np.zeros(64, dtype=np.uint64)
h._lib.husky_debug_small_times(buf.ctypes.data_as(ctypes.c_void_p))
t = buf.astype(np.int64)
names = {1: "encode", 2: "agree", 12: "runs", 13: "offsets", 14: "units"}
prev = t[0]
for i in range(1, 15):
    if t[i] == 0:
        continue
    print(f"{names.get(i, 'pass%d' % (i - 3)):8s} {(t[i] - prev) / 1e3:8.2f} us")
    prev = t[i]
print("kernel span", (t[14] - t[0]) / 1e3, "us; event time of the whole sort", a.elapsed_time(b) * 1e3, "us")
