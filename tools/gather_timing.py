"""Per-tile phase timing of the last main gather (needs HUSKY_NVCC_DEFS=-DHUSKY_TIMING)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W

w = W.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
u = torch.from_numpy(w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units).cuda()
o = torch.from_numpy(w.offsets).cuda()
for _ in range(3):
    h.sort(w.coder, u, o)
lib = h._lib
lib.husky_debug_gather_times.restype = ctypes.c_int
ntiles = (w.n + 1023) // 1024
buf = np.zeros((16384, 8), dtype=np.uint64)
k = lib.husky_debug_gather_times(buf.ctypes.data_as(ctypes.c_void_p), 16384)
t = buf[:min(ntiles, k)].astype(np.int64)
t0 = t[:, 0].min()
names = ["loads+scan", "stage window", "lookback+sync", "check+runs", "writes"]
for i, nm in enumerate(names):
    d = t[:, i + 1] - t[:, i]
    print(f"{nm:16s} median {np.median(d)/1e3:7.2f} us  p90 {np.percentile(d,90)/1e3:7.2f}  mean {d.mean()/1e3:7.2f}")
tot = t[:, 5] - t[:, 0]
print(f"{'tile total':16s} median {np.median(tot)/1e3:7.2f} us  mean {tot.mean()/1e3:7.2f}")
print("span us", (t[:, 5].max() - t0) / 1e3, "tiles", len(t))
print("mean tiles in flight", tot.sum() / (t[:, 5].max() - t0))
# start-time order vs tile id: how far the look-back chain lags the tile starts
st = t[:, 0] - t0
lb_end = t[:, 3] - t0
print("tile-start rate (tiles/us)", len(t) / (st.max() / 1e3 + 1e-9))
