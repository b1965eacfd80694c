"""Per-tile phase timing of the last onesweep pass (needs a -DHUSKY_TIMING build)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
if cfg == "C5":  # python tools/tile_timing.py C5 <log2n>: device generator
    import workloads.gpu as G
    u, o = G.c5_device(1 << int(sys.argv[2]))
    coder, n = 0, int(o.numel() - 1)
else:
    w = W.make(cfg)
    u = torch.from_numpy(w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units).cuda()
    o = torch.from_numpy(w.offsets).cuda()
    coder, n = w.coder, w.n
for _ in range(3):
    h.sort(coder, u, o)
lib = h.lib()
lib.husky_debug_tile_times.restype = ctypes.c_int
import os; TS = int(os.environ.get("TILE", "6144")); ntiles = (n + TS - 1) // TS
buf = np.zeros((8192, 8), dtype=np.uint64)
k = lib.husky_debug_tile_times(buf.ctypes.data_as(ctypes.c_void_p), 8192)
t = buf[:min(ntiles, k)].astype(np.int64)
t0 = t[:, 0].min()
names = ["start->first key", "rank", "counts+scan", "exchange+lookback(t0)", "lookback wait rest", "scatter"]
for i, nm in enumerate(names):
    d = t[:, i + 1] - t[:, i]
    print(f"{nm:24s} median {np.median(d)/1e3:7.2f} us  p90 {np.percentile(d,90)/1e3:7.2f} us  mean {d.mean()/1e3:7.2f}")
tot = t[:, 6] - t[:, 0]
print(f"{'tile total':24s} median {np.median(tot)/1e3:7.2f} us  mean {tot.mean()/1e3:7.2f}")
print("pass span us", (t[:, 6].max() - t0) / 1e3, "tiles", len(t))
st = np.sort(t[:, 0] - t0) / 1e3
print("start times (us) quantiles", [round(float(np.percentile(st, q)), 1) for q in (0, 10, 25, 50, 75, 90, 100)])
it = (t[:, 7] & 0xFFFFFFFF); polls = (t[:, 7] >> 32)
print("lookback iterations (digit 0): median", np.median(it), "mean", it.mean(), "p90", np.percentile(it, 90))
print("blocked polls (digit 0): median", np.median(polls), "mean", polls.mean(), "p90", np.percentile(polls, 90), "frac>0", (polls > 0).mean())
# distance from each tile to the nearest predecessor that had finished its look-back when it started looking
