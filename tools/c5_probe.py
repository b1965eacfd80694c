"""Probe: C5 at a given n on one B200 -- generation time, husky_sort per-stage
breakdown (profiler mode 1, one event pair per launch), GPU verifier, and the
same with HUSKY_KEYSORT=msd if requested.  Not a bench line.

  python tools/c5_probe.py [log2n=30] [reps=3] [config=C5]   (C1-C4: numpy generator, n = 2^log2n)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import checker  # noqa: E402
import paper_2012_00866_b200 as h  # noqa: E402
import workloads.gpu as G  # noqa: E402


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    N = 1 << lg if lg <= 40 else lg  # a log2 size, or an exact n
    cfg = sys.argv[3] if len(sys.argv) > 3 else "C5"
    torch.cuda.set_device(0)
    t0 = time.time()
    if cfg == "C5":
        u, o = G.c5_device(N)
    else:
        import numpy as np
        import workloads as W
        w = W.make(cfg, N)
        uu = w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units
        u = torch.from_numpy(np.concatenate([uu, np.zeros(16, uu.dtype)])).cuda()
        o = torch.from_numpy(w.offsets).cuda()
    coder = 1 if cfg == "C3" else 0
    if cfg != "C5":
        coder = w.coder
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    total = int(o[-1].item())
    ws = torch.empty(h.husky_sort_workspace(coder, N, total), dtype=torch.uint8, device="cuda")
    perm = torch.empty(N, dtype=torch.int32, device="cuda")
    su = torch.empty(total + 16, dtype=u.dtype, device="cuda")
    so = torch.empty(N + 1, dtype=torch.int64, device="cuda")
    res = {"lib": os.environ.get("HUSKY_LIB", "default"), "config": cfg, "n": N, "gen_s": round(gen_s, 2), "ws_gb": round(ws.numel() / 1e9, 2),
           "mem_alloc_gb": round(torch.cuda.memory_allocated() / 1e9, 2)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        outc = h.husky_sort(coder, u, o, perm, su, so, ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.husky_sort(coder, u, o, perm, su, so, ws)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res["ms"] = ts
    h.husky_profile_reset()
    h.husky_profile_enable(1)
    flush.fill_(2)
    h.husky_sort(coder, u, o, perm, su, so, ws)
    torch.cuda.synchronize()
    h.husky_profile_enable(False)
    res["stages"] = {k: round(v["ms"], 3) for k, v in h.husky_profile_read().items() if v["launches"]}
    res["outcome"] = outc
    t0 = time.time()
    res["verify"] = checker.verify(u, o, perm, su[:total], so)
    res["verify_s"] = round(time.time() - t0, 2)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
