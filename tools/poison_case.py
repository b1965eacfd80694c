"""Poison helper: run degenerate sorts with workspace/outputs pre-filled with a byte pattern."""
import random, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W
import oracle

pat = int(sys.argv[1], 0)
for seed in range(int(sys.argv[2]), int(sys.argv[3])):
    for coder in (0, 1):
        rng = random.Random(seed)
        base = [[0x61], [0x61, 0], [0x61, 0, 0], [0x61, 0, 0, 0], [0x61, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]]
        strings = [list(rng.choice(base)) for _ in range(5000)]
        w = W.from_strings(strings, coder)
        u = torch.from_numpy(w.units.view(np.int16) if coder else w.units).cuda()
        o = torch.from_numpy(w.offsets).cuda()
        n = w.n; total = int(u.numel())
        ws = torch.empty(h.husky_sort_workspace(coder, n, total), dtype=torch.uint8, device="cuda").fill_(pat)
        perm = torch.empty(max(n, 1), dtype=torch.int32, device="cuda").fill_(-1)
        su = torch.empty(max(total, 1) + 8, dtype=u.dtype, device="cuda").fill_(0x55)
        so = torch.empty(n + 1, dtype=torch.int64, device="cuda").fill_(-1)
        try:
            outc = h.husky_sort(coder, u, o, perm, su, so, ws)
            p = perm.cpu().numpy().view(np.uint32)
            ref = oracle.sort(coder, w.units, w.offsets)
            if not np.array_equal(p, ref):
                print("mismatch", seed, coder, outc, flush=True)
        except Exception as e:
            print("seed", seed, "coder", coder, "error", e, flush=True)
            sys.exit(1)
print("done")
