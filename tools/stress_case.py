"""Stress helper: repeat one degenerate sort many times (debugging races on the GPU box)."""
import random, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W
import oracle

coder = int(sys.argv[1]); reps = int(sys.argv[2])
rng = random.Random(int(sys.argv[3]) if len(sys.argv) > 3 else 1)
base = [[0x61], [0x61, 0], [0x61, 0, 0], [0x61, 0, 0, 0], [0x61, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]]
strings = [list(rng.choice(base)) for _ in range(5000)]
w = W.from_strings(strings, coder)
u = torch.from_numpy(w.units.view(np.int16) if coder else w.units).cuda()
o = torch.from_numpy(w.offsets).cuda()
ref = oracle.sort(coder, w.units, w.offsets)
bad = 0
for i in range(reps):
    try:
        perm, su, so, outc = h.sort(coder, u, o)
        p = perm.cpu().numpy().view(np.uint32)
        if not np.array_equal(p, ref):
            bad += 1
            print("mismatch rep", i, outc, flush=True)
    except Exception as e:
        print("rep", i, "error", e, flush=True)
        break
print("reps", reps, "bad", bad, outc)
