"""Stress helper: the nul_ext degenerate case over many seeds, both coders."""
import random, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W
import oracle

for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    for coder in (0, 1):
        rng = random.Random(seed)
        base = [[0x61], [0x61, 0], [0x61, 0, 0], [0x61, 0, 0, 0], [0x61, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]]
        strings = [list(rng.choice(base)) for _ in range(5000)]
        w = W.from_strings(strings, coder)
        u = torch.from_numpy(w.units.view(np.int16) if coder else w.units).cuda()
        o = torch.from_numpy(w.offsets).cuda()
        ref = oracle.sort(coder, w.units, w.offsets)
        try:
            perm, su, so, outc = h.sort(coder, u, o)
            p = perm.cpu().numpy().view(np.uint32)
            if not np.array_equal(p, ref):
                print("mismatch seed", seed, coder, outc, flush=True)
        except Exception as e:
            print("seed", seed, "coder", coder, "error", e, flush=True)
            sys.exit(1)
print("done")
