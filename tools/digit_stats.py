"""Per-digit statistics of a workload's husky codes (distinct values, largest bin share)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import workloads as W
for name in sys.argv[1:] or ["C2", "C3"]:
    w = W.make(name)
    codes, _ = oracle.encode(w.coder, w.units, w.offsets)
    for d in range(8):
        dig = ((codes >> np.uint64(8 * d)) & np.uint64(255)).astype(np.int64)
        h = np.bincount(dig, minlength=256)
        print(f"{name} digit {d}: distinct {np.count_nonzero(h):3d}  max share {h.max() / w.n:.3f}")
