"""Probe: the sample-sort phases (loopback driver: P virtual ranks on ONE GPU,
same kernels as husky_sort_multi) at scale on C5 and C4, checked against the
single-GPU sort (the order is unique, so the perms must be equal).  Not a bench.

  python tools/loopback_large.py [log2n=26] [P=8]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import checker  # noqa: E402
import paper_2012_00866_b200 as h  # noqa: E402
import workloads as W  # noqa: E402
import workloads.gpu as G  # noqa: E402


def run(name, u, o, P):
    n = o.numel() - 1
    total = int(o[-1].item())
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    su = torch.empty(total + 16, dtype=u.dtype, device="cuda")
    so = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    ws = torch.empty(h.husky_sort_multi_loopback_workspace(0, P, n, total), dtype=torch.uint8, device="cuda")
    t0 = time.time()
    shards, outc = h.husky_sort_multi_loopback(0, P, u, o, perm, su, so, ws)
    torch.cuda.synchronize()
    dt = time.time() - t0
    del ws
    torch.cuda.empty_cache()
    ref, _, _, _ = h.sort(0, u, o)
    torch.cuda.synchronize()
    same = bool(torch.equal(ref[:n], perm))
    ver = checker.verify(u, o, perm, su[:total], so)
    print(json.dumps({"config": name, "n": n, "P": P, "shards": shards, "max_shard_over_mean": round(max(shards) * P / n, 3),
                      "perm_equals_husky_sort": same, "verify": ver, "wall_s": round(dt, 2)}), flush=True)
    assert same and sum(ver.values()) == 0


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    torch.cuda.set_device(0)
    u, o = G.c5_device(1 << lg)
    run("C5", u, o, P)
    del u, o
    w = W.make("C4", 1 << 22)
    u = torch.from_numpy(np.concatenate([w.units, np.zeros(16, np.uint8)])).cuda()
    o = torch.from_numpy(w.offsets).cuda()
    run("C4", u, o, P)


if __name__ == "__main__":
    main()
