"""Probe: the sharded path (sample sort) through a one-rank communicator on one
B200 -- per-launch times of one step (profiler mode 1) against the step's
CUDA-event time, so host-side gaps show up.  Not a bench line.

  python tools/multi_probe.py [log2n=27] [config=C5]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_00866_b200 as h  # noqa: E402
import workloads.gpu as G  # noqa: E402


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    torch.cuda.set_device(0)
    u, o = G.c5_device(1 << lg)
    comm = h.husky_comm_create(0, 1, h.husky_comm_unique_id())
    for _ in range(3):
        h.sort_multi(comm, 0, u, o, 0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        h.sort_multi(comm, 0, u, o, 0)
        b.record()
        torch.cuda.synchronize()
        ts.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    single = []
    perm = torch.empty(o.numel() - 1, dtype=torch.int32, device="cuda")
    su = torch.empty(u.numel() + 16, dtype=u.dtype, device="cuda")
    so = torch.empty(o.numel(), dtype=torch.int64, device="cuda")
    ws = torch.empty(h.husky_sort_workspace(0, o.numel() - 1, u.numel()), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.husky_sort(0, u, o, perm, su, so, ws)
        b.record()
        torch.cuda.synchronize()
        single.append(a.elapsed_time(b))
    h.husky_profile_reset()
    h.husky_profile_enable(1)
    h.sort_multi(comm, 0, u, o, 0)
    torch.cuda.synchronize()
    h.husky_profile_enable(False)
    L = h.husky_profile_launches()
    print(json.dumps({"n": 1 << lg, "multi_ms_event_wall": ts, "single_ms": single,
                      "launch_sum_ms": round(sum(x[2] for x in L), 3)}))
    for st, el, ms in L:
        print(f"{st:14s} {el:12d} {ms:9.3f}")
    h.husky_comm_destroy(comm)


if __name__ == "__main__":
    main()
