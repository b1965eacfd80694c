"""The N>1 sample-sort path on CPU: world_size-2 gloo process groups.

The data-path kernels need a GPU, so here the per-rank steps that run on the
device are stood in for by the oracle (test infrastructure), while the
cross-rank logic is exercised for real across processes: regular sampling (the
k_sample rule: the string prefix at i*n/s), the library's host splitter
selection (husky_select_splitters, C ABI), bucket = #splitters <= string, the count
exchange, the string exchange in source-rank order, and the rank-order
concatenation.  Checks: concatenation == oracle global sort; equal strings never
straddle ranks; shard sizes add up.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

S = 4096  # kSamplesPerRank in csrc/multi.cu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2012_00866_b200 as h
        import workloads as W
        wl = W.make(name, n) if name != "empty_rank" else W.make("C1", n)
        N = wl.n
        base = [0, N] if name == "empty_rank" else [N * r // world for r in range(world + 1)]
        if name == "empty_rank":
            base = [0] + [N] * world  # rank 0 holds everything, the others nothing
        lo, hi = base[rank], base[rank + 1]
        off = wl.offsets[lo:hi + 1]
        units = wl.units
        codes, _ = oracle.encode(wl.coder, units, off) if hi > lo else (np.zeros(0, np.uint64), True)
        nl = hi - lo
        # sample strings: the first <= 32 units of the strings at i*nl/S
        smp = [tuple(units[off[i * nl // S]:off[i * nl // S + 1]][:32].tolist()) for i in range(S)] if nl else []
        gathered = [None] * world
        dist.all_gather_object(gathered, smp)
        allsmp = [x for g in gathered for x in g]  # rank-major
        sw = W.from_strings([list(x) for x in allsmp], wl.coder)
        idx = h.husky_select_splitters(wl.coder, sw.units, sw.offsets, world)  # the library's rule
        spl = [allsmp[int(i)] for i in idx]
        import bisect
        mine = [tuple(units[off[i]:off[i + 1]].tolist()) for i in range(nl)]
        bucket = np.array([bisect.bisect_right(spl, x) for x in mine], dtype=np.int64)
        # stable partition -> per destination (units, lengths, global indices)
        send = []
        for d in range(world):
            idx = np.nonzero(bucket == d)[0]
            strs = [units[off[i]:off[i + 1]] for i in idx]
            send.append((strs, (lo + idx).astype(np.int64)))
        # the count matrix is all-gathered (row q = rank q's (strings, units) per
        # destination); a rank's displacement in destination d's window is the
        # sum of rows q < rank, column d -- the peer-store exchange (NEXT-2)
        cnt = torch.tensor([[len(send[d][0]), int(sum(len(x) for x in send[d][0]))] for d in range(world)],
                           dtype=torch.int64)
        mat = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(mat, cnt)
        mat = torch.stack(mat).numpy()  # [src][dst][2]
        disp_n = mat[:rank, :, 0].sum(axis=0)
        disp_u = mat[:rank, :, 1].sum(axis=0)
        n_in, u_in = int(mat[:, rank, 0].sum()), int(mat[:, rank, 1].sum())
        # window of this rank, filled by every source at its displacement
        win_lens = np.full(n_in, -1, np.int64)
        win_gidx = np.full(n_in, -1, np.int64)
        win_units = np.full(u_in, -1, np.int64)
        for src in range(world):
            obj = [[(disp_n[d], disp_u[d], send[d]) for d in range(world)]] if src == rank else [None]
            dist.broadcast_object_list(obj, src=src)
            dn, du, (strs_s, gidx_s) = obj[0][rank]
            for k, x in enumerate(strs_s):
                assert win_lens[dn + k] == -1  # no overlap
                win_lens[dn + k] = len(x)
                win_gidx[dn + k] = gidx_s[k]
                win_units[du:du + len(x)] = x
                du += len(x)
        assert (win_lens >= 0).all() and (win_units >= 0).all()  # no gap
        ends = np.concatenate([[0], np.cumsum(win_lens)])
        strs = [win_units[ends[i]:ends[i + 1]].astype(units.dtype) for i in range(n_in)]
        gidx = win_gidx
        assert np.all(np.diff(gidx) > 0)  # source-rank order == ascending global index
        lw = W.from_strings([list(s) for s in strs], wl.coder)
        lperm = oracle.sort(wl.coder, lw.units, lw.offsets) if strs else np.zeros(0, np.uint32)
        shard = gidx[lperm] if strs else np.zeros(0, np.int64)
        shard_strs = [tuple(strs[i].tolist()) for i in lperm] if strs else []
        out = [None] * world
        dist.all_gather_object(out, (shard, shard_strs))
        if rank == 0:
            cat = np.concatenate([o[0] for o in out])
            ref = oracle.sort(wl.coder, wl.units, wl.offsets).astype(np.int64)
            ok = np.array_equal(cat, ref)
            straddle = any(len(out[r][1]) and len(out[r + 1][1]) and out[r][1][-1] == out[r + 1][1][0]
                           for r in range(world - 1))
            q.put((ok, straddle, [len(o[0]) for o in out]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("C1", 30_000), ("C3", 30_000), ("C4", 5_000), ("empty_rank", 5_000)])
def test_sample_sort_world2_gloo(name, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    ok, straddle, sizes = q.get(timeout=10)
    assert ok, "concatenation of shards != oracle global sort"
    assert not straddle, "equal strings straddle two ranks"
    assert sum(sizes) == n
    if name == "C4":  # every code collides, yet the string splitters balance the shards (NEXT-1)
        assert max(sizes) <= 0.6 * n
