"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, bit-exact.

Everything on the path is integer (no floating point), so the bar is bit
equality of codes, permutation, sorted units and sorted offsets.  Sizes span
several tiles (radix 4096, scan 2048, gather 1024) with ragged tails; the
full BASELINE.json sizes are checked with the oracle's linear uniqueness
verifier (bijection + strictly increasing adjacent pairs <=> equal to the
oracle's sort, because the order is a strict total order).
"""
import os
import random
import zlib

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

ASCII, UNICODE = 0, 1


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


@pytest.fixture(scope="module")
def h():
    import paper_2012_00866_b200 as m
    return m


def to_dev(torch, w):
    u = w.units
    if u.dtype == np.uint16:
        u = u.view(np.int16)
    if u.size == 0:
        u = np.zeros(1, dtype=u.dtype)
    return torch.from_numpy(np.ascontiguousarray(u)).cuda(), torch.from_numpy(w.offsets).cuda()


GUARD = 4096  # elements of guard zone after every output buffer (checked untouched)


def run_sort(torch, h, w, with_units=True):
    """husky_sort through the C ABI with guard zones after perm, sorted units and
    sorted offsets: any write past an output's end fails the test."""
    u, o = to_dev(torch, w)
    n, total = w.n, int(w.offsets[-1] - w.offsets[0])
    ws = torch.empty(h.husky_sort_workspace(w.coder, n, total) + GUARD, dtype=torch.uint8, device="cuda")
    ws.fill_(0xA5)
    perm = torch.full((n + GUARD,), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    su = so = None
    if with_units:
        su = torch.full((total + GUARD,), 0x5A, dtype=u.dtype, device="cuda")
        so = torch.full((n + 1 + GUARD,), 0x5A5A5A5A, dtype=torch.int64, device="cuda")
    outc = h.husky_sort(w.coder, u, o, perm, su, so, ws)
    torch.cuda.synchronize()
    assert bool((perm[n:] == 0x5A5A5A5A).all()), "write past the end of perm"
    p = perm[:n].cpu().numpy().view(np.uint32)
    if with_units:
        assert bool((su[total:] == 0x5A).all()), "write past the end of sorted_units"
        assert bool((so[n + 1:] == 0x5A5A5A5A).all()), "write past the end of sorted_offsets"
        su = su[:total].cpu().numpy()
        if w.coder == UNICODE:
            su = su.view(np.uint16)
        so = so[:n + 1].cpu().numpy()
    return p, su, so, outc


def check_against_oracle(torch, h, oracle_mod, w, with_units=True):
    perm, su, so, outc = run_sort(torch, h, w, with_units)
    ref = oracle_mod.sort(w.coder, w.units, w.offsets)
    assert perm.shape == ref.shape
    bad = np.nonzero(perm != ref)[0]
    assert bad.size == 0, f"{w.name}: first mismatch at {bad[:5]}, got {perm[bad[:5]]} want {ref[bad[:5]]}"
    if with_units:
        rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
        assert np.array_equal(so, rso)
        assert np.array_equal(su, rsu)
    return outc


def rand_wl(seed, n, alphabet, minlen, maxlen, coder=ASCII, prefix=()):
    rng = np.random.default_rng(seed)
    lens = rng.integers(minlen, maxlen + 1, size=n)
    alph = np.asarray(alphabet, dtype=np.uint8 if coder == ASCII else np.uint16)
    strings = []
    for L in lens:
        strings.append(list(prefix) + alph[rng.integers(0, alph.size, size=int(L))].tolist())
    return W.from_strings(strings, coder, name=f"rand{seed}")


# --------------------------------------------------------------------- A1
@pytest.mark.parametrize("name,n", [("C1", 100_000), ("C2", 300_000), ("C3", 300_000), ("C4", 100_000),
                                    ("C5", 1 << 16)])
def test_encode_parity_configs(torch, h, oracle_mod, name, n):
    w = W.make(name, n)
    u, o = to_dev(torch, w)
    codes, perfect = h.husky_encode(w.coder, u, o)
    ref, rperf = oracle_mod.encode(w.coder, w.units, w.offsets)
    assert np.array_equal(codes.cpu().numpy().view(np.uint64), ref)
    assert perfect == rperf


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_encode_parity_edge_units(torch, h, oracle_mod, coder):
    """All unit values incl. > 0x7F (Alg. 4 masks them), empty strings, every
    length 0..20, every start alignment."""
    rng = random.Random(1)
    hi = 255 if coder == ASCII else 0xFFFF
    strings = [[rng.randint(0, hi) for _ in range(L)] for L in range(21) for _ in range(40)]
    strings += [[], [0], [hi] * 12, [0] * 12]
    w = W.from_strings(strings, coder)
    u, o = to_dev(torch, w)
    codes, perfect = h.husky_encode(coder, u, o)
    ref, rperf = oracle_mod.encode(coder, w.units, w.offsets)
    assert np.array_equal(codes.cpu().numpy().view(np.uint64), ref)
    assert perfect == rperf
    # perfect flag boundary (Alg. 3): all lengths <= PL
    pl = 9 if coder == ASCII else 3
    w2 = W.from_strings([[0x61] * k for k in range(pl + 1)] * 50, coder)
    _, p2 = h.husky_encode(coder, *to_dev(torch, w2))
    assert p2 is True


def test_encode_rejects_bad_offsets(torch, h):
    w = W.from_strings([b"abc", b"de"], ASCII)
    u, o = to_dev(torch, w)
    o[1] = 5  # 0, 5, 5 ok; make it decreasing
    o[2] = 4
    with pytest.raises(h.HuskyError) as e:
        h.husky_encode(ASCII, u, o)
    assert e.value.status == 1


# ------------------------------------------------------------ full sort
@pytest.mark.parametrize("n", [0, 1, 2, 3, 17, 1023, 1024, 1025, 2047, 2049, 4095, 4096, 4097, 6143, 6144, 6145,
                               12287, 12289, 18433, 70001, 499_999, 500_000, 614_399, 614_401])
# (below 5e5 keys the radix uses 2048-key tiles, from 5e5 on 6144-key tiles: the
# last four sizes straddle the switch and a ragged 6144-key tail)
def test_sort_sizes_ragged(torch, h, oracle_mod, n):
    w = rand_wl(n, n, range(0x61, 0x65), 0, 14)
    check_against_oracle(torch, h, oracle_mod, w)


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
@pytest.mark.parametrize("case", ["nul_ext", "all_equal", "tiny_alpha", "empties", "long_tail", "sorted",
                                  "reverse"])
def test_sort_degenerate(torch, h, oracle_mod, coder, case):
    rng = random.Random(zlib.crc32(case.encode()) + 7 * coder)
    hi = 0x7F if coder == ASCII else 0xFFFF
    if case == "nul_ext":  # equal codes, order decided by length (short-rule, reading R6)
        base = [[0x61], [0x61, 0], [0x61, 0, 0], [0x61, 0, 0, 0], [0x61, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]]
        strings = [list(rng.choice(base)) for _ in range(5000)]
    elif case == "all_equal":
        strings = [[0x62] * 30] * 9000
    elif case == "tiny_alpha":
        strings = [[rng.choice((0, 1, hi)) for _ in range(rng.randint(0, 12))] for _ in range(9000)]
    elif case == "empties":
        strings = [[] for _ in range(3000)] + [[1]] + [[] for _ in range(3000)]
    elif case == "long_tail":  # long strings (> stage budget per tile for some tiles)
        strings = [[rng.randint(1, hi) for _ in range(rng.choice((1, 5, 300, 2000)))] for _ in range(3000)]
    elif case == "sorted":
        strings = sorted([[rng.randint(0x61, 0x7A) for _ in range(rng.randint(1, 12))] for _ in range(9000)])
    else:
        strings = sorted([[rng.randint(0x61, 0x7A) for _ in range(rng.randint(1, 12))] for _ in range(9000)],
                         reverse=True)
    check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, coder))


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_sort_refinement_subruns_regather(torch, h, oracle_mod, coder):
    """Regression: a giant run whose refinement leaves medium/small dirty sub-runs.
    Their spans may only be re-gathered after the whole giant span (their bases
    move when the refinement reorders the span); guard zones catch overruns."""
    base = [[0x61], [0x61, 0], [0x61, 0, 0], [0x61, 0, 0, 0], [0x61] + [0] * 10, [0x61] + [0] * 3 + [1] * 9]
    for seed in range(12):
        rng = random.Random(seed)
        strings = [list(rng.choice(base)) for _ in range(5000 + 37 * seed)]
        outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, coder))
        assert outc["refine_rounds"] >= 1


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
@pytest.mark.parametrize("group", [2, 7, 32, 33, 500, 4096, 4097, 30000])
def test_sort_dirty_runs_every_class(torch, h, oracle_mod, coder, group):
    """Groups of strings sharing a long common prefix (equal codes) with random
    suffixes in random order: dirty runs of every class -- warp (<=32), CTA
    (<=4096) and giant (refinement rounds, A6)."""
    rng = np.random.default_rng(group + 10 * coder)
    pre = [0x41 + i % 26 for i in range(11)] if coder == ASCII else [0x4E00 + i for i in range(5)]
    alph = np.arange(0x61, 0x64) if coder == ASCII else np.arange(0x4E00, 0x4E03)
    strings = []
    ngroups = max(1, 60000 // group)
    for gi in range(ngroups):
        p = list(pre)
        if coder == ASCII:  # group id inside the 9-unit code window -> distinct codes per group
            p[4], p[5], p[6] = 0x41 + gi % 26, 0x41 + (gi // 26) % 26, 0x41 + (gi // 676) % 26
        else:  # inside the 4-unit window
            p[1] += gi
        for _ in range(group):
            L = int(rng.integers(0, 10))
            strings.append(p + alph[rng.integers(0, alph.size, size=L)].tolist())
    order = rng.permutation(len(strings))
    strings = [strings[i] for i in order]
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, coder))
    assert outc["n_runs"] > 0


def test_sort_giant_run_c4(torch, h, oracle_mod):
    w = W.c4(300_000)
    outc = check_against_oracle(torch, h, oracle_mod, w)
    assert outc["max_run"] == w.n and outc["refine_rounds"] >= 1 and outc["radix_passes"] > 0


@pytest.mark.parametrize("name,n", [("C1", 100_000), ("C2", 1_000_000), ("C3", 1_000_000), ("C5", 1 << 20)])
def test_sort_configs_vs_oracle(torch, h, oracle_mod, name, n):
    check_against_oracle(torch, h, oracle_mod, W.make(name, n))


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_sort_full_size_verifier(torch, h, oracle_mod, name):
    """BASELINE.json full sizes: linear verifier (unique order) + units gather."""
    w = W.make(name)
    perm, su, so, outc = run_sort(torch, h, w)
    assert oracle_mod.verify(w.coder, w.units, w.offsets, perm) == 0
    rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, perm)
    assert np.array_equal(so, rso) and np.array_equal(su, rsu)
    if name == "C2":
        assert outc["runs_by_class"][0] == outc["n_runs"]  # every run already ordered


def test_sort_perm_only_mode(torch, h, oracle_mod):
    w = W.make("C1", 50_000)
    perm, _, _, _ = run_sort(torch, h, w, with_units=False)
    assert np.array_equal(perm, oracle_mod.sort(w.coder, w.units, w.offsets))


def test_sort_off_domain_general_cleanup_and_beyond_window(torch, h, oracle_mod):
    """A unit > 0x7F inside the ASCII code window makes Alg. 4's masked code
    non-monotone (reading R5): the general cleanup (NEXT-4, whole-array
    refinement from unit 0) still yields the exact order; beyond the window the
    exact byte comparator handles any byte."""
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings([b"abc", b"a\x80c", b"a\x00c"] * 7, ASCII))
    assert not outc["domain_ok"] and outc["refine_rounds"] >= 1
    rng = random.Random(4)
    strings = [b"abcdefghi" + bytes(rng.randint(0, 255) for _ in range(rng.randint(0, 6))) for _ in range(5000)]
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, ASCII))
    assert outc["domain_ok"]


@pytest.mark.parametrize("n", [3000, 70_001])
def test_sort_arbitrary_bytes_ascii_coder(torch, h, oracle_mod, n):
    """UTF-8-like arbitrary bytes with the ASCII coder: off-domain everywhere, so
    the general cleanup sorts the whole array (several refinement rounds)."""
    rng = np.random.default_rng(n)
    strings = [rng.integers(0, 256, size=int(rng.integers(0, 30))).tolist() for _ in range(n)]
    strings += [strings[i] for i in range(0, n, 7)]  # duplicates
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, ASCII))
    assert not outc["domain_ok"]


def test_sort_offsets_not_starting_at_zero(torch, h, oracle_mod):
    w = W.make("C1", 20_000)
    pad = np.concatenate([np.full(13, 0x7A, dtype=np.uint8), w.units])
    w2 = W.Workload("shifted", ASCII, pad, w.offsets + 13, {})
    perm, su, so, _ = run_sort(torch, h, w2)
    ref = oracle_mod.sort(ASCII, w.units, w.offsets)
    assert np.array_equal(perm, ref)
    rsu, rso = oracle_mod.gather(ASCII, w.units, w.offsets, ref)
    assert np.array_equal(su, rsu) and np.array_equal(so, rso)


def test_sort_host_api(torch, h, oracle_mod):
    w = W.make("C3", 200_000)
    n, tot = w.n, w.units.size
    ws = torch.empty(h.husky_sort_host_workspace(w.coder, n, tot), dtype=torch.uint8, device="cuda")
    perm = np.zeros(n, dtype=np.uint32)
    su = np.zeros(tot, dtype=np.uint16)
    so = np.zeros(n + 1, dtype=np.int64)
    h.husky_sort_host(w.coder, w.units, w.offsets, perm, su, so, ws)
    ref = oracle_mod.sort(w.coder, w.units, w.offsets)
    assert np.array_equal(perm, ref)
    rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
    assert np.array_equal(su, rsu) and np.array_equal(so, rso)


def test_sort_repeatable_and_workspace_reuse(torch, h):
    w = W.make("C2", 200_000)
    u, o = to_dev(torch, w)
    ws = torch.empty(h.husky_sort_workspace(0, w.n), dtype=torch.uint8, device="cuda")
    ws.fill_(0xAB)  # garbage workspace contents must not matter
    a = h.sort(0, u, o, ws=ws)[0].clone()
    ws.fill_(0x5C)
    b = h.sort(0, u, o, ws=ws)[0]
    assert torch.equal(a, b)


# ------------------------------------------------------- sharded (loopback)
@pytest.mark.parametrize("exchange", ["peer", "copy"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("name,n", [("C1", 60_000), ("C3", 100_000), ("C4", 50_000), ("C2", 80_000)])
def test_multi_loopback_vs_oracle(torch, h, oracle_mod, monkeypatch, exchange, world, name, n):
    """Sample sort over `world` virtual ranks on one GPU: concatenation of the
    shards == oracle; equal strings never straddle shards; shard sizes follow
    the splitter rule; C4 (all codes equal) spreads evenly.  Both transports:
    the peer-store gather into per-rank windows (NEXT-2) and copies."""
    monkeypatch.setenv("HUSKY_EXCHANGE", exchange)
    w = W.make(name, n)
    u, o = to_dev(torch, w)
    tot = w.units.size
    ws = torch.empty(h.husky_sort_multi_loopback_workspace(w.coder, world, w.n, tot), dtype=torch.uint8,
                     device="cuda")
    perm = torch.empty(w.n, dtype=torch.int32, device="cuda")
    su = torch.empty(tot + 8, dtype=u.dtype, device="cuda")
    so = torch.empty(w.n + 1, dtype=torch.int64, device="cuda")
    shards, outc = h.husky_sort_multi_loopback(w.coder, world, u, o, perm, su, so, ws)
    assert outc["exchange"] == (4 if exchange == "peer" else 3)
    assert sum(shards) == w.n
    p = perm.cpu().numpy().view(np.uint32)
    ref = oracle_mod.sort(w.coder, w.units, w.offsets)
    assert np.array_equal(p, ref)
    rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
    s_u = su[:tot].cpu().numpy()
    if w.coder == UNICODE:
        s_u = s_u.view(np.uint16)
    assert np.array_equal(so.cpu().numpy(), rso) and np.array_equal(s_u, rsu)
    # shard boundaries never split equal strings (composite splitters may split
    # equal-code runs), and the shard sizes are those of the splitter rule
    # (husky_select_splitters, host copy) applied to the same samples
    strs = w.strings()
    b = np.cumsum(shards)[:-1]
    b = b[(b > 0) & (b < w.n)]
    assert not any(strs[ref[i]] == strs[ref[i - 1]] for i in b)
    assert list(shards) == expected_shards(h, w, world)
    if name == "C4" and world > 1:  # all codes collide: still balanced (NEXT-1)
        assert max(shards) <= 2 * w.n / world


def expected_shards(h, w, world, s=4096, cap=32):
    """Shard sizes of the sample sort by its documented rule: rank r holds
    block [n*r/P, n*(r+1)/P); samples at local positions i*n_r/s, each the
    string's first <= 32 units; splitters by husky_select_splitters; bucket(x) =
    number of splitter strings <= x in the sort order."""
    import bisect
    n = w.n
    strs = w.strings()
    samples = []
    for r in range(world):
        lo, hi = n * r // world, n * (r + 1) // world
        nl = hi - lo
        if nl == 0:
            continue
        samples += [list(strs[lo + i * nl // s][:cap]) for i in range(s)]
    if world == 1:
        return [n]
    sw = W.from_strings(samples, w.coder)
    idx = h.husky_select_splitters(w.coder, sw.units, sw.offsets, world)
    spl = [tuple(samples[int(i)]) for i in idx]
    counts = [0] * world
    for x in strs:
        counts[bisect.bisect_right(spl, x)] += 1
    return counts


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_multi_nccl_single_rank(torch, h, oracle_mod, monkeypatch, exchange):
    """The NCCL plan/exec path with a one-rank communicator, through the
    symmetric-window peer stores (NEXT-2) and through ncclSend/ncclRecv; the
    window is reused and grown across calls of different sizes."""
    monkeypatch.setenv("HUSKY_EXCHANGE", exchange)
    uid = h.husky_comm_unique_id()
    comm = h.husky_comm_create(0, 1, uid)
    try:
        for name, n in (("C1", 30_000), ("C3", 20_000), ("C2", 90_000)):
            w = W.make(name, n)
            u, o = to_dev(torch, w)
            perm, su, so, outc = h.sort_multi(comm, w.coder, u, o, 0)
            torch.cuda.synchronize()
            assert outc["exchange"] == (2 if exchange == "peer" else 1)
            ref = oracle_mod.sort(w.coder, w.units, w.offsets)
            assert np.array_equal(perm.cpu().numpy().view(np.uint32), ref)
            rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
            s_u = su.cpu().numpy()
            if w.coder == UNICODE:
                s_u = s_u.view(np.uint16)
            assert np.array_equal(so.cpu().numpy(), rso) and np.array_equal(s_u[:rsu.size], rsu)
    finally:
        h.husky_comm_destroy(comm)


@pytest.mark.parametrize("world", [3, 7])
def test_multi_loopback_peer_edges(torch, h, oracle_mod, monkeypatch, world):
    """Peer-store exchange edge cases: empty buckets (half the strings equal),
    empty strings, strings longer than the gather's shared-memory window (one
    tile over several windows, bucket boundaries inside a window)."""
    monkeypatch.setenv("HUSKY_EXCHANGE", "peer")
    rng = np.random.default_rng(world)
    strings = []
    for i in range(30_000):
        r = rng.random()
        if r < 0.5:
            strings.append([0x61, 0x62, 0x63])
        elif r < 0.55:
            strings.append([])
        elif r < 0.56:
            strings.append(rng.integers(0x61, 0x7B, size=int(rng.integers(2000, 9000))).tolist())
        else:
            strings.append(rng.integers(0x61, 0x65, size=int(rng.integers(1, 30))).tolist())
    w = W.from_strings(strings, ASCII)
    u, o = to_dev(torch, w)
    tot = w.units.size
    ws = torch.empty(h.husky_sort_multi_loopback_workspace(w.coder, world, w.n, tot), dtype=torch.uint8,
                     device="cuda")
    perm = torch.empty(w.n, dtype=torch.int32, device="cuda")
    su = torch.empty(tot + 8, dtype=u.dtype, device="cuda")
    so = torch.empty(w.n + 1, dtype=torch.int64, device="cuda")
    shards, outc = h.husky_sort_multi_loopback(w.coder, world, u, o, perm, su, so, ws)
    assert outc["exchange"] == 4 and sum(shards) == w.n
    ref = oracle_mod.sort(w.coder, w.units, w.offsets)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), ref)
    rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
    assert np.array_equal(so.cpu().numpy(), rso) and np.array_equal(su[:tot].cpu().numpy(), rsu)


def test_sort_host_many_pipelined(torch, h, oracle_mod):
    """The pipelined host API: several batches (different configs and sizes,
    one empty) through 1, 2 and 3 workspace slots, each bit-exact against the
    oracle (three streams: H2D copies, kernels, D2H copies)."""
    wls = [W.make("C1", 50_000), W.make("C3", 70_000), W.make("C2", 120_000),
           W.from_strings([], ASCII), W.make("C1", 3)]
    for depth in (1, 2, 3):
        for coder in (ASCII, UNICODE):
            sel = [w for w in wls if w.coder == coder]
            batches = []
            for w in sel:
                tot = int(w.offsets[-1] - w.offsets[0]) if w.n else 0
                batches.append((w.units if w.units.size else np.zeros(1, w.units.dtype), w.offsets,
                                np.zeros(max(w.n, 1), np.uint32), np.zeros(tot + 8, w.units.dtype),
                                np.zeros(w.n + 1, np.int64)))
            n_max = max(w.n for w in sel)
            u_max = max(int(w.offsets[-1] - w.offsets[0]) if w.n else 0 for w in sel)
            ws = torch.empty(h.husky_sort_host_many_workspace(coder, n_max, u_max, depth), dtype=torch.uint8,
                             device="cuda")
            h.husky_sort_host_many(coder, batches, ws, depth)
            for w, b in zip(sel, batches):
                ref = oracle_mod.sort(w.coder, w.units, w.offsets)
                assert np.array_equal(b[2][:w.n], ref)
                rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
                assert np.array_equal(b[4], rso)
                assert np.array_equal(b[3][:rsu.size], rsu)


@pytest.mark.parametrize("depth", [1, 2])
def test_sort_host_many_growing_batches_pinned(torch, h, oracle_mod, depth):
    """Pinned host buffers and batches that GROW within a slot: a later batch's
    input copy must not land on an earlier batch's outputs while they are still
    being copied to the host (the slot layout is sized by the largest batch)."""
    sizes = [20_000, 60_000, 150_000, 300_000, 40_000, 500_000]
    wls = [W.make("C1", n) for n in sizes]
    batches = []
    for w in wls:
        tot = int(w.offsets[-1])
        batches.append((torch.from_numpy(w.units).pin_memory(), torch.from_numpy(w.offsets).pin_memory(),
                        torch.zeros(w.n, dtype=torch.int32).pin_memory(),
                        torch.zeros(tot + 8, dtype=torch.uint8).pin_memory(),
                        torch.zeros(w.n + 1, dtype=torch.int64).pin_memory()))
    ws = torch.empty(h.husky_sort_host_many_workspace(ASCII, max(sizes), max(int(w.offsets[-1]) for w in wls), depth),
                     dtype=torch.uint8, device="cuda")
    h.husky_sort_host_many(ASCII, batches, ws, depth)
    torch.cuda.synchronize()
    for w, b in zip(wls, batches):
        ref = oracle_mod.sort(ASCII, w.units, w.offsets)
        assert np.array_equal(b[2].numpy().view(np.uint32), ref)
        rsu, rso = oracle_mod.gather(ASCII, w.units, w.offsets, ref)
        assert np.array_equal(b[4].numpy(), rso)
        assert np.array_equal(b[3].numpy()[:rsu.size], rsu)


@pytest.mark.parametrize("world", [2, 5])
def test_multi_loopback_off_domain(torch, h, oracle_mod, world):
    """Off-domain ASCII bytes through the sample sort: buckets compare strings
    only (codes are not monotone there) and every shard runs the general
    cleanup; the concatenation is the oracle's order."""
    rng = np.random.default_rng(world)
    strings = [rng.integers(0, 256, size=int(rng.integers(0, 14))).tolist() for _ in range(40_000)]
    w = W.from_strings(strings, ASCII)
    u, o = to_dev(torch, w)
    tot = w.units.size
    ws = torch.empty(h.husky_sort_multi_loopback_workspace(w.coder, world, w.n, tot), dtype=torch.uint8,
                     device="cuda")
    perm = torch.empty(w.n, dtype=torch.int32, device="cuda")
    su = torch.empty(tot + 8, dtype=u.dtype, device="cuda")
    so = torch.empty(w.n + 1, dtype=torch.int64, device="cuda")
    shards, outc = h.husky_sort_multi_loopback(w.coder, world, u, o, perm, su, so, ws)
    ref = oracle_mod.sort(w.coder, w.units, w.offsets)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), ref)
    assert sum(shards) == w.n and max(shards) < w.n


def test_programmatic_launch_off_matches(torch, h, tmp_path):
    """HUSKY_PDL=0 (plain launches, read once per process) sorts exactly like
    the default programmatic dependent launches: run in a subprocess."""
    import subprocess
    import sys
    w = W.make("C2", 200_000)
    u, o = to_dev(torch, w)
    p_pdl = h.sort(w.coder, u, o)[0].cpu().numpy()
    script = tmp_path / "nopdl.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})\n"
        "import paper_2012_00866_b200 as h, workloads as W\n"
        "w = W.make('C2', 200_000)\n"
        "u = torch.from_numpy(w.units).cuda(); o = torch.from_numpy(w.offsets).cuda()\n"
        f"np.save({repr(str(tmp_path / 'p.npy'))}, h.sort(w.coder, u, o)[0].cpu().numpy())\n")
    env = dict(os.environ, HUSKY_PDL="0")
    r = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert np.array_equal(np.load(tmp_path / "p.npy"), p_pdl)


# ---------------------------------------------------------------- slab records
@pytest.mark.parametrize("name,n", [("C1", 70_001), ("C2", 300_000), ("C3", 200_003), ("C4", 50_000),
                                    ("C5", 300_000)])
def test_slab_records_forced(torch, h, oracle_mod, monkeypatch, name, n):
    """The gather's slab path (one 16-B record per string: length + the units
    after the code window) forced at sizes where it is normally off; bit-exact
    against the oracle for every config (packed: only strings longer than PL
    have records)."""
    monkeypatch.setenv("HUSKY_SLAB", "1")
    check_against_oracle(torch, h, oracle_mod, W.make(name, n))


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_slab_record_boundaries(torch, h, oracle_mod, monkeypatch, coder):
    """Lengths around the record's capacity (ASCII 24 / UNICODE 10 units: longer
    strings fall back to offsets + units), around PL and S, empty strings, NUL
    and extreme units, shared prefixes (equal codes: the order check compares
    slab-staged bytes)."""
    monkeypatch.setenv("HUSKY_SLAB", "1")
    rng = np.random.default_rng(77 + coder)
    hi = 0x7F if coder == ASCII else 0xFFFF
    cap = 24 if coder == ASCII else 10
    lens = [0, 1, 2, 3, 4, 8, 9, 10, cap - 1, cap, cap + 1, cap + 7, 40]
    strings = []
    prefix = rng.integers(1, hi, size=50).tolist()
    for i in range(60_000):
        L = int(lens[i % len(lens)])
        if i % 3 == 0:
            s = prefix[:L]  # shared prefixes: equal codes, exact compare from unit S
            if L and i % 6 == 0:
                s = s[:-1] + [int(rng.integers(0, hi + 1))]
        else:
            s = rng.integers(0, hi + 1, size=L).tolist()
        strings.append(s)
    w = W.from_strings(strings, coder)
    check_against_oracle(torch, h, oracle_mod, w)


# --------------------------------------------------------- alphabet compression
@pytest.mark.parametrize("alpha", [1, 2, 26, 31, 32, 33, 62, 63, 64, 100])
def test_alphabet_compression_sizes(torch, h, oracle_mod, alpha):
    """ASCII keys re-packed as field ranks (cbits = ceil(log2(#values incl. 0))):
    alphabet sizes around the 5/6/7-bit boundaries (63 values + padding = 64 is
    the last one that compresses), NUL among them, lengths 0..14 so padding
    and truncation occur; bit-exact against the oracle (perm, sorted units --
    the gather rebuilds units from the compressed codes)."""
    rng = np.random.default_rng(1000 + alpha)
    vals = rng.choice(np.arange(0, 128), size=alpha, replace=False)
    strings = [rng.choice(vals, size=int(rng.integers(0, 15))).tolist() for _ in range(120_000)]
    w = W.from_strings(strings, ASCII)
    outc = check_against_oracle(torch, h, oracle_mod, w)
    if alpha <= 31:  # main key sort: at most 6 passes (refinement passes come on top of radix_passes)
        assert outc["keys_partitioned"] <= 6 * w.n


def test_alphabet_compression_off_matches(torch, h, oracle_mod, monkeypatch):
    """HUSKY_ALPHA=0 (raw 7-bit fields) sorts C1 identically, with more passes."""
    w = W.make("C1", 200_000)
    on = check_against_oracle(torch, h, oracle_mod, w)
    monkeypatch.setenv("HUSKY_ALPHA", "0")
    off = check_against_oracle(torch, h, oracle_mod, w)
    assert on["keys_partitioned"] < off["keys_partitioned"]


# ------------------------------------------------------------------ CUDA graphs
@pytest.mark.parametrize("name,n", [("C1", 100_000), ("C3", 70_001), ("C4", 30_000)])
def test_graph_replay_same_buffers_new_content(torch, h, oracle_mod, name, n):
    """Repeated calls with the same buffers replay a cached CUDA graph of the
    launch sequence: results must follow the CURRENT input content (a second
    dataset of the same shape written into the same buffers), including the
    refinement that runs after the graph (C4's giant run)."""
    w1 = W.make(name, n)
    # same shape, different content: the strings in reverse order
    rev = np.arange(n)[::-1]
    lens = (w1.offsets[1:] - w1.offsets[:-1])[rev]
    off2 = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off2[1:])
    units2 = np.concatenate([w1.units[w1.offsets[i]:w1.offsets[i + 1]] for i in rev])
    w2 = W.Workload(name, w1.coder, units2, off2, {})
    u, o = to_dev(torch, w1)
    total = int(w1.offsets[-1])
    ws = torch.empty(h.husky_sort_workspace(w1.coder, n, total), dtype=torch.uint8, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    su = torch.empty(total + 64, dtype=u.dtype, device="cuda")
    so = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    for w in (w1, w1, w2, w1, w2):
        uu, oo = to_dev(torch, w)
        u.copy_(uu)
        o.copy_(oo)
        h.husky_sort(w.coder, u, o, perm, su, so, ws)
        torch.cuda.synchronize()
        ref = oracle_mod.sort(w.coder, w.units, w.offsets)
        assert np.array_equal(perm.cpu().numpy().view(np.uint32), ref)
        rsu, rso = oracle_mod.gather(w.coder, w.units, w.offsets, ref)
        gsu = su[:total].cpu().numpy()
        if w.coder == UNICODE:
            gsu = gsu.view(np.uint16)
        assert np.array_equal(so.cpu().numpy(), rso) and np.array_equal(gsu, rsu)


def test_graph_off_matches(torch, h, oracle_mod, monkeypatch):
    """HUSKY_GRAPH=0 (direct launches) gives the same bytes as the graph path."""
    w = W.make("C2", 200_000)
    a = run_sort(torch, h, w)
    monkeypatch.setenv("HUSKY_GRAPH", "0")
    b = run_sort(torch, h, w)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


# ------------------------------------------------ staged fix-up (A5, fixup.cu)
@pytest.mark.parametrize("coder,gmax,smax", [(ASCII, 4096, 10), (ASCII, 32, 6), (UNICODE, 4096, 8),
                                             (ASCII, 4096, 40), (UNICODE, 2000, 40)])
def test_staged_fixup_dirty_runs(torch, h, oracle_mod, coder, gmax, smax):
    """D1-shaped input: many equal-code runs of 100..gmax strings, all dirty.
    Runs whose units fit the 96 KB stage are sorted in shared memory from one
    bulk copy and written back in place; longer ones (suffixes up to 40 units:
    4096 x 52 B > 96 KB) take the global-memory kernels + re-gather.  Bit-exact
    against the oracle either way."""
    w = W.d1(150_000, group_min=min(100, gmax), group_max=gmax, suffix_max=smax, coder=coder)
    outc = check_against_oracle(torch, h, oracle_mod, w)
    assert outc["runs_by_class"][0] < outc["n_runs"]  # the runs were dirty
    # perm-only mode: the runs' strings are gathered into the stage from the
    # input (perm -> offsets -> units) and only perm is written back
    check_against_oracle(torch, h, oracle_mod, w, with_units=False)


def test_staged_fixup_ties_nul_and_prefixes(torch, h, oracle_mod):
    """Runs whose strings tie on the 8-byte key: shared suffix prefixes, NUL
    units, proper prefixes, exact duplicates (index tie-break)."""
    rng = np.random.default_rng(91)
    strings = []
    for i in range(60_000):
        g = i % 37  # 37 runs of ~1600 strings: a distinct 9-unit prefix (code) each
        tail = [0x61 + g % 3] * int(rng.integers(0, 12)) + rng.integers(0, 3, size=int(rng.integers(0, 4))).tolist()
        strings.append([0x61 + g // 26, 0x61 + g % 26] + [0x61] * 7 + tail)
    perm = rng.permutation(len(strings))
    w = W.from_strings([strings[p] for p in perm], ASCII)
    check_against_oracle(torch, h, oracle_mod, w)
    check_against_oracle(torch, h, oracle_mod, w, with_units=False)


@pytest.mark.parametrize("with_units", [True, False])
def test_refinement_medium_subruns(torch, h, oracle_mod, with_units):
    """A giant run (every code equal) whose refinement leaves medium sub-runs
    (groups of 100..3000 strings equal on the 7-unit refinement window and
    dirty past it): the sub-runs take the gather-staged fix-up, then the span
    is gathered again (with sorted strings)."""
    rng = np.random.default_rng(17)
    strings = []
    while len(strings) < 40_000:
        g = int(rng.integers(100, 3000))
        head = [0x61] * 12 + rng.integers(0x61, 0x7B, size=7).tolist()
        for _ in range(g):
            strings.append(head + rng.integers(0x61, 0x7B, size=int(rng.integers(1, 9))).tolist())
    strings = strings[:40_000]
    perm = rng.permutation(len(strings))
    w = W.from_strings([strings[p] for p in perm], ASCII)
    outc = check_against_oracle(torch, h, oracle_mod, w, with_units=with_units)
    assert outc["refine_rounds"] >= 1


# ------------------------------------- partial key sort (lowest digit unsorted)
@pytest.mark.parametrize("name,n", [("C1", 100_000), ("C2", 300_000), ("C5", 300_000), ("C4", 40_000),
                                    ("D1", 150_000), ("C3", 300_000)])
def test_lowest_digit_unsorted_forced(torch, h, oracle_mod, monkeypatch, name, n):
    """HUSKY_SKIP=2 leaves the lowest varying digit of the ASCII / UNICODE keys unsorted
    whenever the plan allows (R19): run detection then compares keys under the
    mask, equal masked keys fix fewer leading units and the short rule shrinks
    with them; every extra equal-key pair is resolved by the run machinery.
    Bit-exact against the oracle, with fewer key-sort passes."""
    w = W.make(name, n)
    monkeypatch.setenv("HUSKY_SKIP", "0")
    ref = check_against_oracle(torch, h, oracle_mod, w)
    monkeypatch.setenv("HUSKY_SKIP", "2")
    forced = check_against_oracle(torch, h, oracle_mod, w)
    if ref["keys_partitioned"] >= 2 * n:
        assert forced["keys_partitioned"] == ref["keys_partitioned"] - n
    # two digits (HUSKY_SKIP=3): many more equal masked keys, fewer fixed units;
    # the extra pairs are tiny dirty runs (a thread each, fixup.cu fix_tiny)
    monkeypatch.setenv("HUSKY_SKIP", "3")
    forced2 = check_against_oracle(torch, h, oracle_mod, w)
    if ref["keys_partitioned"] >= 3 * n:
        assert forced2["keys_partitioned"] == ref["keys_partitioned"] - 2 * n


@pytest.mark.parametrize("seed", range(0, 300, 7))
@pytest.mark.parametrize("skip", ["2", "3"])
def test_lowest_digit_unsorted_fuzz(torch, h, oracle_mod, monkeypatch, seed, skip):
    """The fuzz cases (every coder, NULs, prefixes, duplicates, ragged sizes)
    with the partial key sort forced (one / two digits)."""
    import test_gpu_fuzz as F
    monkeypatch.setenv("HUSKY_SKIP", skip)
    check_against_oracle(torch, h, oracle_mod, F._case(1000 + seed))


@pytest.mark.parametrize("n", [5_000, 70_001])
def test_tiny_runs_lane_fixup(torch, h, oracle_mod, n):
    """Dirty runs of 2, 3 and 4 strings (a thread each: fix_tiny and the
    lane re-gather) beside runs of 5..32 (a warp each), all sharing their
    9-unit prefix (equal codes) and differing later, in shuffled order."""
    rng = np.random.default_rng(n)
    strings = []
    while len(strings) < n:
        size = int(rng.choice([2, 3, 4, 5, 9, 32]))
        head = rng.integers(0x61, 0x7B, size=9).tolist()
        for _ in range(size):
            strings.append(head + rng.integers(0x61, 0x64, size=int(rng.integers(0, 6))).tolist())
    strings = strings[:n]
    perm = rng.permutation(len(strings))
    w = W.from_strings([strings[p] for p in perm], ASCII)
    out = check_against_oracle(torch, h, oracle_mod, w)
    assert out["runs_by_class"][1] > 0
    check_against_oracle(torch, h, oracle_mod, w, with_units=False)  # perm-only mode


def test_refinement_partial_sort_with_giant_cluster(torch, h, oracle_mod):
    """The refinement's partial sort (the key2 windows sorted on their first 5
    units when the entropy rule allows): one giant run (a shared 16-unit prefix,
    so every code is equal) whose suffixes are mostly random -- the rule takes
    the partial sort -- plus a cluster of 10,000 strings sharing the next 5 units
    and differing only in the 2 masked ones and beyond: that cluster is a giant
    run under the mask and is refined again from 5 units further, not 7."""
    rng = np.random.default_rng(21)
    alpha = np.frombuffer(b"0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz", dtype=np.uint8)
    prefix = list(b"SHARED-PREFIX-16")
    strings = [prefix + alpha[rng.integers(0, 62, size=8)].tolist() for _ in range(90_000)]
    head = list(b"QQQQQ")
    strings += [prefix + head + alpha[rng.integers(0, 62, size=int(rng.integers(0, 6)))].tolist()
                for _ in range(10_000)]
    order = rng.permutation(len(strings))
    w = W.from_strings([strings[i] for i in order], ASCII)
    outc = check_against_oracle(torch, h, oracle_mod, w)
    assert outc["refine_rounds"] >= 2
