"""Generators produce the shapes BASELINE.json's configs describe (CPU only)."""
import numpy as np
import pytest

import workloads as W


def _lens(w):
    return w.offsets[1:] - w.offsets[:-1]


def test_c1_shape():
    w = W.make("C1")
    L = _lens(w)
    assert w.n == 100_000 and L.min() == 4 and L.max() == 12
    assert w.units.min() >= ord("a") and w.units.max() <= ord("z")
    w2 = W.make("C1")
    assert np.array_equal(w.units, w2.units)  # seeded


def test_c2_vocab_and_zipf():
    words = W.c2_vocab(W.MASTER_SEED + 2, 2000)
    assert len(set(words)) == 2000 and max(len(x) for x in words) <= 20
    w = W.c2(200_000, vocab_size=2000)
    L = _lens(w)
    assert L.min() >= 1 and L.max() <= 20
    # the most frequent word has probability 1/H_2000 ~ 12.2%
    strings = {}
    for i in range(0, w.n, 50):
        s = w.units[w.offsets[i]:w.offsets[i + 1]].tobytes()
        strings[s] = strings.get(s, 0) + 1
    top = max(strings.values()) / (w.n / 50)
    assert 0.09 < top < 0.16


def test_c3_shape():
    w = W.c3(50_000)
    L = _lens(w)
    assert w.units.dtype == np.uint16 and L.min() == 2 and L.max() == 4
    assert w.units.min() >= 0x4E00 and w.units.max() <= 0x9FFF


def test_c4_shape():
    w = W.c4(10_000)
    assert (_lens(w) == 24).all()
    u = w.units.reshape(-1, 24)
    assert (u[:, :16] == u[0, :16]).all()
    assert len(np.unique(u[:, 16:], axis=0)) > 9_900


def test_c5_shape():
    w = W.c5(1 << 16)
    L = _lens(w)
    assert L.min() == 8 and L.max() == 24
    assert abs(L.mean() - 16.0) < 0.1
    assert set(np.unique(w.units).tolist()) == set(W.ALNUM.tolist())
    n_sorted = w.meta["sorted"]
    assert n_sorted == (1 << 16) // 10
    s = [w.units[w.offsets[i]:w.offsets[i + 1]].tobytes() for i in range(w.n)]
    assert all(s[i] <= s[i + 1] for i in range(n_sorted - 1))
    assert not all(s[i] <= s[i + 1] for i in range(n_sorted, w.n - 1))
    # ~1% Bernoulli targets; each copies a non-target's string
    assert 0.008 < w.meta["dup"] / w.n < 0.012
    assert w.n - len(set(s)) >= w.meta["dup"] * 0.9


def test_c5_recipe_counter_based():
    """Targets copy the string (length and units) of a non-target position, and
    the content of a position depends only on its identity."""
    seed, N = W.MASTER_SEED + 5, 1 << 20
    pos = np.arange(200_000, 260_000, dtype=np.int64)
    ident = W.c5_ident(seed, N, pos)
    t = W.c5_is_target(seed, pos)
    assert np.array_equal(ident[~t], pos[~t])
    assert (ident[t] != pos[t]).all() and not W.c5_is_target(seed, ident[t]).any()
    assert (ident >= 0).all() and (ident < N).all()
    u1, o1 = W.c5_chars(seed, ident[t][:50], W.c5_len(seed, ident[t][:50]))
    u2, o2 = W.c5_chars(seed, ident[t][:50].copy(), W.c5_len(seed, ident[t][:50]))
    assert np.array_equal(u1, u2) and np.array_equal(o1, o2)


@pytest.mark.parametrize("base,n", [(0, 1000), (3000, 9000), (6000, 500), (65000, 536)])
def test_c5_blocks_of_one_dataset(base, n):
    """Block [base, base + n) of the global dataset equals the same slice of the
    whole dataset (what each rank of a sharded run generates)."""
    N = 1 << 16
    whole = W.c5(N)
    blk = W.c5(n, base=base, n_total=N)
    o = whole.offsets
    assert np.array_equal(blk.units, whole.units[o[base]:o[base + n]])
    assert np.array_equal(blk.offsets, o[base:base + n + 1] - o[base])


def test_d1_groups():
    """D1: every group is one equal-code run (shared 12-unit prefix), shuffled."""
    w = W.d1(50_000, group_min=100, group_max=4096)
    L = _lens(w)
    assert L.min() >= 13 and L.max() <= 22 and w.n == 50_000
    pre = {}
    for i in range(w.n):
        p = w.units[w.offsets[i]:w.offsets[i] + 12].tobytes()
        pre[p] = pre.get(p, 0) + 1
    assert len(pre) == w.meta["groups"]
    assert all(c <= 4096 for c in pre.values()) and sum(c < 100 for c in pre.values()) <= 1  # the last group is cut
