"""Pins for the oracle's NEXT-3 additions (no GPU): the English 5-bit / 6-bit
coders (parameters per SPEC.md:224-240, reading R15) and the
numeric-key sort for perfect codings (PAPER.md:213-217, SPEC.md:264-275,
reading R16).  Pinned against closed forms (a sum, not the oracle's fold), the
worked values in tests/golden (test_oracle_pins.py), sorted-scan and grouping
checks over exhaustive tiny alphabets, the paper's capacity claims, Python's
library sort, and numpy's stable argsort."""
import functools
import itertools
import math
import random
import struct

import numpy as np
import pytest

import workloads as W

E5, E6 = 2, 3


def _codes(oracle_mod, strings, coder):
    w = W.from_strings(strings, coder)
    codes, perfect = oracle_mod.encode(coder, w.units, w.offsets)
    return [int(c) for c in codes], perfect


def cf_english5(s):
    """Alg. 4 with (12, 5, 0x1F) as a sum."""
    return sum((s[i] & 0x1F) << (5 * (11 - i)) for i in range(min(len(s), 12)))


def cf_english6(s):
    """Alg. 4 with (10, 6, 0x3F) as a sum."""
    return sum((s[i] & 0x3F) << (6 * (9 - i)) for i in range(min(len(s), 10)))


@pytest.mark.parametrize("coder,cf", [(E5, cf_english5), (E6, cf_english6)])
def test_closed_form_random(oracle_mod, coder, cf):
    rng = random.Random(11 + coder)
    strings = [[rng.randint(0, 255) for _ in range(rng.randint(0, 16))] for _ in range(5000)]
    strings += [[0xFF] * k for k in range(14)] + [[0x7A] * k for k in range(14)]
    codes, _ = _codes(oracle_mod, strings, coder)
    for s, c in zip(strings, codes):
        assert c == cf(s), s
    assert max(codes) < 2**60  # 12 x 5 = 10 x 6 = 60 bits


def _all_strings(alphabet, maxlen):
    out = [()]
    for L in range(1, maxlen + 1):
        out += list(itertools.product(alphabet, repeat=L))
    return out


def _sorted_scan_and_collisions(oracle_mod, coder, alphabet, maxlen, K):
    """Over EVERY string of the alphabet up to maxlen (> K, so truncation is
    exercised): codes are non-decreasing along the library's lexicographic
    order (== weak monotonicity over all pairs), and code(a) == code(b) iff the
    K-unit zero-padded prefixes agree (the exact collision law)."""
    strings = sorted(_all_strings(alphabet, maxlen))
    codes, _ = _codes(oracle_mod, [list(s) for s in strings], coder)
    assert all(a <= b for a, b in zip(codes, codes[1:]))
    pad = [tuple(s[:K]) + (0,) * (K - min(len(s), K)) for s in strings]
    by_code, by_pad = {}, {}
    for c, p in zip(codes, pad):
        by_code.setdefault(c, set()).add(p)
        by_pad.setdefault(p, set()).add(c)
    assert all(len(v) == 1 for v in by_code.values())
    assert all(len(v) == 1 for v in by_pad.values())


@pytest.mark.parametrize("alphabet", [b"ab", b"AB", b"az"])
def test_english5_single_case_domain(oracle_mod, alphabet):
    _sorted_scan_and_collisions(oracle_mod, E5, tuple(alphabet), 13, 12)


def test_english6_letter_domain(oracle_mod):
    _sorted_scan_and_collisions(oracle_mod, E6, tuple(b"AZaz"), 8, 10)
    _sorted_scan_and_collisions(oracle_mod, E6, tuple(b"Za"), 11, 10)


def test_english5_mixed_case_is_not_monotone(oracle_mod):
    """Why husky_sort requires a single case (reading R15): 'B' < 'a' as code
    units, but the 5-bit mask folds case, so code('B') = 2 > code('a') = 1."""
    c, _ = _codes(oracle_mod, [b"B", b"a"], E5)
    assert b"B" < b"a" and c[0] > c[1]
    c6, _ = _codes(oracle_mod, [b"B", b"a", b"0"], E6)
    assert c6[0] < c6[1]        # letters stay monotone under the 6-bit mask
    assert b"0" < b"B" and c6[2] > c6[0]  # a digit does not (0x30 & 0x3F = 48 > 'B' = 2)


@pytest.mark.parametrize("coder,K", [(E5, 12), (E6, 10)])
def test_perfect_boundaries(oracle_mod, coder, K):
    """12 (5-bit) and 10 (6-bit) characters code uniquely."""
    for L, want in [(0, True), (K - 1, True), (K, True), (K + 1, False)]:
        _, perfect = _codes(oracle_mod, [b"a" * L, b"b"], coder)
        assert perfect is want, (coder, L)
    _, perfect = _codes(oracle_mod, [], coder)
    assert perfect is True


@pytest.mark.parametrize("coder", [E5, E6])
def test_sort_byte_coders_vs_library(oracle_mod, coder):
    rng = random.Random(5 + coder)
    strings = [bytes(rng.choice(b"abcAZ") for _ in range(rng.randint(0, 14))) for _ in range(4000)]
    w = W.from_strings([list(s) for s in strings], coder)
    perm = oracle_mod.sort(coder, w.units, w.offsets)
    assert perm.tolist() == sorted(range(len(strings)), key=lambda i: (strings[i], i))


# ------------------------------------------------------------ numeric keys
@pytest.mark.parametrize("key_type,dtype", [(0, np.uint64), (1, np.int64)])
def test_sort_keys_integers_vs_numpy(oracle_mod, key_type, dtype):
    rng = np.random.default_rng(3 + key_type)
    info = np.iinfo(dtype)
    k = rng.integers(info.min, info.max, size=20000, dtype=dtype, endpoint=True)
    k[::7] = k[3]  # duplicates
    k[:6] = [info.min, info.max, 0, 1, info.max - 1, info.min + 1] if key_type else [0, info.max, 0, 1, 2, 2**63]
    perm = oracle_mod.sort_keys(key_type, k)
    assert np.array_equal(perm, np.argsort(k, kind="stable").astype(np.uint32))


def _java_double_key(x, i):
    """Double.compare order, stated independently: NaNs last and equal; -0.0
    before +0.0; otherwise numeric; ties by index."""
    if math.isnan(x):
        return (1, 0.0, 0, i)
    return (0, x, 1 if (x == 0 and math.copysign(1.0, x) > 0) else 0, i)


def test_sort_keys_doubles_java_order(oracle_mod):
    rng = random.Random(17)
    nans = [struct.unpack("<d", struct.pack("<Q", b))[0]
            for b in (0x7FF8000000000000, 0xFFF8000000000000, 0x7FF0000000000001, 0xFFFFFFFFFFFFFFFF)]
    special = [0.0, -0.0, math.inf, -math.inf, 5e-324, -5e-324, 1.0, -1.0, 2.2250738585072014e-308] + nans
    xs = special * 3 + [rng.uniform(-1e6, 1e6) for _ in range(3000)] + [float(rng.randint(-5, 5)) for _ in range(500)]
    rng.shuffle(xs)
    arr = np.array(xs, dtype=np.float64)
    perm = oracle_mod.sort_keys(2, arr)
    assert perm.tolist() == sorted(range(len(xs)), key=lambda i: _java_double_key(xs[i], i))


# ---------------------------------------------- T-thread oracle (CPU baseline)
@pytest.mark.parametrize("threads", [1, 2, 3, 5, 8, 13])
def test_sort_mt_matches_library_sort(oracle_mod, threads):
    """oracle_sort_mt (chunk merge sorts + pairwise merge rounds) reaches the
    plain definition: pinned against Python's library sort (duplicates across
    chunk boundaries, empty strings, prefixes), not only against oracle_sort."""
    rng = random.Random(100 + threads)
    pool = [bytes(rng.choice(b"ab\x00z") for _ in range(rng.randint(0, 5))) for _ in range(300)]
    strings = [rng.choice(pool) for _ in range(5000)]
    w = W.from_strings([list(s) for s in strings], 0)
    perm = oracle_mod.sort_mt(0, w.units, w.offsets, threads)
    assert perm.tolist() == sorted(range(len(strings)), key=lambda i: (strings[i], i))


@pytest.mark.parametrize("n", [0, 1, 2, 7, 16, 17])
def test_sort_mt_tiny(oracle_mod, n):
    rng = random.Random(n)
    strings = [[rng.randint(0, 0xFFFF) for _ in range(rng.randint(0, 3))] for _ in range(n)]
    w = W.from_strings(strings, 1)
    for t in (1, 4, 8):
        assert np.array_equal(oracle_mod.sort_mt(1, w.units, w.offsets, t), oracle_mod.sort(1, w.units, w.offsets))
