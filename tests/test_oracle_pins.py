"""Pins for the CPU oracle (runs without a GPU).

The oracle is pinned to things other than itself (task rule 3):
  * worked values the spec states (tests/golden/encode_worked_values.txt),
  * closed forms of Alg. 4 (a sum, not the fold the oracle uses),
  * brute force over ALL pairs of tiny alphabets (weak monotonicity, equality,
    the exact collision law), and a sorted-scan over 265,720 strings,
  * Python's library sort for the full comparator,
  * the paper-literal Alg. 1 (introsort + insertion cleanup) for the sort,
  * mutation checks for the linear verifier.
"""
import itertools
import os
import random

import numpy as np
import pytest

import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))
ASCII, UNICODE = 0, 1


def _wl(strings, coder):
    return W.from_strings(strings, coder)


def _codes(oracle_mod, strings, coder):
    w = _wl(strings, coder)
    codes, perfect = oracle_mod.encode(coder, w.units, w.offsets)
    return [int(c) for c in codes], perfect


# ------------------------------------------------------------ encode pins
def test_worked_values_golden(oracle_mod):
    """SPEC.md:201, 210, 220, 221, 604 worked values."""
    path = os.path.join(HERE, "golden", "encode_worked_values.txt")
    n = 0
    for line in open(path):
        if not line.strip() or line.startswith("#"):
            continue
        coder_s, units_s, expect_s, cite = [x.strip() for x in line.split("|")]
        coder = {"ascii": ASCII, "unicode": UNICODE, "english5": 2, "english6": 3}[coder_s]
        units = [int(x, 16) for x in units_s.split(",")] if units_s else []
        codes, _ = _codes(oracle_mod, [units], coder)
        assert codes[0] == int(expect_s), cite
        n += 1
    assert n == 8


def closed_form_ascii(s):
    """Alg. 4 with (9, 7, 0x7F) as a sum: sum_{i<m} (u_i & 0x7F) * 2^(7*(8-i))."""
    m = min(len(s), 9)
    return sum((s[i] & 0x7F) << (7 * (8 - i)) for i in range(m))


def closed_form_unicode(s):
    """Alg. 4 with (4, 16, 0xFFFF) then >>> 1: (sum_{i<m} u_i * 2^(16*(3-i))) >> 1."""
    m = min(len(s), 4)
    return sum(s[i] << (16 * (3 - i)) for i in range(m)) >> 1


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_closed_form_random(oracle_mod, coder):
    rng = random.Random(7)
    hi = 255 if coder == ASCII else 0xFFFF
    strings = [[rng.randint(0, hi) for _ in range(rng.randint(0, 14))] for _ in range(5000)]
    strings += [[hi] * k for k in range(12)] + [[0] * k for k in range(12)]
    codes, _ = _codes(oracle_mod, strings, coder)
    cf = closed_form_ascii if coder == ASCII else closed_form_unicode
    for s, c in zip(strings, codes):
        assert c == cf(s), s


def test_max_codes_and_sign_bit(oracle_mod):
    """Reading R1: every code < 2^63, so signed (Java) and unsigned order agree."""
    a, _ = _codes(oracle_mod, [[0x7F] * 9, [0xFF] * 12], ASCII)
    u, _ = _codes(oracle_mod, [[0xFFFF] * 4, [0xFFFF] * 9], UNICODE)
    assert a == [2**63 - 1, 2**63 - 1]
    assert u == [2**63 - 1, 2**63 - 1]


def test_truncation_and_unicode_low_bit_collisions(oracle_mod):
    """SPEC.md:330 truncation law; PAPER.md:256 '3 15/16ths characters'."""
    a, _ = _codes(oracle_mod, [b"abcdefghi", b"abcdefghij", b"abcdefghiz"], ASCII)
    assert a[0] == a[1] == a[2] == closed_form_ascii(list(b"abcdefghi"))
    u, _ = _codes(oracle_mod, [[0x4E00] * 4, [0x4E00] * 3 + [0x4E01], [0x4E00] * 3 + [0x4E02]], UNICODE)
    assert u[0] == u[1] != u[2]
    assert u[0] == 0x2700270027002700


def _all_strings(alphabet, maxlen):
    out = [()]
    for L in range(1, maxlen + 1):
        out += list(itertools.product(alphabet, repeat=L))
    return out


def _rank_by_library_sort(strings):
    order = sorted(range(len(strings)), key=lambda i: strings[i])
    rank = np.empty(len(strings), dtype=np.int64)
    rank[order] = np.arange(len(strings))
    return rank


def _check_all_pairs(strings, codes, pad_key):
    """All pairs: a<b => code(a)<=code(b); a==b => equal (distinct here);
    code(a)==code(b) <=> pad_key(a)==pad_key(b)."""
    codes = np.array(codes, dtype=np.uint64)
    rank = _rank_by_library_sort(strings)
    n = len(strings)
    # weak monotonicity over all ordered pairs, vectorised in row blocks
    for s in range(0, n, 512):
        r = rank[s:s + 512, None] < rank[None, :]
        bad = r & (codes[s:s + 512, None] > codes[None, :])
        assert not bad.any(), "monotonicity violated"
    # collision law
    groups = {}
    for s, c in zip(strings, codes.tolist()):
        groups.setdefault(c, set()).add(pad_key(s))
    assert all(len(g) == 1 for g in groups.values()), "codes collide for different padded prefixes"
    keys = {}
    for s, c in zip(strings, codes.tolist()):
        assert keys.setdefault(pad_key(s), c) == c, "equal padded prefixes, different codes"


def test_bruteforce_ascii_ab_len11(oracle_mod):
    """Set (i): every string over {a,b} of length <= 11 (4,095 strings, 16.8M pairs):
    exercises the truncation at K = 9."""
    strings = _all_strings((0x61, 0x62), 11)
    codes, _ = _codes(oracle_mod, strings, ASCII)
    _check_all_pairs(strings, codes, lambda s: tuple(s[:9]) + (0,) * (9 - min(9, len(s))))


def test_bruteforce_ascii_nul_extremes_len6(oracle_mod):
    """Set (ii): every string over {NUL, a, b, 0x7F} of length <= 6 (5,461 strings)."""
    strings = _all_strings((0x00, 0x61, 0x62, 0x7F), 6)
    codes, _ = _codes(oracle_mod, strings, ASCII)
    _check_all_pairs(strings, codes, lambda s: tuple(s[:9]) + (0,) * (9 - min(9, len(s))))


def test_sorted_scan_ascii_abc_len11(oracle_mod):
    """Sorted-scan: all 265,720 strings over {a,b,c}, length <= 11, sorted by the
    library; codes must be non-decreasing along that order (== pairwise weak
    monotonicity)."""
    strings = _all_strings((0x61, 0x62, 0x63), 11)
    strings.sort()
    codes, _ = _codes(oracle_mod, strings, ASCII)
    c = np.array(codes, dtype=np.uint64)
    assert (c[1:] >= c[:-1]).all()
    # strict wherever the 9-prefixes differ
    p9 = [s[:9] for s in strings]
    for i in range(len(strings) - 1):
        if p9[i] != p9[i + 1]:
            assert c[i] < c[i + 1]


def test_bruteforce_unicode(oracle_mod):
    """All strings over {U+0000, U+0001, U+4E00, U+4E01, U+FFFF} of length <= 5
    (3,906 strings).  Collision law: equal codes <=> equal pad4 after clearing the
    low bit of unit 3 (the '>>> 1')."""
    strings = _all_strings((0x0000, 0x0001, 0x4E00, 0x4E01, 0xFFFF), 5)
    codes, _ = _codes(oracle_mod, strings, UNICODE)

    def pad(s):
        p = list(s[:4]) + [0] * (4 - min(4, len(s)))
        p[3] &= 0xFFFE
        return tuple(p)

    _check_all_pairs(strings, codes, pad)


@pytest.mark.parametrize("coder,ok,bad", [(ASCII, 9, 10), (UNICODE, 3, 4)])
def test_perfect_flag_boundaries(oracle_mod, coder, ok, bad):
    """Alg. 3; ASCII 9/10, UNICODE 3/4 (reading R4)."""
    _, p = _codes(oracle_mod, [[0x61] * k for k in range(ok + 1)], coder)
    assert p is True
    _, p = _codes(oracle_mod, [[0x61] * 2, [0x61] * bad, [0x61]], coder)
    assert p is False
    _, p = _codes(oracle_mod, [], coder)
    assert p is True  # empty array: vacuous AND


# -------------------------------------------------------------- sort pins
def _library_perm(strings):
    return sorted(range(len(strings)), key=lambda i: (strings[i], i))


def _random_strings(rng, n, alphabet, maxlen):
    return [tuple(rng.choice(alphabet) for _ in range(rng.randint(0, maxlen))) for _ in range(n)]


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
@pytest.mark.parametrize("case", range(6))
def test_sort_matches_library_sort(oracle_mod, coder, case):
    rng = random.Random(100 + case)
    if coder == ASCII:
        alphabets = [(0x61, 0x62), (0, 0x61, 0x7F), tuple(range(0x61, 0x7B)),
                     (0, 1, 0x80, 0xFF), tuple(range(256)), (0x61,)]
    else:
        alphabets = [(0x4E00, 0x4E01), (0, 1, 0xFFFF), tuple(range(0x4E00, 0x4E20)),
                     (0, 0x8000, 0xFFFF), (0x61, 0x4E00, 0xFFFE, 0xFFFF), (0x4E00,)]
    n = rng.choice([0, 1, 2, 3, 50, 700, 3000])
    strings = _random_strings(rng, n, alphabets[case], rng.choice([3, 12, 25]))
    w = _wl(strings, coder)
    perm = oracle_mod.sort(coder, w.units, w.offsets)
    assert perm.tolist() == _library_perm(strings)


@pytest.mark.parametrize("kind", ["all_equal", "reverse", "sorted", "empties", "nul_ext"])
def test_sort_degenerate(oracle_mod, kind):
    base = [b"", b"a", b"ab", b"abc", b"b", b"ba", b"zzzzzzzzzzzz"]
    strings = {
        "all_equal": [b"same"] * 100,
        "reverse": sorted(base * 5, reverse=True),
        "sorted": sorted(base * 5),
        "empties": [b""] * 20 + [b"x"] + [b""] * 5,
        "nul_ext": [b"a\0\0", b"a", b"a\0", b"a\0\0", b"a", b"a\0"] * 3,
    }[kind]
    strings = [tuple(s) for s in strings]
    w = _wl(strings, ASCII)
    perm = oracle_mod.sort(ASCII, w.units, w.offsets)
    assert perm.tolist() == _library_perm(strings)


def test_sort_c1_sample_matches_library(oracle_mod):
    w = W.c1(20000)
    strings = w.strings()
    perm = oracle_mod.sort(w.coder, w.units, w.offsets)
    assert perm.tolist() == _library_perm(strings)


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_alg1_paper_literal_equals_plain_definition(oracle_mod, coder):
    """Alg. 1 (introsort with co-swap + cleanup) reaches exactly the plain sort."""
    rng = random.Random(5 + coder)
    alph = (0, 0x61, 0x62, 0x7F) if coder == ASCII else (0, 0x4E00, 0x4E01, 0xFFFF)
    for n in (0, 1, 2, 17, 300, 2000):
        strings = _random_strings(rng, n, alph, 12)
        w = _wl(strings, coder)
        perm, _, _ = oracle_mod.huskysort_alg1(coder, w.units, w.offsets)
        assert perm.tolist() == oracle_mod.sort(coder, w.units, w.offsets).tolist()


def test_alg1_key_phase_alone_sorts_distinct_short_strings(oracle_mod):
    """Pins the introsort on its own: distinct NUL-free strings of length <= 9 get
    distinct codes, so the cleanup must find zero inversions."""
    w = W.c1(5000)
    keep = (w.offsets[1:] - w.offsets[:-1]) <= 9
    strings = sorted(set(s for s, k in zip(w.strings(), keep) if k))
    random.Random(3).shuffle(strings)
    ww = _wl(strings, ASCII)
    perm, perfect, resid = oracle_mod.huskysort_alg1(ASCII, ww.units, ww.offsets)
    assert perfect and resid == 0
    assert perm.tolist() == _library_perm(strings)


def test_verify_accepts_and_rejects(oracle_mod):
    strings = [tuple(s) for s in [b"b", b"a", b"a", b"ab", b"", b"ba", b"a"]]
    w = _wl(strings, ASCII)
    perm = oracle_mod.sort(ASCII, w.units, w.offsets)
    assert perm.tolist() == [4, 1, 2, 6, 3, 0, 5]
    assert oracle_mod.verify(ASCII, w.units, w.offsets, perm) == 0
    p = perm.copy(); p[1], p[2] = p[2], p[1]        # equal strings, tie-break violated
    assert oracle_mod.verify(ASCII, w.units, w.offsets, p) == 2 + 1
    p = perm.copy(); p[4], p[5] = p[5], p[4]        # distinct strings swapped
    assert oracle_mod.verify(ASCII, w.units, w.offsets, p) >= 2
    p = perm.copy(); p[0] = p[1]                    # not a bijection
    assert oracle_mod.verify(ASCII, w.units, w.offsets, p) == 1
    assert oracle_mod.verify(ASCII, w.units, w.offsets, perm[:-1]) == 1


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_gather_matches_python_concat(oracle_mod, coder):
    rng = random.Random(11)
    alph = (0, 0x61, 0x62) if coder == ASCII else (0, 0x4E00, 0xFFFF)
    strings = _random_strings(rng, 400, alph, 9)
    w = _wl(strings, coder)
    perm = oracle_mod.sort(coder, w.units, w.offsets)
    su, so = oracle_mod.gather(coder, w.units, w.offsets, perm)
    cat = [u for i in perm for u in strings[i]]
    assert su.tolist() == cat
    assert so.tolist() == [0] + list(np.cumsum([len(strings[i]) for i in perm]))
