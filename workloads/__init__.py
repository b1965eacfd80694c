"""Seeded synthetic string workloads C1-C5 (BASELINE.json ``configs``).

This module holds INPUT GENERATORS ONLY -- none of the method's arithmetic (no
coder, no comparison, no sort of the method).  Both the CUDA path (tests,
bench) and the CPU oracle consume the exact bytes produced here.

Every generator returns a ``Workload``: coder id (0 = ASCII / uint8 units,
1 = UNICODE / uint16 UTF-16 code units), ``units`` (numpy 1-D) and ``offsets``
(int64[n+1], offsets[0] == 0), string i = units[offsets[i]:offsets[i+1]].

The paper benchmarks on Leipzig English/Chinese word lists;
those corpora are not available here, so C2 (English-like Zipf words) and C3
(CJK UTF-16) are synthetic stand-ins shaped like them.
"""
from __future__ import annotations

import dataclasses

import numpy as np

MASTER_SEED = 20120866
ASCII = 0
UNICODE = 1
ENGLISH5 = 2
ENGLISH6 = 3

ALNUM = np.frombuffer(b"0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz", dtype=np.uint8)
LOWER = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)

FULL_N = {"C1": 100_000, "C2": 10_000_000, "C3": 10_000_000, "C4": 10_000_000, "C5": 1 << 30, "D1": 10_000_000}


@dataclasses.dataclass
class Workload:
    name: str
    coder: int
    units: np.ndarray
    offsets: np.ndarray
    meta: dict

    @property
    def n(self) -> int:
        return self.offsets.size - 1

    @property
    def unit_bytes(self) -> int:
        return self.units.dtype.itemsize

    def strings(self):
        """Python list of tuples of units (small n only)."""
        u, o = self.units, self.offsets
        return [tuple(int(x) for x in u[o[i]:o[i + 1]]) for i in range(self.n)]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _offsets(lens: np.ndarray) -> np.ndarray:
    off = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return off


def from_strings(strings, coder: int = ASCII, name: str = "custom") -> Workload:
    """Build a workload from a list of bytes / str / sequences of ints."""
    dt = np.uint16 if coder == UNICODE else np.uint8  # byte coders: ASCII, ENGLISH5, ENGLISH6
    parts = []
    for s in strings:
        if isinstance(s, str):
            s = list(s.encode("latin-1")) if coder != UNICODE else list(s.encode("utf-16-le"))
            if coder == UNICODE:
                s = [s[2 * k] | (s[2 * k + 1] << 8) for k in range(len(s) // 2)]
        parts.append(np.asarray(list(s), dtype=dt))
    lens = np.array([p.size for p in parts], dtype=np.int64)
    units = np.concatenate(parts) if parts else np.zeros(0, dtype=dt)
    return Workload(name, coder, units.astype(dt), _offsets(lens), {})


def c1(n: int = FULL_N["C1"], seed: int = MASTER_SEED + 1) -> Workload:
    """C1: lowercase a-z i.i.d. uniform, length uniform in [4, 12]."""
    g = _rng(seed)
    lens = g.integers(4, 13, size=n, dtype=np.int64)
    off = _offsets(lens)
    units = LOWER[g.integers(0, 26, size=int(off[-1]), dtype=np.uint8)]
    return Workload("C1", ASCII, units, off, {"seed": seed, "n": n})


def c2_vocab(seed: int, size: int = 50_000):
    """50,000 distinct lowercase words, len = min(20, Geometric(1/7)), redraw duplicates."""
    g = _rng(seed)
    words, seen = [], set()
    while len(words) < size:
        L = int(min(20, g.geometric(1.0 / 7.0)))
        w = LOWER[g.integers(0, 26, size=L, dtype=np.uint8)].tobytes()
        if w in seen:
            continue
        seen.add(w)
        words.append(w)
    return words


def c2(n: int = FULL_N["C2"], seed: int = MASTER_SEED + 2, vocab_size: int = 50_000) -> Workload:
    """C2: English-like words: Zipf(s=1) draws from a 50,000-word synthetic vocabulary."""
    words = c2_vocab(seed, vocab_size)
    vlen = np.array([len(w) for w in words], dtype=np.int64)
    vstart = _offsets(vlen)
    vflat = np.frombuffer(b"".join(words), dtype=np.uint8)
    g = _rng(seed + 7919)
    w = 1.0 / np.arange(1, vocab_size + 1, dtype=np.float64)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    ranks = np.minimum(np.searchsorted(cdf, g.random(n), side="right"), vocab_size - 1)
    lens = vlen[ranks]
    off = _offsets(lens)
    units = np.empty(int(off[-1]), dtype=np.uint8)
    step = 1 << 20
    for s in range(0, n, step):
        e = min(n, s + step)
        r = ranks[s:e]
        L = lens[s:e]
        base = off[s]
        rel = np.arange(int(off[e] - base), dtype=np.int64) - np.repeat(off[s:e] - base, L)
        units[base:off[e]] = vflat[np.repeat(vstart[r], L) + rel]
    return Workload("C2", ASCII, units, off, {"seed": seed, "n": n, "vocab": vocab_size})


def c3(n: int = FULL_N["C3"], seed: int = MASTER_SEED + 3) -> Workload:
    """C3: UTF-16 CJK strings, length uniform in [2, 4], units uniform in U+4E00..U+9FFF."""
    g = _rng(seed)
    lens = g.integers(2, 5, size=n, dtype=np.int64)
    off = _offsets(lens)
    units = g.integers(0x4E00, 0xA000, size=int(off[-1]), dtype=np.uint16)
    return Workload("C3", UNICODE, units, off, {"seed": seed, "n": n})


def c4(n: int = FULL_N["C4"], seed: int = MASTER_SEED + 4) -> Workload:
    """C4: one fixed 16-char [0-9A-Za-z] prefix + 8 uniform [0-9A-Za-z] chars (len 24)."""
    g = _rng(seed)
    prefix = ALNUM[g.integers(0, 62, size=16)]
    body = ALNUM[g.integers(0, 62, size=(n, 8), dtype=np.uint8)]
    units = np.empty((n, 24), dtype=np.uint8)
    units[:, :16] = prefix
    units[:, 16:] = body
    off = np.arange(n + 1, dtype=np.int64) * 24
    return Workload("C4", ASCII, units.reshape(-1), off,
                    {"seed": seed, "n": n, "prefix": prefix.tobytes().decode()})


# ------------------------------------------------------------------- C5
# Counter-based recipe (reading R14): every quantity of global
# position i is a function of (seed, stream, counter), so any rank can produce
# block [base, base + n) of ONE global dataset without the others (the CUDA
# twin in workloads/gen.cu implements the same arithmetic; tests compare them).
#   len_i      = 8 + hi32(h(0, i)) * 17 >> 32                       (U{8..24})
#   target_i   = hi32(h(1, i)) < 42949673   (= ceil(0.01 * 2^32))  (Bernoulli 1%)
#   source_i   = first j_a = hi32(h(2, 64 i + a)) * N >> 32, a = 0, 1, ..., that
#                is not a target (a < 64)                            (uniform non-target)
#   ident_i    = source_i if target_i else i;  the string of i is the string of ident_i
#   char k of identity x = ALNUM[hi32(h(3, 32 x + k)) * 62 >> 32]
#   positions [0, floor(0.1 N)) then hold their strings in ascending order
#   (stable: equal strings keep position order).
# h(s, x) = splitmix64(x + splitmix64(seed * 0x100000001B3 + s)).
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
C5_DUP_THRESH = 42949673      # ceil(0.01 * 2^32)
C5_SRC_TRIES = 64


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based generator (splitmix64 finaliser) on uint64 arrays."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _c5_stream(seed: int, s: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return _splitmix64(np.array([seed], dtype=np.uint64) * np.uint64(0x100000001B3) + np.uint64(s))[0]


def _h(seed: int, s: int, x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return _splitmix64(np.asarray(x, dtype=np.uint64) + _c5_stream(seed, s))


def _hi_mul(h: np.ndarray, m: int) -> np.ndarray:
    """(hi32(h) * m) >> 32 as int64 (m < 2^32)."""
    return (((h >> np.uint64(32)) * np.uint64(m)) >> np.uint64(32)).astype(np.int64)


def c5_len(seed: int, pos: np.ndarray) -> np.ndarray:
    return 8 + _hi_mul(_h(seed, 0, pos), 17)


def c5_is_target(seed: int, pos: np.ndarray) -> np.ndarray:
    return (_h(seed, 1, pos) >> np.uint64(32)) < np.uint64(C5_DUP_THRESH)


def c5_ident(seed: int, N: int, pos: np.ndarray) -> np.ndarray:
    """Identity (whose string position i carries) before the prefix sort."""
    pos = np.asarray(pos, dtype=np.int64)
    ident = pos.copy()
    t = np.nonzero(c5_is_target(seed, pos))[0]
    pend = t
    for a in range(C5_SRC_TRIES):
        if pend.size == 0:
            break
        with np.errstate(over="ignore"):
            j = _hi_mul(_h(seed, 2, pos[pend].astype(np.uint64) * np.uint64(64) + np.uint64(a)), N)
        ok = ~c5_is_target(seed, j)
        ident[pend[ok]] = j[ok]
        pend = pend[~ok]
    return ident


def c5_chars(seed: int, ident: np.ndarray, lens: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """units + offsets of the strings of the given identities and lengths."""
    off = _offsets(lens)
    units = np.empty(int(off[-1]), dtype=np.uint8)
    step = 1 << 22
    for s in range(0, ident.size, step):
        e = min(ident.size, s + step)
        L = lens[s:e]
        base = int(off[s])
        cnt = int(off[e]) - base
        rel = (np.arange(cnt, dtype=np.int64) - np.repeat(off[s:e] - base, L)).astype(np.uint64)
        with np.errstate(over="ignore"):
            ctr = (np.repeat(ident[s:e].astype(np.uint64), L) << np.uint64(5)) + rel
        units[base:base + cnt] = ALNUM[_hi_mul(_h(seed, 3, ctr), 62)]
    return units, off


def c5_sorted_prefix_ident(seed: int, N: int) -> np.ndarray:
    """Identities of positions [0, floor(0.1 N)) after the prefix sort."""
    ns = N // 10
    ident = c5_ident(seed, N, np.arange(ns, dtype=np.int64))
    lens = c5_len(seed, ident)
    units, off = c5_chars(seed, ident, lens)
    # NUL-padded 24-byte keys: strings are alphanumeric (no NUL), so padded
    # comparison is lexicographic order with a proper prefix first
    fixed = np.zeros((ns, 24), dtype=np.uint8)
    rel = np.arange(int(off[-1]), dtype=np.int64) - np.repeat(off[:-1], lens)
    fixed[np.repeat(np.arange(ns), lens), rel] = units
    order = np.argsort(fixed.view("S24").reshape(-1), kind="stable")
    return ident[order]


def c5_block(N: int, base: int, n: int, seed: int = MASTER_SEED + 5) -> tuple[np.ndarray, np.ndarray]:
    """Identities + lengths of positions [base, base + n) of the global N-string C5."""
    pos = np.arange(base, base + n, dtype=np.int64)
    ident = c5_ident(seed, N, pos)
    ns = N // 10
    if base < ns and ns > 1:
        pre = c5_sorted_prefix_ident(seed, N)
        e = min(ns, base + n)
        ident[:e - base] = pre[base:e]
    return ident, c5_len(seed, ident)


def c5(n: int = FULL_N["C5"], seed: int = MASTER_SEED + 5, base: int = 0, n_total: int | None = None) -> Workload:
    """C5: len uniform in [8, 24], chars uniform [0-9A-Za-z], ~1% of positions
    (Bernoulli) carry a copy of a uniformly chosen non-target position's string,
    and the first floor(0.1 N) positions are in ascending order (partially
    ordered input).  base / n_total: block [base, base + n) of an n_total-string
    dataset (default: the whole dataset of n strings)."""
    N = n if n_total is None else n_total
    ident, lens = c5_block(N, base, n, seed)
    units, off = c5_chars(seed, ident, lens)
    return Workload("C5", ASCII, units, off,
                    {"seed": seed, "n": n, "N": N, "base": base,
                     "dup": int(np.count_nonzero(c5_is_target(seed, np.arange(base, base + n)))),
                     "sorted": N // 10})


def d1(n: int = 10_000_000, seed: int = MASTER_SEED + 6, group_min: int = 100, group_max: int = 4096,
       suffix_max: int = 10, coder: int = ASCII) -> Workload:
    """D1 (fix-up workload, not a BASELINE config): n strings in groups of
    U[group_min, group_max] strings; a group shares a distinct 12-unit prefix
    (so its husky codes are all equal: one equal-code run) followed by a
    random suffix of U[1, suffix_max] units; all strings shuffled, so nearly
    every run is dirty and goes through the segmented fix-up (A5).  Units:
    a-z (ASCII) or U+4E00..U+9FFF (UNICODE)."""
    g = _rng(seed)
    sizes = []
    while sum(sizes) < n:
        sizes.append(int(g.integers(group_min, group_max + 1)))
    sizes[-1] -= sum(sizes) - n
    ng = len(sizes)
    lo, hi = (0x61, 0x7B) if coder != UNICODE else (0x4E00, 0xA000)
    dt = np.uint8 if coder != UNICODE else np.uint16
    prefixes = g.integers(lo, hi, size=(ng, 12)).astype(dt)
    grp = np.repeat(np.arange(ng), sizes)
    g.shuffle(grp)
    slen = g.integers(1, suffix_max + 1, size=n)
    lens = 12 + slen
    off = _offsets(lens)
    units = np.empty(int(off[-1]), dtype=dt)
    starts = off[:-1]
    for k in range(12):
        units[starts + k] = prefixes[grp, k]
    rel = np.arange(int(off[-1]), dtype=np.int64) - np.repeat(starts, lens)
    sfx = rel >= 12
    units[sfx] = g.integers(lo, hi, size=int(sfx.sum())).astype(dt)
    return Workload("D1", coder, units, off, {"seed": seed, "n": n, "groups": ng})


GENERATORS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5, "D1": d1}


def make(name: str, n: int | None = None, seed_offset: int = 0) -> Workload:
    """Workload `name` at size n (default: BASELINE.json full size)."""
    idx = int(name[1])
    return GENERATORS[name](n if n is not None else FULL_N[name], seed=MASTER_SEED + idx + seed_offset)
