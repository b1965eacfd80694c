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

FULL_N = {"C1": 100_000, "C2": 10_000_000, "C3": 10_000_000, "C4": 10_000_000, "C5": 1 << 30}


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
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based generator (splitmix64 finaliser) on uint64 arrays."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _c5_units(ident: np.ndarray, lens: np.ndarray, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """String content is a function of (seed, identity, position): copies share identity."""
    off = _offsets(lens)
    units = np.empty(int(off[-1]), dtype=np.uint8)
    step = 1 << 22
    with np.errstate(over="ignore"):
        s64 = np.uint64(seed) * np.uint64(0x100000001B3)
    for s in range(0, ident.size, step):
        e = min(ident.size, s + step)
        L = lens[s:e]
        base = int(off[s])
        cnt = int(off[e]) - base
        rel = (np.arange(cnt, dtype=np.int64) - np.repeat(off[s:e] - base, L)).astype(np.uint64)
        with np.errstate(over="ignore"):
            ctr = (np.repeat(ident[s:e].astype(np.uint64), L) << np.uint64(5)) + rel + s64
        units[base:base + cnt] = ALNUM[(_splitmix64(ctr) % np.uint64(62)).astype(np.int64)]
    return units, off


def c5(n: int = FULL_N["C5"], seed: int = MASTER_SEED + 5, dup_frac: float = 0.01,
       sorted_frac: float = 0.10) -> Workload:
    """C5: len uniform in [8, 24], chars uniform [0-9A-Za-z]; floor(0.01 n) positions are
    overwritten with copies of uniformly chosen non-target positions; then the first
    floor(0.1 n) strings are put in ascending order (partially ordered input)."""
    g = _rng(seed)
    lens = g.integers(8, 25, size=n, dtype=np.int64)
    ident = np.arange(n, dtype=np.int64)
    n_dup = int(n * dup_frac)
    if n_dup:
        is_t = np.zeros(n, dtype=bool)
        t = np.unique(g.integers(0, n, size=n_dup + n_dup // 4 + 16))
        while t.size < n_dup:
            t = np.unique(np.concatenate([t, g.integers(0, n, size=n_dup)]))
        t = g.permutation(t)[:n_dup]
        is_t[t] = True
        src = g.integers(0, n, size=n_dup + n_dup // 8 + 16)
        src = src[~is_t[src]]
        while src.size < n_dup:
            more = g.integers(0, n, size=n_dup)
            src = np.concatenate([src, more[~is_t[more]]])
        src = src[:n_dup]
        ident[t] = ident[src]
        lens[t] = lens[src]
    units, off = _c5_units(ident, lens, seed)
    n_sorted = int(n * sorted_frac)
    if n_sorted > 1:
        # input preparation: put the first n_sorted strings in ascending order.
        # Strings are alphanumeric (no NUL), so NUL-padded fixed-width byte
        # comparison equals lexicographic order with shorter-prefix-first.
        fixed = np.zeros((n_sorted, 24), dtype=np.uint8)
        L = lens[:n_sorted]
        rel = np.arange(int(off[n_sorted]), dtype=np.int64) - np.repeat(off[:n_sorted], L)
        fixed[np.repeat(np.arange(n_sorted), L), rel] = units[:off[n_sorted]]
        order = np.argsort(fixed.view("S24").reshape(-1), kind="stable")
        ident[:n_sorted] = ident[:n_sorted][order]
        lens[:n_sorted] = lens[:n_sorted][order]
        units, off = _c5_units(ident, lens, seed)
    return Workload("C5", ASCII, units, off, {"seed": seed, "n": n, "dup": n_dup, "sorted": n_sorted})


GENERATORS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def make(name: str, n: int | None = None, seed_offset: int = 0) -> Workload:
    """Workload `name` at size n (default: BASELINE.json full size)."""
    idx = int(name[1])
    return GENERATORS[name](n if n is not None else FULL_N[name], seed=MASTER_SEED + idx + seed_offset)
