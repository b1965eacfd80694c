"""GPU parity of the A2 key sort (LSD onesweep) on key distributions that stress
it: heavy all-equal digit bins, common prefixes that make whole digits
constant (skipped passes), group sizes around tile boundaries (2048 / 2049
keys), and UNICODE codes.  (These cases were first written for the MSD key
sort variant, since removed: measured slower at every size.)
Every case is compared with the CPU oracle bit-exactly (perm, sorted units,
sorted offsets)."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import ASCII, UNICODE, check_against_oracle, h, torch  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture
def keysort():
    return "lsd"


def _wl(strings, coder=ASCII):
    return W.from_strings(strings, coder)


def test_heavy_duplicates(torch, h, oracle_mod, keysort):
    """Buckets that are all-equal and larger than the local-sort threshold."""
    rng = np.random.default_rng(11)
    heavy = [list(b"abcdefghijkl"), list(b"abcdefghijkm"), list(b"zz"), list(b"q" * 20)]
    strings = []
    for i in range(150_000):
        u = rng.random()
        if u < 0.3:
            strings.append(heavy[0])
        elif u < 0.45:
            strings.append(heavy[1])
        elif u < 0.5:
            strings.append(heavy[2])
        elif u < 0.52:
            strings.append(heavy[3])
        else:
            strings.append(list(rng.integers(0x61, 0x7B, size=int(rng.integers(1, 14)))))
    outc = check_against_oracle(torch, h, oracle_mod, _wl(strings))
    assert outc["radix_passes"] >= 1


@pytest.mark.parametrize("coder", [ASCII, UNICODE])
def test_common_prefix_groups(torch, h, oracle_mod, keysort, coder):
    """Groups sharing long prefixes: inside a bucket the next byte is often the
    same for every key, so the MSD level re-queues the segment on a lower byte."""
    rng = np.random.default_rng(12 + coder)
    hi = 0x7F if coder == ASCII else 0xFFFF
    lo = 0x20 if coder == ASCII else 0x4E00
    prefixes = [list(rng.integers(lo, hi, size=int(rng.integers(3, 8)))) for _ in range(40)]
    strings = []
    for i in range(200_000):
        p = prefixes[int(rng.integers(0, len(prefixes)))]
        strings.append(p + list(rng.integers(lo, hi, size=int(rng.integers(0, 6)))))
    check_against_oracle(torch, h, oracle_mod, _wl(strings, coder))


@pytest.mark.parametrize("bucket", [2047, 2048, 2049, 4095, 4097])
def test_bucket_size_at_threshold(torch, h, oracle_mod, keysort, bucket):
    """Buckets of exactly the local-sort threshold (+-1) next to small ones."""
    rng = np.random.default_rng(bucket)
    strings = []
    for c in range(0x61, 0x61 + 6):
        m = bucket if c % 2 else int(rng.integers(1, 300))
        for _ in range(m):
            strings.append([c] + list(rng.integers(0x61, 0x7B, size=int(rng.integers(0, 12)))))
    order = rng.permutation(len(strings))
    check_against_oracle(torch, h, oracle_mod, _wl([strings[i] for i in order]))


@pytest.mark.parametrize("n", [4096, 4097, 6144, 8191, 8193])
def test_local_capacity_edges(torch, h, oracle_mod, keysort, n):
    rng = np.random.default_rng(n)
    strings = [list(rng.integers(0x30, 0x7B, size=int(rng.integers(0, 16)))) for _ in range(n)]
    check_against_oracle(torch, h, oracle_mod, _wl(strings))


@pytest.mark.parametrize("name,n", [("C2", 600_000), ("C3", 600_000), ("C5", 1 << 19)])
def test_configs_both_keysorts(torch, h, oracle_mod, keysort, name, n):
    check_against_oracle(torch, h, oracle_mod, W.make(name, n))


def test_few_distinct_codes_many_levels(torch, h, oracle_mod, keysort):
    """Codes that differ only in their lowest byte (9th char), so partition
    passes descend through every level before the buckets become small."""
    rng = np.random.default_rng(5)
    base = list(b"mmmmmmmm")
    strings = [base + [int(rng.integers(0x61, 0x64))] + list(rng.integers(0x61, 0x7B, size=int(rng.integers(0, 4))))
               for _ in range(120_000)]
    check_against_oracle(torch, h, oracle_mod, _wl(strings))
