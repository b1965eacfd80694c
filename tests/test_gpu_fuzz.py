"""Randomised GPU parity sweep through the C ABI: many small seeded cases with
different sizes (0 .. ~30k, ragged against every tile width), alphabets (tiny,
binary with NULs, printable, full byte / UTF-16 range), length mixes (empty,
short, straddling the code window, long) and duplicate rates, for every coder,
each compared bit-exactly with the CPU oracle (perm, sorted units, offsets).
Catches what the targeted tests miss: rare tile/run-boundary interactions."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import check_against_oracle, h, torch  # noqa: F401

pytestmark = pytest.mark.gpu

ALPHABETS = {
    0: [b"ab", b"\x00\x01a", b"abcdefghijklmnopqrstuvwxyz", bytes(range(32, 127)), bytes(range(128))],
    1: [[0x4E00, 0x4E01], [0, 1, 0xFFFF], list(range(0x4E00, 0x4E40)), list(range(0, 0x10000, 257))],
    2: [b"ab", b"abcdefghijklmnopqrstuvwxyz", b"ABCXYZ"],
    3: [b"Ab", b"AZaz", b"abcdefgHIJKLMNOPQRSTUVWXYZ"],
}


def _case(seed):
    rng = np.random.default_rng(seed)
    coder = int(rng.integers(0, 4))
    alph = ALPHABETS[coder][int(rng.integers(0, len(ALPHABETS[coder])))]
    alph = np.frombuffer(alph, dtype=np.uint8) if isinstance(alph, bytes) else np.asarray(alph, dtype=np.uint16)
    n = int(rng.choice([0, 1, 2, 31, 33, 1023, 1025, 2049, 4095, 4097, 8193, 12345, 30000, 614401]))
    maxlen = int(rng.choice([0, 3, 9, 10, 13, 24, 40]))
    dup = float(rng.choice([0.0, 0.3, 0.9]))
    strings = []
    for i in range(n):
        if strings and rng.random() < dup:
            strings.append(strings[int(rng.integers(0, len(strings)))])
        else:
            L = int(rng.integers(0, maxlen + 1))
            strings.append(alph[rng.integers(0, alph.size, size=L)].tolist())
    return W.from_strings(strings, coder, name=f"fuzz{seed}")


@pytest.mark.parametrize("seed", range(300))
def test_fuzz_vs_oracle(torch, h, oracle_mod, seed):
    check_against_oracle(torch, h, oracle_mod, _case(1000 + seed))
