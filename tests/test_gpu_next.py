"""GPU parity of the NEXT-3 additions through the C ABI, bit-exact against the
CPU oracle: the English 5-bit / 6-bit coders (reading R15) --
encode, full sort on their domains (including dirty and giant equal-code runs),
domain errors -- and the numeric-key sort for perfect codings (PAPER.md:213-217,
reading R16)."""
import struct

import numpy as np
import pytest

import workloads as W
from test_gpu_parity import check_against_oracle, h, to_dev, torch  # noqa: F401

pytestmark = pytest.mark.gpu
E5, E6 = 2, 3


def _rand_words(seed, n, alphabet, lo, hi, prefixes=None):
    rng = np.random.default_rng(seed)
    alph = np.frombuffer(alphabet, dtype=np.uint8)
    out = []
    for i in range(n):
        s = alph[rng.integers(0, alph.size, size=int(rng.integers(lo, hi + 1)))].tolist()
        if prefixes is not None:
            s = list(prefixes[int(rng.integers(0, len(prefixes)))]) + s
        out.append(s)
    return out


@pytest.mark.parametrize("coder", [E5, E6])
def test_encode_parity(torch, h, oracle_mod, coder):
    rng = np.random.default_rng(coder)
    strings = [rng.integers(0, 256, size=int(rng.integers(0, 20))).tolist() for _ in range(30_000)]
    strings += [[0x7A] * k for k in range(16)] + [[] for _ in range(5)]
    w = W.from_strings(strings, coder)
    u, o = to_dev(torch, w)
    codes, perfect = h.husky_encode(coder, u, o)
    ref, rperfect = oracle_mod.encode(coder, w.units, w.offsets)
    assert np.array_equal(codes.cpu().numpy().view(np.uint64), ref)
    assert perfect == rperfect


@pytest.mark.parametrize("coder,alphabet", [(E5, b"abcdefghijklmnopqrstuvwxyz"), (E5, b"ABCXYZ"),
                                            (E6, b"AZaz"), (E6, b"abcdefgHIJKLMNOPQRSTUVWXYZ")])
@pytest.mark.parametrize("n", [1, 2, 4097, 100_000])
def test_sort_domain_words(torch, h, oracle_mod, coder, alphabet, n):
    strings = _rand_words(n, n, alphabet, 0, 16)
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, coder))
    assert outc["domain_ok"]


@pytest.mark.parametrize("coder", [E5, E6])
def test_sort_long_shared_prefixes_dirty_and_giant_runs(torch, h, oracle_mod, coder):
    """Strings past the code window sharing it: equal-code runs of every class,
    one giant (> 4096) run refined by A6."""
    al = b"abc" if coder == E5 else b"aBc"
    pre = [b"q" * 14, b"qrstuvwxyzab", b"abcabcabca"]
    strings = _rand_words(7 + coder, 60_000, al, 0, 9, prefixes=pre)
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, coder))
    assert outc["n_runs"] > 0 and outc["max_run"] > 4096


def test_sort_beyond_window_units_are_free(torch, h, oracle_mod):
    """Units after the 12-unit window are compared exactly and need not be
    letters (only code-window units define the domain)."""
    strings = _rand_words(3, 20_000, b"ab", 12, 12)
    rng = np.random.default_rng(4)
    strings = [s + rng.integers(0, 256, size=int(rng.integers(0, 5))).tolist() for s in strings]
    check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, E5))


@pytest.mark.parametrize("coder,strings", [(E5, [b"abc", b"ABC", b"x", b"Ba", b"aB"] * 50), (E5, [b"ab1", b"ab"] * 50),
                                           (E6, [b"abc", b"ab0", b"AB9z"] * 50), (E6, [b"a b"] * 3)])
def test_sort_off_domain_general_cleanup(torch, h, oracle_mod, coder, strings):
    """Outside the coder's domain (mixed case for ENGLISH5, non-letters for
    ENGLISH6) the code is not monotone; the general cleanup (NEXT-4) sorts the
    whole array exactly and the outcome reports domain_ok = False."""
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings([list(s) for s in strings], coder))
    assert not outc["domain_ok"]


def test_sort_mixed_case_english5_large(torch, h, oracle_mod):
    strings = _rand_words(21, 150_000, b"abcdefgABCDEFG", 0, 15)
    outc = check_against_oracle(torch, h, oracle_mod, W.from_strings(strings, E5))
    assert not outc["domain_ok"] and outc["refine_rounds"] >= 1


# ------------------------------------------------------------ numeric keys
def _keys_case(key_type, n, seed):
    rng = np.random.default_rng(seed)
    if key_type == 0:
        k = rng.integers(0, 2**64, size=n, dtype=np.uint64, endpoint=False)
        k[::5] = k[1] if n > 1 else k[::5]
        return k
    if key_type == 1:
        k = rng.integers(-2**63, 2**63 - 1, size=n, dtype=np.int64, endpoint=True)
        k[::3] = rng.integers(-3, 3, size=k[::3].size)
        return k
    x = rng.standard_normal(n) * 1e3
    special = np.array([0.0, -0.0, np.inf, -np.inf, 5e-324, -5e-324, 1.0, -1.0]
                       + [struct.unpack("<d", struct.pack("<Q", b))[0]
                          for b in (0x7FF8000000000000, 0xFFF8000000000000, 0x7FF0000000000001, 0xFFFFFFFFFFFFFFFF)])
    if n >= special.size:
        idx = rng.choice(n, size=min(n, 200), replace=False)
        x[idx] = special[rng.integers(0, special.size, size=idx.size)]
    x[::7] = np.round(x[::7])
    return x


@pytest.mark.parametrize("key_type", [0, 1, 2])
@pytest.mark.parametrize("n", [1, 2, 4095, 4097, 6143, 6145, 12289, 300_001, 614_401, 2_000_000])
def test_sort_keys_vs_oracle(torch, h, oracle_mod, key_type, n):
    k = _keys_case(key_type, n, 100 + n + key_type)
    dk = torch.from_numpy(k.view(np.int64).copy()).cuda()
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    sk = torch.empty(n, dtype=torch.int64, device="cuda")
    h.husky_sort_keys(key_type, dk, perm, sk)
    torch.cuda.synchronize()
    ref = oracle_mod.sort_keys(key_type, k)
    got = perm.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, ref)
    assert np.array_equal(sk.cpu().numpy().view(np.uint64), k.view(np.uint64)[ref])


def test_sort_keys_all_equal_and_presorted(torch, h, oracle_mod):
    for k in (np.full(50_000, 7, dtype=np.int64), np.arange(50_000, dtype=np.int64),
              np.arange(50_000, 0, -1, dtype=np.int64)):
        dk = torch.from_numpy(k).cuda()
        perm = torch.empty(k.size, dtype=torch.int32, device="cuda")
        h.husky_sort_keys(1, dk, perm)
        torch.cuda.synchronize()
        assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle_mod.sort_keys(1, k))
