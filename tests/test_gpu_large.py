"""Parity above 2^28 strings (slow): where the packed payload (index | length
<< 28) turns off and every string goes through its slab record.  The C5
recipe is generated on the device (workloads/gen.cu, pinned byte-exact to the
numpy twin by test_gpu_infra.py); the result is checked on the device by the
linear verifier and, independently, by the CPU oracle's linear verifier on a
copy (bijection + strictly increasing adjacent pairs == the oracle's sort,
because the order is a strict total order) plus the sorted offsets / units
against a host gather."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c5_above_2p28(oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import checker
    import paper_2012_00866_b200 as h
    import workloads.gpu as G
    n = (1 << 28) + 12_345
    u, o = G.c5_device(n)
    total = int(o[-1].item())
    perm, su, so, outc = h.sort(0, u, o)
    torch.cuda.synchronize()
    # alphabet-compressed 54-bit keys: 7 passes, 5 or 6 with the lowest one or two
    # digits left unsorted (R19)
    assert outc["keys_partitioned"] in (5 * n, 6 * n, 7 * n)
    r = checker.verify(u, o, perm, su, so)
    assert r == {"pairs": 0, "perm": 0, "content": 0, "offsets": 0}
    # independent host check (CPU oracle's verifier on the whole result)
    hu = u[:total].cpu().numpy()
    ho = o.cpu().numpy()
    hp = perm.cpu().numpy().view(np.uint32)
    assert oracle_mod.verify(0, hu, ho, hp) == 0
    lens = (ho[1:] - ho[:-1])[hp]
    ref_so = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=ref_so[1:])
    assert np.array_equal(so.cpu().numpy(), ref_so)
    # sampled strings of the output against the input
    hsu = su.cpu().numpy()
    for k in np.random.default_rng(3).integers(0, n, size=2000):
        i = hp[k]
        assert np.array_equal(hsu[ref_so[k]:ref_so[k + 1]], hu[ho[i]:ho[i + 1]])
    # perm-only mode at the same size (the run scan and the gather-staged
    # fix-up instead of the gather): the unique order, so the same perm
    del su, so
    torch.cuda.empty_cache()
    perm2, _, _, _ = h.sort(0, u, o, with_units=False)
    torch.cuda.synchronize()
    assert torch.equal(perm2[:n], perm[:n])
