"""GPU test infrastructure pinned before it is trusted:
* the device C5 generator (workloads/gen.cu) produces the numpy twin's bytes;
* the GPU linear verifier (checker/) accepts exactly what oracle.verify accepts,
  including mutated results (swapped pair, repeated index, changed unit,
  wrong length) that it must reject.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


@pytest.mark.parametrize("N,base,n", [(1 << 16, 0, 1 << 16), (1 << 16, 3000, 9000), (1 << 16, 60000, 5536),
                                      (100_003, 0, 100_003), (1 << 20, 1 << 19, 4096)])
def test_device_c5_equals_numpy_twin(torch, N, base, n):
    import workloads.gpu as G
    u, o = G.c5_device(N, base, n)
    ref = W.c5(n, base=base, n_total=N)
    assert np.array_equal(o.cpu().numpy(), ref.offsets)
    total = int(ref.offsets[-1])
    assert np.array_equal(u[:total].cpu().numpy(), ref.units)
    assert int(u[total:].sum().item()) == 0  # zero slack


def _upload(torch, w):
    u = w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units
    return torch.from_numpy(np.ascontiguousarray(u)).cuda(), torch.from_numpy(w.offsets).cuda()


def _oracle_result(torch, oracle_mod, w):
    perm = oracle_mod.sort(w.coder, w.units, w.offsets)
    su, so = oracle_mod.gather(w.coder, w.units, w.offsets, perm)
    su_t = torch.from_numpy(np.ascontiguousarray(su.view(np.int16) if su.dtype == np.uint16 else su)).cuda()
    return (torch.from_numpy(perm.view(np.int32).copy()).cuda(), su_t, torch.from_numpy(so).cuda(), perm)


@pytest.mark.parametrize("name,n", [("C1", 20_000), ("C3", 20_000), ("C5", 30_000)])
def test_checker_against_oracle_verify(torch, oracle_mod, name, n):
    import checker
    w = W.make(name, n)
    u, o = _upload(torch, w)
    perm, su, so, perm_np = _oracle_result(torch, oracle_mod, w)
    assert oracle_mod.verify(w.coder, w.units, w.offsets, perm_np) == 0
    assert checker.verify(u, o, perm, su, so) == {"pairs": 0, "perm": 0, "content": 0, "offsets": 0}

    # a swapped adjacent pair (output rebuilt consistently): both verifiers reject
    p2 = perm_np.copy()
    p2[10], p2[11] = p2[11], p2[10]
    su2, so2 = oracle_mod.gather(w.coder, w.units, w.offsets, p2)
    assert oracle_mod.verify(w.coder, w.units, w.offsets, p2) != 0
    su2_t = torch.from_numpy(np.ascontiguousarray(su2.view(np.int16) if su2.dtype == np.uint16 else su2)).cuda()
    r = checker.verify(u, o, torch.from_numpy(p2.view(np.int32).copy()).cuda(), su2_t, torch.from_numpy(so2).cuda())
    assert r["pairs"] >= 1
    # a repeated index
    p3 = perm.clone()
    p3[5] = p3[6]
    assert checker.verify(u, o, p3, su, so)["perm"] >= 1
    # one output unit changed
    su4 = su.clone()
    su4[int(so[n // 2].item())] += 1
    assert checker.verify(u, o, perm, su4, so)["content"] >= 1
    # output offsets claiming a wrong length
    so5 = so.clone()
    so5[n // 3] += 1
    r = checker.verify(u, o, perm, su, so5)
    assert r["content"] >= 1


def test_checker_hash_sums(torch):
    """Sharded check: the (gidx, string) hash sum of an output equals the
    input's iff the multisets agree."""
    import checker
    w = W.make("C5", 10_000)
    u, o = _upload(torch, w)
    perm = torch.randperm(w.n, device="cuda").to(torch.int32)
    p_np = perm.cpu().numpy().view(np.uint32)
    lens = w.offsets[1:] - w.offsets[:-1]
    so = np.zeros(w.n + 1, dtype=np.int64)
    np.cumsum(lens[p_np], out=so[1:])
    su = np.concatenate([w.units[w.offsets[i]:w.offsets[i + 1]] for i in p_np])
    su_t, so_t = torch.from_numpy(su).cuda(), torch.from_numpy(so).cuda()
    a = checker.hash_sum(u, o, gbase=0)
    b = checker.hash_sum(su_t, so_t, perm=perm)
    assert int(a.item()) == int(b.item())
    perm2 = perm.clone()
    perm2[0], perm2[1] = perm[1], perm[0]  # gidx no longer matches its string
    assert int(checker.hash_sum(su_t, so_t, perm=perm2).item()) != int(a.item())
