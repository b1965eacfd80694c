"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck), each
checked against the CPU oracle: the smoke sizes, a 70K ragged case, the slab
gather, a giant dirty run (refinement), off-domain input (general cleanup),
the English coder, numeric keys and the sample-sort loopback driver.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_00866_b200 as h  # noqa: E402
import workloads as W  # noqa: E402


def dev(w):
    u = w.units.view(np.int16) if w.units.dtype == np.uint16 else w.units
    if u.size == 0:
        u = np.zeros(1, dtype=u.dtype)
    return torch.from_numpy(np.ascontiguousarray(u)).cuda(), torch.from_numpy(w.offsets).cuda()


def check(w, tag):
    u, o = dev(w)
    perm, su, so, _ = h.sort(w.coder, u, o)
    torch.cuda.synchronize()
    ref = oracle.sort(w.coder, w.units, w.offsets)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), ref), tag
    rsu, rso = oracle.gather(w.coder, w.units, w.offsets, ref)
    g = su.cpu().numpy()
    if w.coder == 1:
        g = g.view(np.uint16)
    assert np.array_equal(g, rsu) and np.array_equal(so.cpu().numpy(), rso), tag
    print("ok", tag, flush=True)


def main():
    oracle.build()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(5)
    check(W.c1(20_000), "C1 20K")
    check(W.c3(20_000), "C3 20K")
    check(W.c4(20_000), "C4 20K (giant run: refinement)")
    check(W.c2(70_001, vocab_size=3000), "C2-like 70K ragged")
    check(W.c5(70_001), "C5 70K")
    os.environ["HUSKY_SLAB"] = "1"
    check(W.c5(30_000), "C5 30K slab records")
    check(W.c3(30_000), "C3 30K slab records")
    os.environ.pop("HUSKY_SLAB")
    strings = [rng.integers(0, 256, size=int(rng.integers(0, 12))).tolist() for _ in range(20_000)]
    check(W.from_strings(strings, 0), "off-domain bytes (general cleanup)")
    words = [bytes(rng.choice(list(b"abcdefghij"), size=int(rng.integers(0, 15)))) for _ in range(20_000)]
    check(W.from_strings([list(x) for x in words], 2), "ENGLISH5")
    # numeric keys
    k = rng.integers(-2**62, 2**62, size=50_000, dtype=np.int64)
    kt = torch.from_numpy(k).cuda()
    perm = torch.empty(k.size, dtype=torch.int32, device="cuda")
    h.husky_sort_keys(1, kt, perm)
    torch.cuda.synchronize()
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.sort_keys(1, k)), "keys"
    print("ok keys i64", flush=True)
    # sample-sort loopback (3 virtual ranks)
    w = W.c1(30_000)
    u, o = dev(w)
    total = int(w.offsets[-1])
    ws = torch.empty(h.husky_sort_multi_loopback_workspace(0, 3, w.n, total), dtype=torch.uint8, device="cuda")
    perm = torch.empty(w.n, dtype=torch.int32, device="cuda")
    su = torch.empty(total + 8, dtype=torch.uint8, device="cuda")
    so = torch.empty(w.n + 1, dtype=torch.int64, device="cuda")
    h.husky_sort_multi_loopback(0, 3, u, o, perm, su, so, ws)
    torch.cuda.synchronize()
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.sort(0, w.units, w.offsets)), "loopback"
    print("ok loopback P=3", flush=True)
    print("all cases ok")


if __name__ == "__main__":
    main()
