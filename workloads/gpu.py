"""Device-side C5 generator (INPUT GENERATION ONLY; twin of workloads.c5).

Builds ``libhuskygen.so`` from ``gen.cu`` (nvcc, sm_100a) and produces block
[base, base + n) of one global N-string C5 dataset directly in HBM, so a 2^30
string input takes about a second instead of the numpy twin's ~15 minutes, and
each rank of a sharded run generates only its own block.  The prefix sort
(positions [0, N // 10) ascending) is input preparation with ``torch.sort``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

from . import MASTER_SEED

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cu")
_LIB = os.path.join(_HERE, "libhuskygen.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                               "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P, U = ctypes.c_void_p, ctypes.c_uint64
        lib.gen_c5_ident.argtypes = [U, U, U, U, P, P]
        lib.gen_c5_len.argtypes = [U, P, U, P, P]
        lib.gen_c5_keys.argtypes = [U, P, U, P, P, P, P]
        lib.gen_c5_fill.argtypes = [U, P, P, U, P, P]
        for f in (lib.gen_c5_ident, lib.gen_c5_len, lib.gen_c5_keys, lib.gen_c5_fill):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: cuda error {rc}")


def c5_device(N: int, base: int = 0, n: int | None = None, device=None, seed: int = MASTER_SEED + 5):
    """-> (units uint8 tensor [total + 16], offsets int64 tensor [n + 1]) of
    positions [base, base + n) of the global N-string C5 (offsets start at 0).
    The units tensor has 16 bytes of zero slack past the last string."""
    import torch
    lib = _load()
    n = N - base if n is None else n
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    s = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    ident = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    _chk(lib.gen_c5_ident(seed, N, base, n, ident.data_ptr(), s), "gen_c5_ident")
    ns = N // 10
    if base < ns and ns > 1:
        pre = torch.empty(ns, dtype=torch.int64, device=dev)
        _chk(lib.gen_c5_ident(seed, N, 0, ns, pre.data_ptr(), s), "gen_c5_ident")
        w = [torch.empty(ns, dtype=torch.int64, device=dev) for _ in range(3)]
        _chk(lib.gen_c5_keys(seed, pre.data_ptr(), ns, w[0].data_ptr(), w[1].data_ptr(), w[2].data_ptr(), s),
             "gen_c5_keys")
        # stable LSD over the three big-endian words = stable lexicographic order
        order = torch.arange(ns, dtype=torch.int64, device=dev)
        for k in (2, 1, 0):
            _, o = torch.sort(w[k][order], stable=True)
            order = order[o]
        del w
        e = min(ns, base + n)
        ident[:e - base] = pre[order[base:e]]
        del pre, order
    lens = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    _chk(lib.gen_c5_len(seed, ident.data_ptr(), n, lens.data_ptr(), s), "gen_c5_len")
    off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lens[:n], 0, out=off[1:])
    del lens
    total = int(off[-1].item())
    units = torch.zeros(total + 16, dtype=torch.uint8, device=dev)
    _chk(lib.gen_c5_fill(seed, ident.data_ptr(), off.data_ptr(), n, units.data_ptr(), s), "gen_c5_fill")
    del ident
    return units, off
