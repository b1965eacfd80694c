"""GPU linear verifier of sort results -- TEST / BENCH INFRASTRUCTURE ONLY.

``verify.cu`` checks a claimed result against the definition of the order
(bijection, strictly increasing adjacent pairs, output string i == input string
perm[i]); it shares no code with the product (``paper_2012_00866_b200``) or the
oracle.  ``bench.py`` runs it on every timed output; tests pin it against
``oracle.verify`` (including mutated results it must reject).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "verify.cu")
_LIB = os.path.join(_HERE, "libhuskycheck.so")
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
        P, U, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        lib.check_pairs.argtypes = [P, I, P, P, U, P, P]
        lib.check_content.argtypes = [P, P, U, P, P, P, U, I, P, P, P]
        lib.check_hash.argtypes = [P, P, P, U, U, I, P, P]
        for f in (lib.check_pairs, lib.check_content, lib.check_hash):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _s(torch, stream):
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def verify(units, offsets, perm, sorted_units, sorted_offsets, stream=None) -> dict:
    """Single-GPU result check (CUDA tensors; units uint8 or int16 for UTF-16).
    -> {"pairs": bad adjacent pairs, "perm": non-bijective entries,
        "content": outputs != input[perm], "offsets": bad ends}; all 0 = valid."""
    import torch
    lib = _load()
    n_in = offsets.numel() - 1
    n = perm.numel()
    w = units.element_size()
    dev = offsets.device
    bad = torch.zeros(4, dtype=torch.int64, device=dev)
    bitmap = torch.zeros(n_in // 32 + 1, dtype=torch.int32, device=dev)
    s = _s(torch, stream)
    rc = lib.check_pairs(sorted_units.data_ptr(), w, sorted_offsets.data_ptr(), perm.data_ptr(), n, bad.data_ptr(), s)
    rc = rc or lib.check_content(units.data_ptr(), offsets.data_ptr(), n_in, sorted_units.data_ptr(),
                                 sorted_offsets.data_ptr(), perm.data_ptr(), n, w, bitmap.data_ptr(),
                                 bad.data_ptr(), s)
    if rc:
        raise RuntimeError(f"checker: cuda error {rc}")
    b = bad.cpu().tolist()
    if n != n_in:
        b[1] += abs(n - n_in)
    if n and int(sorted_offsets[n].item()) != int(offsets[n_in].item() - offsets[0].item()):
        b[3] += 1
    return {"pairs": b[0], "perm": b[1], "content": b[2], "offsets": b[3]}


def shard_pairs(perm, sorted_units, sorted_offsets, stream=None) -> int:
    """Bad adjacent pairs inside one shard of a sharded result."""
    import torch
    lib = _load()
    bad = torch.zeros(4, dtype=torch.int64, device=perm.device)
    rc = lib.check_pairs(sorted_units.data_ptr(), sorted_units.element_size(), sorted_offsets.data_ptr(),
                         perm.data_ptr(), perm.numel(), bad.data_ptr(), _s(torch, stream))
    if rc:
        raise RuntimeError(f"checker: cuda error {rc}")
    return int(bad[0].item())


def hash_sum(units, offsets, perm=None, gbase=0, stream=None):
    """Order-independent sum of H(gidx, string) over a block (perm None: gidx =
    gbase + i) or over an output shard (gidx = perm[i]).  -> int64 CUDA tensor [1]."""
    import torch
    lib = _load()
    n = offsets.numel() - 1
    out = torch.zeros(1, dtype=torch.int64, device=offsets.device)
    rc = lib.check_hash(units.data_ptr(), offsets.data_ptr(), None if perm is None else perm.data_ptr(), gbase, n,
                        units.element_size(), out.data_ptr(), _s(torch, stream))
    if rc:
        raise RuntimeError(f"checker: cuda error {rc}")
    return out
