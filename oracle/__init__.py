"""CPU oracle for the Huskysort hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2012_00866_b200``) never imports it and shares no code with it.

Thin numpy/ctypes wrapper over ``husky_oracle.c`` (plain C, built with gcc).
See that file's header for the paper passages each function transcribes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ASCII = 0
UNICODE = 1
ENGLISH5 = 2
ENGLISH6 = 3
KEY_U64, KEY_I64, KEY_F64 = 0, 1, 2

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "husky_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile husky_oracle.c -> liboracle.so with gcc (no CUDA involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        U64 = ctypes.c_uint64
        lib.oracle_encode.argtypes = [ctypes.c_int, P, P, U64, P, P]
        lib.oracle_encode.restype = ctypes.c_int
        lib.oracle_sort.argtypes = [ctypes.c_int, P, P, U64, P]
        lib.oracle_sort.restype = ctypes.c_int
        lib.oracle_gather.argtypes = [ctypes.c_int, P, P, U64, P, P, P]
        lib.oracle_gather.restype = ctypes.c_int
        lib.oracle_verify.argtypes = [ctypes.c_int, P, P, U64, P]
        lib.oracle_verify.restype = ctypes.c_int64
        lib.oracle_huskysort_alg1.argtypes = [ctypes.c_int, P, P, U64, P, P, P]
        lib.oracle_huskysort_alg1.restype = ctypes.c_int
        lib.oracle_sort_mt.argtypes = [ctypes.c_int, P, P, U64, P, ctypes.c_int]
        lib.oracle_sort_mt.restype = ctypes.c_int
        lib.oracle_sort_keys.argtypes = [ctypes.c_int, P, U64, P]
        lib.oracle_sort_keys.restype = ctypes.c_int
        _lib = lib
    return _lib


def _prep(coder, units, offsets):
    dt = np.uint16 if coder == UNICODE else np.uint8
    units = np.ascontiguousarray(units, dtype=dt)
    if units.size == 0:
        units = np.zeros(1, dtype=dt)  # valid pointer for empty inputs
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    return units, offsets, offsets.size - 1


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def encode(coder, units, offsets):
    """-> (codes uint64[n], perfect bool).  Alg. 3 + Alg. 4."""
    units, offsets, n = _prep(coder, units, offsets)
    codes = np.zeros(max(n, 1), dtype=np.uint64)
    perfect = ctypes.c_int32(0)
    rc = _load().oracle_encode(coder, _p(units), _p(offsets), n, _p(codes), ctypes.byref(perfect))
    if rc:
        raise ValueError(f"oracle_encode rc={rc}")
    return codes[:n], bool(perfect.value)


def sort(coder, units, offsets):
    """-> perm uint32[n]: stable merge sort under (units, length, index)."""
    units, offsets, n = _prep(coder, units, offsets)
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rc = _load().oracle_sort(coder, _p(units), _p(offsets), n, _p(perm))
    if rc:
        raise ValueError(f"oracle_sort rc={rc}")
    return perm[:n]


def sort_mt(coder, units, offsets, threads):
    """-> perm uint32[n]: the same result as sort(), computed as `threads` chunk
    merge sorts + pairwise merge rounds (CPU baseline at T = nproc)."""
    units, offsets, n = _prep(coder, units, offsets)
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rc = _load().oracle_sort_mt(coder, _p(units), _p(offsets), n, _p(perm), int(threads))
    if rc:
        raise ValueError(f"oracle_sort_mt rc={rc}")
    return perm[:n]


def gather(coder, units, offsets, perm):
    """-> (sorted_units, sorted_offsets) for a given perm."""
    units, offsets, n = _prep(coder, units, offsets)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    lens = offsets[1:] - offsets[:-1]
    total = int(lens.sum()) if n else 0
    su = np.zeros(max(total, 1), dtype=units.dtype)
    so = np.zeros(n + 1, dtype=np.int64)
    _load().oracle_gather(coder, _p(units), _p(offsets), n, _p(perm if n else np.zeros(1, np.uint32)),
                          _p(su), _p(so))
    return su[:total], so


def verify(coder, units, offsets, perm) -> int:
    """0 iff perm is THE sorted order (bijection + strictly increasing pairs)."""
    units, offsets, n = _prep(coder, units, offsets)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    if perm.size != n:
        return 1
    return int(_load().oracle_verify(coder, _p(units), _p(offsets), n,
                                     _p(perm if n else np.zeros(1, np.uint32))))


def huskysort_alg1(coder, units, offsets):
    """Paper-literal Alg. 1 (introsort with co-swap + insertion cleanup), small n.
    -> (perm, perfect, residual_moves)."""
    units, offsets, n = _prep(coder, units, offsets)
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    perfect = ctypes.c_int32(0)
    resid = ctypes.c_uint64(0)
    rc = _load().oracle_huskysort_alg1(coder, _p(units), _p(offsets), n, _p(perm),
                                       ctypes.byref(perfect), ctypes.byref(resid))
    if rc:
        raise ValueError(f"oracle_huskysort_alg1 rc={rc}")
    return perm[:n], bool(perfect.value), int(resid.value)


def sort_keys(key_type, keys):
    """-> perm uint32[n]: stable merge sort of 8-byte keys (u64 / i64 / f64 in
    Java compareTo order), equal keys by index."""
    k = np.ascontiguousarray(keys).view(np.uint64)
    n = k.size
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rc = _load().oracle_sort_keys(key_type, _p(k if n else np.zeros(1, np.uint64)), n, _p(perm))
    if rc:
        raise ValueError(f"oracle_sort_keys rc={rc}")
    return perm[:n]
