"""Python binding of libhusky.so -- B200-native Huskysort hot path.

Argument marshalling only: every step of the path runs in the CUDA kernels of
``libhusky.so`` (``csrc/``) behind the C ABI declared in ``include/husky.h``.
PyTorch supplies device memory and streams.  There is no CPU fallback: if the
library is missing this module raises at import, and calls on a machine without
a GPU fail with HUSKY_ERR_CUDA.

The public functions carry the C names:
  husky_unit_bytes, husky_encode, husky_sort_workspace, husky_sort,
  husky_sort_keys_workspace, husky_sort_keys,
  husky_sort_host_workspace, husky_sort_host, husky_select_splitters,
  husky_comm_unique_id, husky_comm_create, husky_comm_destroy,
  husky_sort_multi_workspace, husky_sort_multi_plan, husky_sort_multi_recv_workspace,
  husky_sort_multi_exec, husky_plan_destroy, husky_last_error
plus ``sort()`` / ``sort_multi()`` conveniences that allocate the outputs.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

ASCII = 0
UNICODE = 1
ENGLISH5 = 2
ENGLISH6 = 3
KEY_U64, KEY_I64, KEY_F64 = 0, 1, 2
HUSKY_OK = 0
STATUS = {0: "HUSKY_OK", 1: "HUSKY_ERR_INVALID_ARG", 2: "HUSKY_ERR_DOMAIN", 3: "HUSKY_ERR_CUDA",
          4: "HUSKY_ERR_NCCL", 5: "HUSKY_ERR_WORKSPACE", 6: "HUSKY_ERR_CAPACITY"}

_HERE = os.path.dirname(os.path.abspath(__file__))
# HUSKY_LIB: load another build of the same sources (lab A/B builds only)
LIB_PATH = os.environ.get("HUSKY_LIB") or os.path.join(_HERE, "libhusky.so")


class HuskyError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class husky_outcome(ctypes.Structure):
    _fields_ = [("perfect", ctypes.c_int32), ("domain_ok", ctypes.c_int32),
                ("n_runs", ctypes.c_uint64), ("n_in_runs", ctypes.c_uint64),
                ("max_run", ctypes.c_uint64), ("runs_by_class", ctypes.c_uint64 * 4),
                ("refine_rounds", ctypes.c_uint32), ("radix_passes", ctypes.c_uint32),
                ("keys_partitioned", ctypes.c_uint64), ("exchange", ctypes.c_uint32),
                ("bytes_to_peers", ctypes.c_uint64), ("bytes_from_peers", ctypes.c_uint64)]

    def as_dict(self):
        return {"perfect": bool(self.perfect), "domain_ok": bool(self.domain_ok),
                "n_runs": self.n_runs, "n_in_runs": self.n_in_runs, "max_run": self.max_run,
                "runs_by_class": list(self.runs_by_class), "refine_rounds": self.refine_rounds,
                "radix_passes": self.radix_passes,
                "keys_partitioned": self.keys_partitioned, "exchange": self.exchange,
                "bytes_to_peers": self.bytes_to_peers, "bytes_from_peers": self.bytes_from_peers}


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                      " (no CPU fallback exists)")
_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_I = ctypes.c_int
_SZ = ctypes.c_size_t
_ST = ctypes.c_int


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("husky_unit_bytes", _SZ, _I)
_sig("husky_encode", _ST, _I, _P, _P, _U64, _P, _P, _P)
_sig("husky_sort_workspace", _ST, _I, _U64, _U64, ctypes.POINTER(_SZ))
_sig("husky_sort", _ST, _I, _P, _P, _U64, _P, _P, _P, _P, _SZ, ctypes.POINTER(husky_outcome), _P)
_sig("husky_sort_host_workspace", _ST, _I, _U64, _U64, ctypes.POINTER(_SZ))
_sig("husky_sort_host", _ST, _I, _P, _P, _U64, _P, _P, _P, _P, _SZ, ctypes.POINTER(husky_outcome), _P)
_sig("husky_last_error", ctypes.c_char_p)
_sig("husky_sort_keys_workspace", _ST, _I, _U64, ctypes.POINTER(_SZ))
_sig("husky_sort_keys", _ST, _I, _P, _U64, _P, _P, _P, _SZ, _P)
_sig("husky_sort_host_many_workspace", _ST, _I, _U64, _U64, _I, ctypes.POINTER(_SZ))
_sig("husky_sort_host_many", _ST, _I, _I, _P, _P, _P, _P, _P, _P, _I, _P, _SZ, ctypes.POINTER(husky_outcome))

EXPORTED = ["husky_unit_bytes", "husky_encode", "husky_sort_workspace", "husky_sort",
            "husky_sort_host_workspace", "husky_sort_host", "husky_comm_unique_id",
            "husky_comm_create", "husky_comm_destroy", "husky_sort_multi_workspace",
            "husky_sort_multi_plan", "husky_sort_multi_recv_workspace", "husky_sort_multi_exec",
            "husky_plan_destroy", "husky_sort_multi", "husky_sort_multi_loopback_workspace",
            "husky_sort_multi_loopback", "husky_select_splitters", "husky_last_error",
            "husky_profile_enable", "husky_profile_reset", "husky_profile_read",
            "husky_profile_stage_name", "husky_launch_count", "husky_sort_keys_workspace",
            "husky_sort_keys", "husky_sort_host_many_workspace", "husky_sort_host_many",
            "husky_profile_launches", "husky_comm_world"]

_sig("husky_profile_enable", None, _I)
_sig("husky_profile_reset", None)
_sig("husky_profile_read", _I, _P, _P, _P, _I)
_sig("husky_profile_stage_name", ctypes.c_char_p, _I)
_sig("husky_launch_count", _U64)
_sig("husky_profile_launches", _I, _P, _P, _P, _I)


def husky_profile_enable(on=True):
    """on: False/0 off; True/1 an event pair per kernel launch; 2 event pairs only
    around launch groups (the radix passes, the encoder) -- cheap enough for a
    timed region."""
    _lib.husky_profile_enable(int(on))


def husky_profile_reset():
    _lib.husky_profile_reset()


def husky_profile_read() -> dict:
    """-> {stage_name: {"ms": total device ms, "launches": n, "elems": n}}"""
    k = 16
    ms = (ctypes.c_double * k)()
    la = (ctypes.c_uint64 * k)()
    el = (ctypes.c_uint64 * k)()
    n = _lib.husky_profile_read(ms, la, el, k)
    return {_lib.husky_profile_stage_name(i).decode(): {"ms": ms[i], "launches": la[i], "elems": el[i]}
            for i in range(min(n, k))}


def husky_profile_launches(max_records=65536) -> list:
    """Mode-1 launch log since the last reset: [(stage_name, elems, ms), ...] in launch order."""
    st = (ctypes.c_int * max_records)()
    el = (ctypes.c_uint64 * max_records)()
    ms = (ctypes.c_double * max_records)()
    k = min(int(_lib.husky_profile_launches(st, el, ms, max_records)), max_records)
    return [(_lib.husky_profile_stage_name(st[i]).decode(), int(el[i]), float(ms[i])) for i in range(k)]


def husky_launch_count() -> int:
    return int(_lib.husky_launch_count())


def lib():
    return _lib


def husky_last_error() -> str:
    return _lib.husky_last_error().decode()


def _check(st: int, where: str):
    if st != HUSKY_OK:
        raise HuskyError(st, where, husky_last_error())


def _ptr(t) -> int:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def husky_unit_bytes(coder: int) -> int:
    return int(_lib.husky_unit_bytes(coder))


def husky_encode(coder, units, offsets, codes=None, want_perfect=True, stream=None):
    """A1 through the C ABI.  units/offsets: CUDA tensors.  -> (codes uint64 as int64 tensor, perfect)."""
    import torch
    n = offsets.numel() - 1
    if codes is None:
        codes = torch.empty(max(n, 1), dtype=torch.int64, device=offsets.device)
    perfect = ctypes.c_int32(-1)
    _check(_lib.husky_encode(coder, _ptr(units), _ptr(offsets), n, _ptr(codes),
                             ctypes.byref(perfect) if want_perfect else None, _stream(stream)),
           "husky_encode")
    return codes[:n], (bool(perfect.value) if want_perfect else None)


def husky_sort_workspace(coder, n, total_units=0) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_workspace(coder, n, total_units, ctypes.byref(b)), "husky_sort_workspace")
    return int(b.value)


def husky_sort(coder, units, offsets, perm, sorted_units, sorted_offsets, ws, stream=None):
    """husky_sort through the C ABI on caller-allocated CUDA tensors.  -> outcome dict."""
    out = husky_outcome()
    n = offsets.numel() - 1
    _check(_lib.husky_sort(coder, _ptr(units), _ptr(offsets), n, _ptr(perm), _ptr(sorted_units),
                           _ptr(sorted_offsets), _ptr(ws), ws.numel() * ws.element_size(),
                           ctypes.byref(out), _stream(stream)), "husky_sort")
    return out.as_dict()


def sort(coder, units, offsets, with_units=True, ws=None, stream=None):
    """Allocating convenience: -> (perm int32 tensor [n], sorted_units, sorted_offsets, outcome)."""
    import torch
    n = offsets.numel() - 1
    dev = offsets.device
    total = int(units.numel())
    if ws is None:
        ws = torch.empty(husky_sort_workspace(coder, n, total), dtype=torch.uint8, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    su = so = None
    if with_units:
        su = torch.empty(max(total, 1) + 8, dtype=units.dtype, device=dev)
        so = torch.empty(n + 1, dtype=torch.int64, device=dev)
    outc = husky_sort(coder, units, offsets, perm, su, so, ws, stream)
    if with_units:
        used = int(so[-1].item()) if n else 0
        su = su[:used]
    return perm[:n], su, so, outc


def husky_sort_host_workspace(coder, n, total_units) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_host_workspace(coder, n, total_units, ctypes.byref(b)), "husky_sort_host_workspace")
    return int(b.value)


def husky_sort_host(coder, h_units, h_offsets, h_perm, h_sorted_units, h_sorted_offsets, ws, stream=None):
    """husky_sort on HOST buffers (numpy arrays or pinned CPU tensors).  -> outcome dict."""
    out = husky_outcome()
    n = (h_offsets.size if isinstance(h_offsets, np.ndarray) else h_offsets.numel()) - 1
    _check(_lib.husky_sort_host(coder, _ptr(h_units), _ptr(h_offsets), n, _ptr(h_perm),
                                _ptr(h_sorted_units), _ptr(h_sorted_offsets), _ptr(ws),
                                ws.numel() * ws.element_size(), ctypes.byref(out), _stream(stream)),
           "husky_sort_host")
    return out.as_dict()


def husky_sort_keys_workspace(key_type, n) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_keys_workspace(key_type, n, ctypes.byref(b)), "husky_sort_keys_workspace")
    return int(b.value)


def husky_sort_keys(key_type, keys, perm, sorted_keys=None, ws=None, stream=None):
    """Numeric keys (perfect coding): keys = CUDA tensor of 8-byte elements
    (uint64 bits / int64 / float64).  perm: int32 CUDA tensor [n].  Returns perm."""
    import torch
    n = keys.numel()
    if ws is None:
        ws = torch.empty(husky_sort_keys_workspace(key_type, n), dtype=torch.uint8, device=keys.device)
    _check(_lib.husky_sort_keys(key_type, _ptr(keys), n, _ptr(perm), _ptr(sorted_keys), _ptr(ws),
                                ws.numel() * ws.element_size(), _stream(stream)), "husky_sort_keys")
    return perm


def husky_sort_host_many_workspace(coder, n_max, units_max, depth=2) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_host_many_workspace(coder, n_max, units_max, depth, ctypes.byref(b)),
           "husky_sort_host_many_workspace")
    return int(b.value)


def husky_sort_host_many(coder, batches, ws, depth=2):
    """Pipelined husky_sort_host over many batches.  batches: list of
    (h_units, h_offsets, h_perm, h_sorted_units | None, h_sorted_offsets | None)
    host arrays (numpy or pinned CPU tensors).  -> list of outcome dicts."""
    k = len(batches)
    arr = lambda vals: (ctypes.c_void_p * max(k, 1))(*vals)
    def n_of(o):
        return (o.size if isinstance(o, np.ndarray) else o.numel()) - 1
    units = arr([_ptr(b[0]) for b in batches])
    offs = arr([_ptr(b[1]) for b in batches])
    ns = (ctypes.c_uint64 * max(k, 1))(*[n_of(b[1]) for b in batches])
    perms = arr([_ptr(b[2]) for b in batches])
    with_units = k > 0 and batches[0][3] is not None
    su = arr([_ptr(b[3]) for b in batches]) if with_units else None
    so = arr([_ptr(b[4]) for b in batches]) if with_units else None
    outs = (husky_outcome * max(k, 1))()
    _check(_lib.husky_sort_host_many(coder, k, units, offs, ns, perms, su, so, depth, _ptr(ws),
                                     ws.numel() * ws.element_size(), outs), "husky_sort_host_many")
    return [outs[i].as_dict() for i in range(k)]


from .multi import (husky_comm_create, husky_comm_destroy, husky_comm_unique_id, husky_comm_world,  # noqa: E402
                    husky_plan_destroy, husky_select_splitters, husky_sort_multi,
                    husky_sort_multi_exec, husky_sort_multi_plan, husky_sort_multi_recv_workspace,
                    husky_sort_multi_loopback, husky_sort_multi_loopback_workspace,
                    husky_sort_multi_workspace, sort_multi)
