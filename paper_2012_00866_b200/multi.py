"""Binding of the multi-GPU (sample sort) entry points of libhusky.so.

One process per GPU: rank 0 creates the 128-byte NCCL id (husky_comm_unique_id),
torch.distributed broadcasts it, every rank calls husky_comm_create on its
device.  husky_sort_multi_plan / _exec then run the sample sort; all kernels
and the NCCL exchange live in csrc/multi.cu.  Argument marshalling only.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _check, _lib, _ptr, _stream, husky_outcome

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_SZ = ctypes.c_size_t
_ST = ctypes.c_int


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("husky_select_splitters", _ST, ctypes.c_int, _P, _P, _U64, ctypes.c_int, _P)
_sig("husky_comm_unique_id", _ST, _P)
_sig("husky_comm_create", _ST, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(_P))
_sig("husky_comm_destroy", _ST, _P)
_sig("husky_comm_world", _ST, _P, ctypes.POINTER(ctypes.c_int))
_sig("husky_sort_multi_workspace", _ST, ctypes.c_int, _U64, _U64, ctypes.c_int, ctypes.POINTER(_SZ))
_sig("husky_sort_multi_plan", _ST, _P, ctypes.c_int, _P, _P, _U64, _U64, _P, _SZ, ctypes.POINTER(_P),
     ctypes.POINTER(_U64), ctypes.POINTER(_U64), _P)
_sig("husky_sort_multi_recv_workspace", _ST, _P, ctypes.POINTER(_SZ))
_sig("husky_sort_multi_exec", _ST, _P, _P, _P, _P, _P, _SZ, ctypes.POINTER(husky_outcome), _P)
_sig("husky_plan_destroy", _ST, _P)
_sig("husky_sort_multi", _ST, _P, ctypes.c_int, _P, _P, _U64, _U64, _P, _P, _P, _U64, _U64,
     ctypes.POINTER(_U64), ctypes.POINTER(_U64), _P, _SZ, ctypes.POINTER(husky_outcome), _P)
_sig("husky_sort_multi_loopback_workspace", _ST, ctypes.c_int, ctypes.c_int, _U64, _U64, ctypes.POINTER(_SZ))
_sig("husky_sort_multi_loopback", _ST, ctypes.c_int, ctypes.c_int, _P, _P, _U64, _P, _P, _P, _P, _SZ, _P,
     ctypes.POINTER(husky_outcome), _P)


def husky_select_splitters(coder: int, units: np.ndarray, offsets: np.ndarray, world: int) -> np.ndarray:
    """Host-only (no GPU): indices of the P-1 splitter samples among the m sample
    strings (units + offsets), by the sample sort's rule."""
    u = np.ascontiguousarray(units)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    m = o.size - 1
    out = np.zeros(max(world - 1, 1), dtype=np.uint64)
    _check(_lib.husky_select_splitters(coder, u.ctypes.data if u.size else None, o.ctypes.data, m, world,
                                       out.ctypes.data), "husky_select_splitters")
    return out[:world - 1]


def husky_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.husky_comm_unique_id(buf), "husky_comm_unique_id")
    return bytes(buf)


def husky_comm_create(rank: int, world: int, uid: bytes):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    comm = _P()
    _check(_lib.husky_comm_create(rank, world, buf, ctypes.byref(comm)), "husky_comm_create")
    return comm


def husky_comm_destroy(comm):
    _check(_lib.husky_comm_destroy(comm), "husky_comm_destroy")


def husky_sort_multi_workspace(coder, n_local, local_units, world) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_multi_workspace(coder, n_local, local_units, world, ctypes.byref(b)),
           "husky_sort_multi_workspace")
    return int(b.value)


def husky_sort_multi_plan(comm, coder, units, offsets, global_base, ws, stream=None):
    """-> (plan, n_out, units_out)."""
    plan = _P()
    n_out, u_out = _U64(0), _U64(0)
    n = offsets.numel() - 1
    _check(_lib.husky_sort_multi_plan(comm, coder, _ptr(units), _ptr(offsets), n, global_base, _ptr(ws),
                                      ws.numel(), ctypes.byref(plan), ctypes.byref(n_out), ctypes.byref(u_out),
                                      _stream(stream)), "husky_sort_multi_plan")
    return plan, int(n_out.value), int(u_out.value)


def husky_sort_multi_recv_workspace(plan) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_multi_recv_workspace(plan, ctypes.byref(b)), "husky_sort_multi_recv_workspace")
    return int(b.value)


def husky_sort_multi_exec(plan, perm_out, sorted_units_out, sorted_offsets_out, recv_ws, stream=None):
    out = husky_outcome()
    _check(_lib.husky_sort_multi_exec(plan, _ptr(perm_out), _ptr(sorted_units_out), _ptr(sorted_offsets_out),
                                      _ptr(recv_ws), recv_ws.numel(), ctypes.byref(out), _stream(stream)),
           "husky_sort_multi_exec")
    return out.as_dict()


def husky_plan_destroy(plan):
    _check(_lib.husky_plan_destroy(plan), "husky_plan_destroy")


def husky_sort_multi(comm, coder, units, offsets, global_base, perm_out, sorted_units_out, sorted_offsets_out,
                     ws, stream=None):
    out = husky_outcome()
    n_out, u_out = _U64(0), _U64(0)
    n = offsets.numel() - 1
    cap_n = perm_out.numel()
    cap_u = sorted_units_out.numel() if sorted_units_out is not None else 0
    _check(_lib.husky_sort_multi(comm, coder, _ptr(units), _ptr(offsets), n, global_base, _ptr(perm_out),
                                 _ptr(sorted_units_out), _ptr(sorted_offsets_out), cap_n, cap_u,
                                 ctypes.byref(n_out), ctypes.byref(u_out), _ptr(ws), ws.numel(),
                                 ctypes.byref(out), _stream(stream)), "husky_sort_multi")
    return int(n_out.value), int(u_out.value), out.as_dict()


def sort_multi(comm, coder, units, offsets, global_base, with_units=True, stream=None):
    """Allocating convenience over plan/exec: -> (perm shard, sorted units, sorted offsets, outcome)."""
    import torch
    dev = offsets.device
    n = offsets.numel() - 1
    total = int(units.numel())
    from . import husky_unit_bytes  # noqa
    ws = torch.empty(husky_sort_multi_workspace(coder, n, total, _world_of(comm)), dtype=torch.uint8, device=dev)
    plan, n_out, u_out = husky_sort_multi_plan(comm, coder, units, offsets, global_base, ws, stream)
    try:
        rws = torch.empty(husky_sort_multi_recv_workspace(plan), dtype=torch.uint8, device=dev)
        perm = torch.empty(max(n_out, 1), dtype=torch.int32, device=dev)
        su = so = None
        if with_units:
            su = torch.empty(max(u_out, 1) + 8, dtype=units.dtype, device=dev)
            so = torch.empty(n_out + 1, dtype=torch.int64, device=dev)
        outc = husky_sort_multi_exec(plan, perm, su, so, rws, stream)
    finally:
        husky_plan_destroy(plan)
    return perm[:n_out], (su[:u_out] if with_units else None), so, outc


def husky_comm_world(comm) -> int:
    w = ctypes.c_int(0)
    _check(_lib.husky_comm_world(comm, ctypes.byref(w)), "husky_comm_world")
    return int(w.value)


def _world_of(comm):
    return husky_comm_world(comm)


def comm_from_process_group(group=None, device=None):
    """Create a husky NCCL communicator spanning torch.distributed's group."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = husky_comm_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8, device=device if device is not None else "cpu")
    dist.broadcast(t, src=0, group=group)
    return husky_comm_create(rank, world, bytes(t.cpu().tolist()))


def husky_sort_multi_loopback_workspace(coder, world, n, total_units) -> int:
    b = _SZ(0)
    _check(_lib.husky_sort_multi_loopback_workspace(coder, world, n, total_units, ctypes.byref(b)),
           "husky_sort_multi_loopback_workspace")
    return int(b.value)


def husky_sort_multi_loopback(coder, world, units, offsets, perm, sorted_units, sorted_offsets, ws, stream=None):
    out = husky_outcome()
    shards = (_U64 * world)()
    n = offsets.numel() - 1
    _check(_lib.husky_sort_multi_loopback(coder, world, _ptr(units), _ptr(offsets), n, _ptr(perm),
                                          _ptr(sorted_units), _ptr(sorted_offsets), _ptr(ws), ws.numel(),
                                          shards, ctypes.byref(out), _stream(stream)),
           "husky_sort_multi_loopback")
    return [int(x) for x in shards], out.as_dict()
