"""ctypes binding of libgxb200.so (include/gxb.h). No fallback: if the native
library is missing or the device is not an sm_100 part, calls fail loudly."""

from __future__ import annotations

import ctypes
import os
import sys


class ProtocolError(RuntimeError):
    """A lifecycle / protocol violation (the reference's accelgraph.channel.ProtocolError)."""


_joint_protocol_error = None


def _protocol_error_type():
    """When the reference package is loaded (the drop-in, dropin.py), raise a type that is
    both this ProtocolError and accelgraph.channel.ProtocolError, so the reference's own
    handlers and tests catch it (A/channel.py ProtocolError)."""
    global _joint_protocol_error
    ref = sys.modules.get("accelgraph.channel")
    ref_cls = getattr(ref, "ProtocolError", None)
    if ref_cls is None or issubclass(ProtocolError, ref_cls):
        return ProtocolError
    if _joint_protocol_error is None or not issubclass(_joint_protocol_error, ref_cls):
        _joint_protocol_error = type("ProtocolError", (ProtocolError, ref_cls), {})
    return _joint_protocol_error

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libgxb200.so")

GXB_OK = 0
GXB_EINVAL = -22
GXB_EPROTO = -71
GXB_ENOMEM = -12
GXB_ECUDA = -5
GXB_ERANGE = -34
GXB_ENOTOWNED = -66
GXB_ESTATE = -77

ALGO_SSSP, ALGO_PAGERANK, ALGO_LP, ALGO_CC = 0, 1, 2, 3
OP_GEN, OP_MERGE, OP_APPLY = 0, 1, 2
BUILD_HOST_INPUT, BUILD_NO_CSR, BUILD_ID_RANGES, BUILD_RANGES = 0x1, 0x2, 0x4, 0x8
DIR_AUTO, DIR_PULL, DIR_PUSH = 0, 1, 2
BUF_VALUES, BUF_SEND, BUF_RECV, BUF_RECORD_SIZE, BUF_VALUES_NEXT = 0, 1, 2, 3, 4
BUF_SPARSE_SEND, BUF_SPARSE_RECV = 5, 6
BUF_CONTRIB0, BUF_CONTRIB1 = 7, 8


class GraphInfo(ctypes.Structure):
    _fields_ = [
        ("num_vertices", ctypes.c_uint64), ("num_edges", ctypes.c_uint64),
        ("owned_lo", ctypes.c_uint64), ("owned_hi", ctypes.c_uint64),
        ("owned_edges", ctypes.c_uint64), ("owned_out_edges", ctypes.c_uint64),
        ("max_id", ctypes.c_uint32), ("max_in_degree", ctypes.c_uint32),
        ("part", ctypes.c_int32), ("nparts", ctypes.c_int32),
        ("weighted", ctypes.c_int32), ("has_csr", ctypes.c_int32),
        ("num_slots", ctypes.c_uint64),
    ]


class IterStats(ctypes.Structure):
    _fields_ = [
        ("iteration", ctypes.c_uint64), ("changed", ctypes.c_uint64),
        ("next_active", ctypes.c_uint64), ("next_units", ctypes.c_uint64),
        ("units", ctypes.c_uint64), ("targets", ctypes.c_uint64),
        ("remote_active", ctypes.c_uint64), ("max_stat", ctypes.c_double),
        ("voted", ctypes.c_int32), ("direction", ctypes.c_int32),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class Profile(ctypes.Structure):
    _fields_ = [
        ("main_kernel_ms", ctypes.c_double), ("main_kernel_launches", ctypes.c_uint64),
        ("kernels_launched", ctypes.c_uint64), ("iterations", ctypes.c_uint64),
        ("rest_ms", ctypes.c_double),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class RmatArgs(ctypes.Structure):
    _fields_ = [
        ("scale", ctypes.c_uint32), ("edge_factor", ctypes.c_uint32), ("seed", ctypes.c_uint64),
        ("a", ctypes.c_uint32), ("b", ctypes.c_uint32), ("c", ctypes.c_uint32),
        ("wmax", ctypes.c_uint32), ("scramble", ctypes.c_uint32), ("symmetric", ctypes.c_uint32),
    ]


class GxbError(RuntimeError):
    """A CUDA / device failure inside libgxb200."""


def _sig(L):
    P, I, U64, U32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32
    PP = ctypes.POINTER(ctypes.c_void_p)
    table = {
        "gxb_last_error": (ctypes.c_char_p, []),
        "gxb_version": (ctypes.c_char_p, []),
        "gxb_init": (I, [I, PP]),
        "gxb_reinit": (I, [P]),
        "gxb_init_count": (I, [P, ctypes.POINTER(I)]),
        "gxb_shutdown": (I, [P]),
        "gxb_set_option": (I, [ctypes.c_char_p, ctypes.c_int64]),
        "gxb_get_option": (I, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]),
        "gxb_rmat_generate": (I, [P, ctypes.POINTER(RmatArgs), P, P, P, P]),
        "gxb_graph_build": (I, [P, P, P, P, U64, I, I, U32, P, PP]),
        "gxb_graph_build_sized": (I, [P, P, P, P, U64, I, I, P, U32, P, PP]),
        "gxb_graph_build_balanced": (I, [P, P, P, P, U64, I, I, P, U32, P, PP]),
        "gxb_graph_get_info": (I, [P, ctypes.POINTER(GraphInfo)]),
        "gxb_graph_ids": (I, [P, P]),
        "gxb_graph_out_degree": (I, [P, P]),
        "gxb_graph_part_bounds": (I, [P, P]),
        "gxb_graph_owned_ids": (I, [P, P, P]),
        "gxb_graph_free": (I, [P]),
        "gxb_graph_xchunks": (I, [P, ctypes.POINTER(I), P]),
        "gxb_iterate_begin": (I, [P, P]),
        "gxb_iterate_chunk": (I, [P, I, P]),
        "gxb_iterate_end": (I, [P, P]),
        "gxb_state_create": (I, [P, I, P, I, PP]),
        "gxb_state_free": (I, [P]),
        "gxb_state_arity": (I, [P, ctypes.POINTER(I)]),
        "gxb_iterate": (I, [P, I, P]),
        "gxb_iterate_local": (I, [P, P, ctypes.POINTER(ctypes.c_int)]),
        "gxb_request": (I, [P, I, U64, U64, P]),
        "gxb_commit": (I, [P, P]),
        "gxb_stats": (I, [P, P, ctypes.POINTER(IterStats)]),
        "gxb_exchange_buffer": (I, [P, I, PP, ctypes.POINTER(U64)]),
        "gxb_exchange_pack": (I, [P, P, ctypes.POINTER(U64)]),
        "gxb_exchange_unpack": (I, [P, P, U64, P]),
        "gxb_exchange_pack_async": (I, [P, P]),
        "gxb_exchange_unpack_regions": (I, [P, P, P, I, U64, U64, U64, P]),
        "gxb_exchange_finish": (I, [P, P]),
        "gxb_exchange_sparse_counts": (I, [P, P, P]),
        "gxb_exchange_delta_arena": (I, [P, P, P]),
        "gxb_exchange_delta_open": (I, [P, P]),
        "gxb_exchange_delta_set_peers": (I, [P, P]),
        "gxb_exchange_delta_buffer": (I, [P, PP]),
        "gxb_exchange_delta_close": (I, [P]),
        "gxb_exchange_delta_pack": (I, [P, P, P]),
        "gxb_exchange_delta_unpack": (I, [P, P, P]),
        "gxb_exchange_dense_install": (I, [P, P]),
        "gxb_exchange_sparse_pack": (I, [P, P]),
        "gxb_exchange_sparse_unpack": (I, [P, P]),
        "gxb_read_attrs": (I, [P, P, I, P]),
        "gxb_write_attrs": (I, [P, P, P]),
        "gxb_attrs_h2d": (I, [P, P, I, P]),
        "gxb_attrs_deliver": (I, [P, P, P, U64, P]),
        "gxb_attrs_scope": (I, [P, I]),
        "gxb_stats_device": (I, [P, P, P]),
        "gxb_stats_async": (I, [P, I]),
        "gxb_round_rollback": (I, [P]),
        "gxb_exchange_ipc_handle": (I, [P, I, P]),
        "gxb_exchange_open_peers": (I, [P, I, P]),
        "gxb_exchange_set_peer_ptrs": (I, [P, I, P]),
        "gxb_exchange_close_peers": (I, [P]),
        "gxb_attrs_install": (I, [P, I, P]),
        "gxb_attrs_extract": (I, [P, I, P]),
        "gxb_attrs_d2h": (I, [P, P, I, P]),
        "gxb_profile_enable": (I, [P, I]),
        "gxb_profile_read": (I, [P, ctypes.POINTER(Profile), I]),
    }
    for name, (res, args) in table.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


_lib = None


def lib():
    """Load libgxb200.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        from . import build as _build
        if _build.needs_build():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libgxb200.so not found at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        _sig(L)
        _lib = L
    return _lib


def set_option(name: str, value: int) -> None:
    check(lib().gxb_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    check(lib().gxb_get_option(name.encode(), ctypes.byref(v)))
    return v.value


def check(rc: int) -> int:
    """Map a status code to the reference's exception types (A/daemon.py, A/channel.py)."""
    if rc == GXB_OK:
        return rc
    msg = (lib().gxb_last_error() or b"").decode(errors="replace")
    if rc in (GXB_EINVAL, GXB_ERANGE, GXB_ENOTOWNED):
        raise ValueError(msg)
    if rc in (GXB_EPROTO, GXB_ESTATE):
        raise _protocol_error_type()(msg)
    if rc == GXB_ENOMEM:
        raise MemoryError(msg)
    raise GxbError(f"{msg} (status {rc})")
