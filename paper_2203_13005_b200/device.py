"""Python handles over the libgxb200 C ABI: daemon context, device graph store,
algorithm state. Thin by design — every byte of per-iteration work runs in the
sm_100a kernels; Python only sequences calls and reads the vote statistics."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

ALGO_IDS = {"sssp": L.ALGO_SSSP, "pagerank": L.ALGO_PAGERANK, "lp": L.ALGO_LP, "cc": L.ALGO_CC}
DIRECTIONS = {"auto": L.DIR_AUTO, "pull": L.DIR_PULL, "push": L.DIR_PUSH}
U32_MAX = 0xFFFFFFFF


def _vp(x) -> ctypes.c_void_p | None:
    """Raw pointer of a numpy array, a torch tensor or an int."""
    if x is None:
        return None
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if isinstance(x, np.ndarray):
        return x.ctypes.data_as(ctypes.c_void_p)
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    raise TypeError(f"cannot take a device/host pointer of {type(x)!r}")


def _stream_ptr(stream) -> ctypes.c_void_p | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


class DeviceContext:
    """One initialised device daemon (Daemon.initialize runs once, A/daemon.py:148-161)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        L.check(L.lib().gxb_init(device, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        if self._h is None:
            raise L.ProtocolError("daemon terminated")
        return self._h

    @property
    def init_count(self) -> int:
        out = ctypes.c_int()
        L.check(L.lib().gxb_init_count(self.handle, ctypes.byref(out)))
        return out.value

    def reinit(self):
        L.check(L.lib().gxb_reinit(self.handle))

    def shutdown(self):
        if self._h is not None:
            L.check(L.lib().gxb_shutdown(self._h))
            self._h = None

    @property
    def alive(self) -> bool:
        return self._h is not None

    def rmat(self, params, stream=None):
        """Generate an R-MAT stream on the device (include/gxb_rmat.h); torch int32 tensors."""
        import torch

        m = params.num_edges
        dev = torch.device("cuda", self.device)
        src = torch.empty(m, dtype=torch.int32, device=dev)
        dst = torch.empty(m, dtype=torch.int32, device=dev)
        w = torch.empty(m, dtype=torch.int32, device=dev) if params.wmax else None
        args = L.RmatArgs(*params.c_args())
        st = _stream_ptr(stream if stream is not None else torch.cuda.current_stream(dev))
        L.check(L.lib().gxb_rmat_generate(self.handle, ctypes.byref(args), _vp(src), _vp(dst), _vp(w), st))
        return src, dst, w


MAX_WEIGHT_SHIFT = 24


def validate_weights(w, num_vertices: int | None = None) -> tuple[np.ndarray | None, int]:
    """Device weights are u32 integers: returns (u32 weights, shift) with w = u32 / 2^shift.

    Integral weights keep shift 0. Non-integral weights that are dyadic rationals (2.5, 0.25,
    1.125 ...) are scaled by the smallest 2^shift that makes them integral: the reference's
    float64 path sums (A/algorithms.py:102-105) of such weights are exact, and so are the
    scaled u32 sums, so distances are bit-identical after dividing by 2^shift. Anything else
    (1e-3, NaN, negative, too large for exact u32 sums) raises ValueError: no silent
    approximation. Negative weights are already rejected by the loader (A/graph.py:161-162)."""
    if w is None:
        return None, 0
    a = np.asarray(w)
    if a.dtype.kind in "iu":
        if a.size and (a.min() < 0 or a.max() > U32_MAX - 1):
            raise ValueError("edge weights must be in [0, 2^32-2]")
        return a.astype(np.uint32, copy=False), 0
    if a.dtype.kind != "f":
        raise ValueError(f"unsupported weight dtype {a.dtype}")
    a = a.astype(np.float64, copy=False)
    if not np.all(np.isfinite(a)) or np.any(a < 0):
        raise ValueError("device SSSP needs finite, non-negative edge weights")
    for shift in range(MAX_WEIGHT_SHIFT + 1):
        sc = np.ldexp(a, shift)
        if np.all(sc == np.floor(sc)):
            top = float(sc.max(initial=0.0))
            bound = top * (num_vertices if num_vertices else 1)
            if top > U32_MAX - 1 or (num_vertices and bound >= U32_MAX):
                break
            return sc.astype(np.uint32), shift
    raise ValueError("device SSSP needs integral (or dyadic-rational) non-negative weights whose "
                     "scaled sums stay below 2^32-1")


class DeviceGraph:
    """Device-resident CSC (+ push CSR) of one destination partition (A/graph.py:175-212)."""

    def __init__(self, ctx: DeviceContext, src, dst, w=None, part: int = 0, nparts: int = 1,
                 csr: bool = True, stream=None, partitioning: str = "edges", sizes=None,
                 capacity=None):
        """partitioning: "edges" = the degree-sorted order dealt round-robin to the
        partitions (balanced edges, vertices and exchange; default); "ranges" = contiguous
        degree-sorted ranges balanced by in-edge cost; "ids" = the reference's contiguous
        ascending-id ranges (even_sizes, or explicit `sizes`).
        capacity: per-partition capacity factors (balancer.capacity_factors); implies
        "ranges" with partition p taking capacity[p] / sum(capacity) of the cost."""
        self.ctx = ctx
        self.weight_shift = 0     # distances are u32 / 2^weight_shift (validate_weights)
        self.max_weight = None    # largest (scaled) u32 weight, when the weights came from the host
        flags = 0 if csr else L.BUILD_NO_CSR
        if partitioning not in ("edges", "ranges", "ids"):
            raise ValueError(f"unknown partitioning {partitioning!r}")
        if partitioning == "ranges":
            flags |= L.BUILD_RANGES
        if partitioning == "ids" or sizes is not None:
            flags |= L.BUILD_ID_RANGES
        sizes_arr = None if sizes is None else np.ascontiguousarray(sizes, dtype=np.uint64)
        if sizes_arr is not None and sizes_arr.size != nparts:
            raise ValueError("one size per partition required")
        cap_arr = None
        if capacity is not None:
            if sizes is not None or partitioning == "ids":
                raise ValueError("capacity factors apply to degree-sorted ranges, not id ranges")
            cap_arr = np.ascontiguousarray(capacity, dtype=np.float64)
            if cap_arr.size != nparts:
                raise ValueError("one capacity factor per partition required")
        if hasattr(src, "is_cuda") and src.is_cuda:
            n = int(src.numel())
            keep = (src, dst, w)
        else:
            src = np.ascontiguousarray(src, dtype=np.uint32)
            dst = np.ascontiguousarray(dst, dtype=np.uint32)
            if src.shape != dst.shape:
                raise ValueError("src/dst length mismatch")
            nv = int(np.union1d(src, dst).size) if w is not None else None
            w, self.weight_shift = validate_weights(w, nv)
            if w is not None:
                self.max_weight = int(w.max(initial=0))
                w = np.ascontiguousarray(w, dtype=np.uint32)
                if w.shape != src.shape:
                    raise ValueError("weight length mismatch")
            n = int(src.size)
            flags |= L.BUILD_HOST_INPUT
            keep = (src, dst, w)
        self._keep = keep  # inputs must outlive the async copies
        h = ctypes.c_void_p()
        if cap_arr is not None:
            L.check(L.lib().gxb_graph_build_balanced(ctx.handle, _vp(src), _vp(dst), _vp(w), n, part, nparts,
                                                     _vp(cap_arr), flags, _stream_ptr(stream), ctypes.byref(h)))
        else:
            L.check(L.lib().gxb_graph_build_sized(ctx.handle, _vp(src), _vp(dst), _vp(w), n, part, nparts,
                                                  _vp(sizes_arr), flags, _stream_ptr(stream), ctypes.byref(h)))
        self._h = h
        self._keep = None
        info = L.GraphInfo()
        L.check(L.lib().gxb_graph_get_info(self._h, ctypes.byref(info)))
        self.info = info
        self.num_vertices = int(info.num_vertices)
        self.num_slots = int(info.num_slots)
        self.num_edges = int(info.num_edges)
        self.part, self.nparts = part, nparts
        self.weighted = bool(info.weighted)

    @property
    def handle(self):
        return self._h

    @property
    def owned(self) -> tuple[int, int]:
        return int(self.info.owned_lo), int(self.info.owned_hi)

    def ids(self) -> np.ndarray:
        out = np.empty(self.num_vertices, dtype=np.uint32)
        L.check(L.lib().gxb_graph_ids(self._h, _vp(out)))
        return out

    def out_degree(self) -> np.ndarray:
        out = np.empty(self.num_vertices, dtype=np.uint32)
        L.check(L.lib().gxb_graph_out_degree(self._h, _vp(out)))
        return out

    def xchunks(self) -> np.ndarray:
        """Relative slot bounds of the exchange chunks of the owned block (K + 1)."""
        k = ctypes.c_int()
        L.check(L.lib().gxb_graph_xchunks(self._h, ctypes.byref(k), None))
        out = np.empty(k.value + 1, dtype=np.uint64)
        L.check(L.lib().gxb_graph_xchunks(self._h, ctypes.byref(k), _vp(out)))
        return out

    def owned_ids(self) -> np.ndarray:
        """This partition's present ids, ascending (the order of owned-scope staging)."""
        n = ctypes.c_uint64()
        L.check(L.lib().gxb_graph_owned_ids(self._h, None, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.uint32)
        L.check(L.lib().gxb_graph_owned_ids(self._h, _vp(out), ctypes.byref(n)))
        return out

    def bounds(self) -> np.ndarray:
        out = np.empty(self.nparts + 1, dtype=np.uint64)
        L.check(L.lib().gxb_graph_part_bounds(self._h, _vp(out)))
        return out

    def free(self):
        if getattr(self, "_h", None):
            L.lib().gxb_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DeviceState:
    """Algorithm values, frontier and statistics of one run on one partition."""

    def __init__(self, graph: DeviceGraph, algo: str, sources=None, max_weight: int | None = None):
        if algo not in ALGO_IDS:
            raise ValueError(f"unknown algorithm {algo!r}")
        self.graph = graph
        self.algo = algo
        srcs = None
        nsrc = 0
        if algo == "sssp":
            if sources is not None:
                srcs = np.ascontiguousarray(sources, dtype=np.uint32)
                nsrc = int(srcs.size)
                if nsrc == 0:
                    raise ValueError("sssp needs at least one source vertex")
                if nsrc > 4:
                    raise ValueError("a DeviceState carries at most 4 SSSP lanes (make_state groups more)")
            # u32 distances are exact iff no message d + w can reach 2^32-1 (the
            # library re-checks this against the stored weights)
            if graph.max_weight is not None:
                max_weight = graph.max_weight  # the scaled weights the device holds
            if max_weight is not None and max_weight * graph.num_vertices >= U32_MAX:
                raise ValueError("edge weights too large for exact 32-bit distances")
        h = ctypes.c_void_p()
        L.check(L.lib().gxb_state_create(graph.handle, ALGO_IDS[algo], _vp(srcs), nsrc, ctypes.byref(h)))
        self._h = h
        self.local_passes = 0  # split rounds: local-source passes launched (iterate_local)
        ar = ctypes.c_int()
        L.check(L.lib().gxb_state_arity(h, ctypes.byref(ar)))
        self.arity = ar.value

    @property
    def handle(self):
        return self._h

    def iterate(self, direction: str = "auto", stream=None):
        L.check(L.lib().gxb_iterate(self._h, DIRECTIONS[direction], _stream_ptr(stream)))

    def iterate_local(self, stream=None):
        """Launch the next round's local-source pass beside the exchange (split rounds:
        option ``split_overlap``; a no-op unless the last round was a dense SSSP / CC pull
        at N > 1). The next :meth:`iterate` combines it with the remote-source pass."""
        launched = ctypes.c_int(0)
        L.check(L.lib().gxb_iterate_local(self._h, _stream_ptr(stream), ctypes.byref(launched)))
        self.local_passes += launched.value
        return bool(launched.value)

    def iterate_begin(self, stream=None):
        L.check(L.lib().gxb_iterate_begin(self._h, _stream_ptr(stream)))

    def iterate_chunk(self, k: int, stream=None):
        L.check(L.lib().gxb_iterate_chunk(self._h, k, _stream_ptr(stream)))

    def iterate_end(self, stream=None):
        L.check(L.lib().gxb_iterate_end(self._h, _stream_ptr(stream)))

    def request(self, op: int, lo: int, hi: int, stream=None):
        L.check(L.lib().gxb_request(self._h, op, lo, hi, _stream_ptr(stream)))

    def commit(self, stream=None):
        L.check(L.lib().gxb_commit(self._h, _stream_ptr(stream)))

    def stats(self, stream=None) -> dict:
        st = L.IterStats()
        L.check(L.lib().gxb_stats(self._h, _stream_ptr(stream), ctypes.byref(st)))
        return st.as_dict()

    def stats_device(self, out, stream=None):
        """Write the closed round's vote block (changed, next_active, next_units, remote_active,
        max_stat; float64) into a device tensor without a host synchronisation."""
        L.check(L.lib().gxb_stats_device(self._h, _vp(out), _stream_ptr(stream)))

    def stats_async(self, on: bool):
        """PageRank: rounds leave their statistics on the device (read with stats_device)."""
        L.check(L.lib().gxb_stats_async(self._h, int(bool(on))))

    def rollback(self):
        """Undo the last PageRank round (its outputs went to the next buffers only)."""
        L.check(L.lib().gxb_round_rollback(self._h))

    def _shift(self) -> int:
        return self.graph.weight_shift if self.algo == "sssp" else 0

    def read_attrs(self, owned_only: bool = False, stream=None) -> np.ndarray:
        V = self.graph.num_vertices
        out = np.empty((V, self.arity), dtype=np.float64)
        L.check(L.lib().gxb_read_attrs(self._h, _vp(out), int(owned_only), _stream_ptr(stream)))
        if self._shift():
            np.ldexp(out, -self._shift(), out=out)  # exact: distances are u32 / 2^shift (inf stays inf)
        return out

    def read_attrs_into(self, out: np.ndarray, owned_only: bool = False, stream=None) -> np.ndarray:
        """Like read_attrs into a caller-provided (e.g. pinned) host array."""
        L.check(L.lib().gxb_read_attrs(self._h, _vp(out), int(owned_only), _stream_ptr(stream)))
        if self._shift():
            np.ldexp(out, -self._shift(), out=out)
        return out

    def write_attrs(self, values, stream=None):
        """Install attributes (ascending-id order) from the host: the agent's pull_from_upper."""
        if isinstance(values, np.ndarray):
            a = np.ascontiguousarray(values, dtype=np.float64)
            if a.size != self.graph.num_vertices * self.arity:
                raise ValueError("attribute array has the wrong length")
            if self._shift():
                a = np.ldexp(a, self._shift())
            L.check(L.lib().gxb_write_attrs(self._h, _vp(a), _stream_ptr(stream)))
        else:  # pinned torch tensor, in the device encoding
            L.check(L.lib().gxb_write_attrs(self._h, _vp(values), _stream_ptr(stream)))

    def deliver(self, dense, values, stream=None):
        """Install mirror values (sources owned by other partitions, by dense index = rank of
        the id among the present ids) delivered by the sync round (A/agent.py:584-592); on
        SSSP / CC / LP they become active sources of the next round."""
        d = np.ascontiguousarray(dense, dtype=np.uint64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if v.size != d.size * self.arity:
            raise ValueError("deliver: one row of `arity` values per vertex required")
        if self._shift():
            v = np.ldexp(v, self._shift())
        L.check(L.lib().gxb_attrs_deliver(self._h, _vp(d), _vp(v), int(d.size), _stream_ptr(stream)))

    # fused PageRank exchange: Apply stores into the peers' replicas (NVLink / NVSwitch)
    IPC_HANDLE_BYTES = 64

    def ipc_handle(self, which: int) -> bytes:
        buf = (ctypes.c_ubyte * self.IPC_HANDLE_BYTES)()
        L.check(L.lib().gxb_exchange_ipc_handle(self._h, which, buf))
        return bytes(buf)

    def open_peers(self, handles: bytes, npeers: int):
        """handles: npeers x (buffer 0, buffer 1) IPC handles of the other ranks' states."""
        if len(handles) != 2 * npeers * self.IPC_HANDLE_BYTES:
            raise ValueError("open_peers: expected 2 handles per peer")
        buf = (ctypes.c_ubyte * max(1, len(handles))).from_buffer_copy(handles or b"\0")
        L.check(L.lib().gxb_exchange_open_peers(self._h, npeers, buf))

    def set_peer_states(self, peers):
        """Same-process peers (other DeviceStates): Apply writes their replicas directly."""
        ptrs = (ctypes.c_void_p * max(1, 2 * len(peers)))()
        for q, st in enumerate(peers):
            for b in range(2):
                ptrs[2 * q + b] = st._contrib_ptr(b)
        L.check(L.lib().gxb_exchange_set_peer_ptrs(self._h, len(peers), ptrs))

    def close_peers(self):
        L.check(L.lib().gxb_exchange_close_peers(self._h))

    def _contrib_ptr(self, b: int) -> int:
        return self.buffer(L.BUF_CONTRIB1 if b else L.BUF_CONTRIB0)[0]

    # asynchronous staging (pipelined agent loop; pinned host tensors, explicit streams)
    def attrs_scope(self, owned_only: bool):
        """Stage every vertex (False) or only this partition's owned vertices (True, in
        `DeviceGraph.owned_ids()` order)."""
        L.check(L.lib().gxb_attrs_scope(self._h, int(bool(owned_only))))

    def attrs_h2d(self, host_in, buf: int, stream):
        L.check(L.lib().gxb_attrs_h2d(self._h, _vp(host_in), buf, _stream_ptr(stream)))

    def attrs_install(self, buf: int, stream=None):
        L.check(L.lib().gxb_attrs_install(self._h, buf, _stream_ptr(stream)))

    def attrs_extract(self, buf: int, stream=None):
        L.check(L.lib().gxb_attrs_extract(self._h, buf, _stream_ptr(stream)))

    def attrs_d2h(self, host_out, buf: int, stream):
        L.check(L.lib().gxb_attrs_d2h(self._h, _vp(host_out), buf, _stream_ptr(stream)))

    def profile(self, enable: bool | None = None, reset: bool = False) -> dict:
        if enable is not None:
            L.check(L.lib().gxb_profile_enable(self._h, int(enable)))
        p = L.Profile()
        L.check(L.lib().gxb_profile_read(self._h, ctypes.byref(p), int(reset)))
        return p.as_dict()

    def buffer(self, which: int) -> tuple[int, int]:
        p = ctypes.c_void_p()
        b = ctypes.c_uint64()
        L.check(L.lib().gxb_exchange_buffer(self._h, which, ctypes.byref(p), ctypes.byref(b)))
        return int(p.value or 0), int(b.value)

    def pack(self, stream=None) -> int:
        n = ctypes.c_uint64()
        L.check(L.lib().gxb_exchange_pack(self._h, _stream_ptr(stream), ctypes.byref(n)))
        return int(n.value)

    def pack_async(self, stream=None):
        """Pack the closed round's changed owned values; the count rides in the vote block."""
        L.check(L.lib().gxb_exchange_pack_async(self._h, _stream_ptr(stream)))

    def unpack_regions(self, ptr: int, counts, block_records: int, frontier_after=None, units_after=None,
                       stream=None):
        """Install counts[q] records from block q of a padded all-gather (0 for the own block);
        frontier_after / units_after: the next frontier's size and GEN units when known."""
        arr = (ctypes.c_uint64 * max(1, len(counts)))(*[int(c) for c in counts])
        unknown = (1 << 64) - 1
        fa = unknown if frontier_after is None else int(frontier_after)
        ua = unknown if units_after is None else int(units_after)
        L.check(L.lib().gxb_exchange_unpack_regions(self._h, ctypes.c_void_p(ptr), arr, len(counts),
                                                     int(block_records), fa, ua, _stream_ptr(stream)))

    def unpack(self, ptr: int, count: int, stream=None):
        L.check(L.lib().gxb_exchange_unpack(self._h, ctypes.c_void_p(ptr), count, _stream_ptr(stream)))

    def sparse_counts(self):
        """Per-peer element counts of the needed-only PageRank exchange (send, recv), or None."""
        n = self.graph.nparts
        if n < 2 or self.algo != "pagerank":
            return None
        snd = np.zeros(n, dtype=np.uint64)
        rcv = np.zeros(n, dtype=np.uint64)
        L.check(L.lib().gxb_exchange_sparse_counts(self._h, _vp(snd), _vp(rcv)))
        return [int(x) for x in snd], [int(x) for x in rcv]

    def exchange_counts(self):
        """Per-peer (send, recv) counts of distinct slots: my owned slots peer q's CSC reads,
        and peer p's slots my CSC reads (nparts >= 2)."""
        n = self.graph.nparts
        snd = np.zeros(n, dtype=np.uint64)
        rcv = np.zeros(n, dtype=np.uint64)
        L.check(L.lib().gxb_exchange_sparse_counts(self._h, _vp(snd), _vp(rcv)))
        return [int(x) for x in snd], [int(x) for x in rcv]

    # per-peer delta exchange (SSSP / CC / LP): changed values stored into the readers' arenas
    def delta_arena(self, cap_matrix) -> bytes:
        """Allocate the receive arena from the all-gathered send counts (rows = senders);
        returns its CUDA IPC handle."""
        m = np.ascontiguousarray(cap_matrix, dtype=np.uint64)
        buf = (ctypes.c_ubyte * self.IPC_HANDLE_BYTES)()
        L.check(L.lib().gxb_exchange_delta_arena(self._h, _vp(m), buf))
        return bytes(buf)

    def delta_open(self, handles: bytes):
        """nparts IPC handles (this rank's own entry is ignored)."""
        if len(handles) != self.graph.nparts * self.IPC_HANDLE_BYTES:
            raise ValueError("delta_open: one handle per partition required")
        buf = (ctypes.c_ubyte * len(handles)).from_buffer_copy(handles)
        L.check(L.lib().gxb_exchange_delta_open(self._h, buf))

    def delta_buffer(self) -> int:
        p = ctypes.c_void_p()
        L.check(L.lib().gxb_exchange_delta_buffer(self._h, ctypes.byref(p)))
        return int(p.value or 0)

    def delta_set_peers(self, states):
        """Same-process partitions (state of partition q at index q; this one ignored)."""
        ptrs = (ctypes.c_void_p * len(states))(*[st.delta_buffer() for st in states])
        L.check(L.lib().gxb_exchange_delta_set_peers(self._h, ptrs))

    def delta_close(self):
        L.check(L.lib().gxb_exchange_delta_close(self._h))

    def delta_pack(self, vote, stream=None):
        """Store the closed round's changed owned values into the readers' arenas; the
        per-receiver counts go to vote[6:] (float64 device tensor of 6 + nparts)."""
        L.check(L.lib().gxb_exchange_delta_pack(self._h, _vp(vote), _stream_ptr(stream)))

    def delta_unpack(self, counts_from, stream=None):
        arr = np.ascontiguousarray([int(c) for c in counts_from], dtype=np.uint64)
        L.check(L.lib().gxb_exchange_delta_unpack(self._h, _vp(arr), _stream_ptr(stream)))

    def dense_install(self, stream=None):
        """After the in-place all-gather of GXB_BUF_VALUES_NEXT: install the changed mirrors."""
        L.check(L.lib().gxb_exchange_dense_install(self._h, _stream_ptr(stream)))

    def sparse_pack(self, stream=None):
        L.check(L.lib().gxb_exchange_sparse_pack(self._h, _stream_ptr(stream)))

    def sparse_unpack(self, stream=None):
        L.check(L.lib().gxb_exchange_sparse_unpack(self._h, _stream_ptr(stream)))

    def free(self):
        if getattr(self, "_h", None):
            L.lib().gxb_state_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class SsspLanes:
    """SSSP with more than 4 sources (the reference takes any source list,
    A/algorithms.py:81-122): the lanes run in groups of 4, one device state per group over
    the same graph. In the reference a vertex whose distance changed on any lane sends all
    its lanes, but a lane that did not change re-sends a value it already sent, which lowers
    nothing; so every lane evolves exactly as in its own group, the joint run converges when
    every group has, and its iteration count is the largest group's. Distances are
    bit-identical; the per-round counters (changed, next-active, units) are summed over the
    groups (a vertex changed in two groups counts twice)."""

    def __init__(self, graph: "DeviceGraph", sources, max_weight: int | None = None):
        srcs = [int(x) for x in sources]
        if not srcs:
            raise ValueError("sssp needs at least one source vertex")
        self.graph = graph
        self.algo = "sssp"
        self.arity = len(srcs)
        self.states = []
        try:
            for i in range(0, len(srcs), 4):
                self.states.append(DeviceState(graph, "sssp", sources=srcs[i:i + 4], max_weight=max_weight))
        except BaseException:
            self.free()
            raise
        self._widths = [st.arity for st in self.states]

    def _split(self, values: np.ndarray):
        cols, a = [], 0
        for wdt in self._widths:
            cols.append(np.ascontiguousarray(values[:, a:a + wdt]))
            a += wdt
        return cols

    def iterate(self, direction: str = "auto", stream=None):
        for st in self.states:
            st.iterate(direction, stream)

    def iterate_local(self, stream=None):
        return any([st.iterate_local(stream) for st in self.states])

    @property
    def local_passes(self) -> int:
        return sum(st.local_passes for st in self.states)

    def request(self, op: int, lo: int, hi: int, stream=None):
        for st in self.states:
            st.request(op, lo, hi, stream)

    def commit(self, stream=None):
        for st in self.states:
            st.commit(stream)

    def stats(self, stream=None) -> dict:
        sts = [st.stats(stream) for st in self.states]
        out = dict(sts[0])
        for k in ("changed", "next_active", "next_units", "units", "targets", "remote_active"):
            out[k] = sum(int(x[k]) for x in sts)
        out["max_stat"] = max(float(x["max_stat"]) for x in sts)
        out["voted"] = int(all(x["voted"] for x in sts))
        return out

    def read_attrs(self, owned_only: bool = False, stream=None) -> np.ndarray:
        return np.concatenate([st.read_attrs(owned_only, stream) for st in self.states], axis=1)

    def write_attrs(self, values, stream=None):
        a = np.asarray(values, dtype=np.float64).reshape(self.graph.num_vertices, self.arity)
        for st, c in zip(self.states, self._split(a)):
            st.write_attrs(c, stream)

    def deliver(self, dense, values, stream=None):
        v = np.asarray(values, dtype=np.float64).reshape(-1, self.arity)
        for st, c in zip(self.states, self._split(v)):
            st.deliver(dense, c, stream)

    def profile(self, enable: bool | None = None, reset: bool = False) -> dict:
        ps = [st.profile(enable, reset) for st in self.states]
        return {k: sum(p[k] for p in ps) for k in ps[0]}

    def free(self):
        for st in self.states:
            st.free()
        self.states = []


def make_state(graph: "DeviceGraph", algo: str, sources=None, max_weight: int | None = None):
    """A DeviceState, or SsspLanes for SSSP with more than 4 sources."""
    if algo == "sssp" and sources is not None and len(sources) > 4:
        return SsspLanes(graph, sources, max_weight)
    return DeviceState(graph, algo, sources=sources, max_weight=max_weight)


@dataclass
class DeviceRun:
    """Result of a run_reference-equivalent loop on the device."""

    ids: np.ndarray
    attrs: np.ndarray
    iterations: int
    converged: bool
    history: list = field(default_factory=list)


def default_cap(algo: str, num_vertices: int) -> int:
    """default_iteration_cap (A/algorithms.py:117-119, 167-168, 201-202; CC = |V|+1)."""
    return {"sssp": num_vertices + 1, "pagerank": 100, "lp": 15, "cc": num_vertices + 1}[algo]


def run_state(state: DeviceState, max_iterations: int | None = None, direction: str = "auto",
              stream=None, keep_history: bool = False) -> tuple[int, bool, list]:
    """Iterate like run_reference (A/algorithms.py:318-341): stop on the vote or the cap."""
    cap = default_cap(state.algo, state.graph.num_vertices) if max_iterations is None else max_iterations
    it, converged, hist = 0, False, []
    while it < cap:
        state.iterate(direction, stream)
        st = state.stats(stream)
        it += 1
        if keep_history:
            hist.append(st)
        if st["voted"]:
            converged = True
            break
    return it, converged, hist
