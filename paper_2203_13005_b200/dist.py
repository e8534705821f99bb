"""Multi-GPU driver: one process per GPU, destination-range partitions, mirror
exchange over torch.distributed (NCCL on NVLink; gloo for the CPU tests).

Mirrors the reference's barrier schedule for one iteration (A/engine.py:226-294,
298-331): compute (Gen/Merge/Apply on the own partition) -> skip decision
(1-bit AND of partition-closedness, A/engine.py:242-246, A/sync.py:201-208) ->
sync round (only the changed values that a peer consumes travel: the lazy upload
of A/sync.py:171-198, realised as a delta all-gather of (slot, value) records, or
a dense all-gather of the contribution slices for PageRank where every vertex
changes) -> verdict (AND of the local votes, A/engine.py:131-136, 267-285).

The collectives are plain NCCL calls issued by torch.distributed on library-owned
device buffers (zero-copy views through __cuda_array_interface__); the per-vertex
work of packing and installing records runs in libgxb200 kernels.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class _CAI:
    """Zero-copy __cuda_array_interface__ wrapper of a library device buffer."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "|u1"):
        itemsize = int(typestr[2:])
        self.__cuda_array_interface__ = {
            "shape": (nbytes // itemsize,), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


def device_view(ptr: int, nbytes: int, dtype: str = "u1"):
    import torch
    typestr = {"u1": "|u1", "f8": "<f8", "f4": "<f4", "u4": "<u4", "i8": "<i8"}[dtype]
    return torch.as_tensor(_CAI(ptr, nbytes, typestr), device="cuda")


@dataclass
class StepRecord:
    """Per-iteration record in the spirit of IterationRecord (A/engine.py:63-85)."""

    iteration: int
    changed: int
    next_active: int
    units: int
    remote_active: int
    max_stat: float
    skipped: bool
    converged: bool
    exchanged_bytes: int = 0
    direction: int = 1

    def to_line(self, model: str = "bsp") -> str:
        return (f"iter={self.iteration} model={model} changed={self.changed} active={self.next_active} "
                f"units={self.units} skipped={str(self.skipped).lower()} "
                f"uploads={self.exchanged_bytes} converged={str(self.converged).lower()}")


class Collective:
    """The few collectives of one iteration, over an optional torch process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def _host_backend(self) -> bool:
        """gloo (the CPU test path): device tensors are gathered through host copies."""
        try:
            return self.dist.get_backend(self.group) == "gloo"
        except Exception:  # noqa: BLE001
            return False

    def all_gather_flat(self, out, mine):
        """out (world * n) <- every rank's mine (n), in rank order."""
        if mine.is_cuda and self._host_backend():
            parts = [mine.new_empty(mine.numel(), device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, mine.cpu(), group=self.group)
            out.copy_(__import__("torch").cat(parts))
            return
        self.dist.all_gather_into_tensor(out, mine, group=self.group)

    def all_min_flag(self, ok: int, device) -> int:
        """MIN over ranks of a 0/1 flag (agreement on an optional path)."""
        import torch
        dev = "cpu" if self._host_backend() else device
        flag = torch.tensor([int(ok)], dtype=torch.int32, device=dev)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(flag.item())

    def vote_start(self, counts: list[int], max_stat: float, device):
        """Launch the vote: one all-gather of every rank's (counters, max statistic)."""
        import torch
        if self.world == 1:
            return (counts, max_stat)
        mine = torch.tensor([float(c) for c in counts] + [max_stat], dtype=torch.float64, device=device)
        out = torch.empty(self.world * mine.numel(), dtype=torch.float64, device=device)
        self.all_gather_flat(out, mine)
        return out

    def vote_start_device(self, mine):
        """The vote from a device-resident block (gxb_stats_device): no host round trip."""
        import torch
        out = torch.empty(self.world * mine.numel(), dtype=torch.float64, device=mine.device)
        self.all_gather_flat(out, mine)
        return out

    def vote_finish(self, handle) -> tuple[list[int], float]:
        """SUM of the counters (exact below 2^53) and MAX of the statistic over ranks."""
        if isinstance(handle, tuple):
            return handle
        rows = handle.view(self.world, -1).cpu().tolist()
        self.last_rows = rows  # per-rank blocks (e.g. the packed record counts, per-peer counts)
        # columns 0-4: counters (SUM), 5: the statistic (MAX), 6+: per-receiver record counts
        counts = [int(sum(r[i] for r in rows)) for i in range(5)]
        return counts, max(r[5] for r in rows)

    def vote(self, counts: list[int], max_stat: float, device) -> tuple[list[int], float]:
        return self.vote_finish(self.vote_start(counts, max_stat, device))

    def allgatherv(self, out_views, my_view):
        """All-gather with uneven sizes into caller-provided views (grouped P2P)."""
        if self.world == 1:
            return
        ops = []
        for peer in range(self.world):
            if peer == self.rank:
                continue
            if my_view.numel():
                ops.append(self.dist.P2POp(self.dist.isend, my_view, peer, self.group))
            if out_views[peer].numel():
                ops.append(self.dist.P2POp(self.dist.irecv, out_views[peer], peer, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def allgather_inplace(self, out, mine):
        """Equal-size all-gather where `mine` is this rank's block of `out` (NCCL in place)."""
        if self.world == 1:
            return
        self.all_gather_flat(out, mine)

    def gather_counts(self, n: int, device) -> list[int]:
        import torch
        if self.world == 1:
            return [n]
        t = torch.tensor([n], dtype=torch.int64, device=device)
        out = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]


@dataclass
class PartitionedRun:
    """One rank's share of a partitioned BSP run."""

    state: object                      # DeviceState (or a test double with the same surface)
    bounds: np.ndarray                 # slot boundaries of the partitions (world + 1)
    comm: Collective
    enable_skip: bool = True
    records: list = field(default_factory=list)
    device: object = None
    phase_times: dict | None = None   # per-phase seconds when profiling (adds a sync per phase)
    needed_only: bool = False         # PR: send each peer only the values its CSC reads (NCCL
                                      # all-to-all; measured slower than the all-gather at N <= 4)
    sparse_ratio: float = 0.8         # ... when that is below this fraction of the dense volume
    peer_writes: bool = True          # PR: Apply stores new contributions into the peers' replicas over
                                      # NVLink (IPC-mapped), fusing the exchange into the kernel
    dense_frac: float = 0.0           # SSSP / CC / LP: a round after one that changed >= this fraction
                                      # of the slots exchanges whole value blocks (all-gather in place +
                                      # install of the changed mirrors) instead of records; 0 = never
                                      # (measured slower than the per-peer records: SSSP S26 at N = 4
                                      # 802 vs 929 GTEPS — records move only changed and needed values)
    peer_delta: bool = True           # SSSP / CC / LP: the pack kernel stores each changed value only
                                      # into the arenas of the peers that read it (IPC, NVLink)
    overlap: bool = False             # pipeline shuffle: chunked PR rounds with the exchange overlapped
                                      # (needs exchange_chunks > 1; measured slower than one all-gather
                                      # at N <= 4, where the tile kernel and NCCL contend for L2)

    def __post_init__(self):
        self.algo = self.state.algo
        self.iteration = 0
        self.skipped_rounds = 0
        self._pr_remote = None
        self._sparse = None
        self._pending = []
        self._peers = None
        self._dpeers = None
        self._prev_changed = 0
        self.xchunks = 1
        if self.overlap and self.algo == "pagerank" and hasattr(self.state, "graph") and \
                hasattr(self.state.graph, "xchunks"):
            self.xchunks = len(self.state.graph.xchunks()) - 1

    # ---- the sync round ---------------------------------------------------
    def _exchange_needed(self) -> int | None:
        """PageRank, needed-only: each peer receives just my values its CSC reads (static,
        slot-sorted lists), packed by a gather kernel and moved with one NCCL all-to-all."""
        if self._sparse is None:
            counts = self.state.sparse_counts() if hasattr(self.state, "sparse_counts") else None
            if counts is None:
                self._sparse = False
            else:
                snd, rcv = counts
                own = int(self.bounds[self.comm.rank + 1] - self.bounds[self.comm.rank])
                dense = int(self.bounds[-1]) - own
                self._sparse = (snd, rcv) if sum(rcv) < self.sparse_ratio * dense else False
        if not self._sparse:
            return None
        snd, rcv = self._sparse
        sptr, sbytes = self.state.buffer(L.BUF_SPARSE_SEND)
        rptr, rbytes = self.state.buffer(L.BUF_SPARSE_RECV)
        width = sbytes // max(1, sum(snd)) if sum(snd) else (rbytes // max(1, sum(rcv)) if sum(rcv) else 8)
        dt = "f8" if width == 8 else "f4"
        self.state.sparse_pack()
        send = self._view(sptr, sbytes, dt)
        recv = self._view(rptr, rbytes, dt)
        self.comm.dist.all_to_all_single(recv, send, output_split_sizes=rcv, input_split_sizes=snd,
                                         group=self.comm.group)
        self.state.sparse_unpack()
        return width * sum(rcv)

    def _exchange_dense(self) -> int:
        """PageRank: every vertex changes, so all-gather each owner's contribution slice.

        The dealt layout pads every partition block to the same size, so this is one
        in-place NCCL all-gather over the replica (ring / NVLS); other layouts fall back
        to a grouped send/recv all-gather-v."""
        moved = self._exchange_needed() if self.needed_only else None
        if moved is not None:
            return moved
        ptr, nbytes = self.state.buffer(L.BUF_VALUES)
        width = nbytes // max(1, int(self.bounds[-1]))   # 8 (f64 messages) or 4 (pr_message_bits = 32)
        values = self._view(ptr, nbytes, "f8" if width == 8 else "f4")
        sizes = np.diff(self.bounds.astype(np.int64))
        r = self.comm.rank
        if (sizes == sizes[0]).all() and hasattr(self.comm, "allgather_inplace"):
            blk = int(sizes[0])
            self.comm.allgather_inplace(values[: blk * self.comm.world], values[r * blk:(r + 1) * blk])
        else:
            views = [values[int(self.bounds[q]):int(self.bounds[q + 1])] for q in range(self.comm.world)]
            self.comm.allgatherv(views, views[r])
        return width * int(self.bounds[-1] - sizes[r])

    def _equal_blocks(self) -> bool:
        sizes = np.diff(self.bounds.astype(np.int64))
        return bool(sizes.size > 1 and (sizes == sizes[0]).all())

    def _exchange_dense_mirror(self) -> int:
        """SSSP / CC / LP rounds where most vertices changed: all-gather every owner's block of
        the next-value replica in place (one NCCL collective, no per-record packing), then
        install the mirrors whose value differs (gxb_exchange_dense_install)."""
        ptr, nbytes = self.state.buffer(L.BUF_VALUES_NEXT)
        S = int(self.bounds[-1])
        width = nbytes // max(1, S)
        blk = (S // self.comm.world) * width
        values = self._view(ptr, nbytes, "u1")
        r = self.comm.rank
        self.comm.allgather_inplace(values[: blk * self.comm.world], values[r * blk:(r + 1) * blk])
        self.state.dense_install(**self._on_stream())
        return blk * (self.comm.world - 1)

    def _exchange_delta(self) -> int:
        """SSSP / CC / LP: only changed owned values travel, as (slot, value) records."""
        rec = self.state.buffer(L.BUF_RECORD_SIZE)[1]
        n = self.state.pack()
        counts = self.comm.gather_counts(n, self.device)
        sptr, sbytes = self.state.buffer(L.BUF_SEND)
        rptr, rbytes = self.state.buffer(L.BUF_RECV)
        send = self._view(sptr, sbytes, "u1")[: n * rec]
        recv = self._view(rptr, rbytes, "u1")
        offs = np.concatenate([[0], np.cumsum(counts)]) * rec
        views = [recv[int(offs[r]):int(offs[r + 1])] for r in range(self.comm.world)]
        views[self.comm.rank].copy_(send)
        self.comm.allgatherv(views, send)
        total = int(sum(counts))
        self.state.unpack(rptr, total)
        return (total - n) * rec

    def _exchange_delta_async(self, packed: list[int]) -> int:
        """SSSP / CC / LP without host round trips: the record counts came with the vote, the
        records move in one padded all-gather, unpack installs each peer's block."""
        rec = self.state.buffer(L.BUF_RECORD_SIZE)[1]
        maxc = max(packed)
        if maxc == 0:
            return 0
        sptr, sbytes = self.state.buffer(L.BUF_SEND)
        rptr, rbytes = self.state.buffer(L.BUF_RECV)
        send = self._view(sptr, sbytes, "u1")[: maxc * rec]
        recv = self._view(rptr, rbytes, "u1")[: self.comm.world * maxc * rec]
        self.comm.all_gather_flat(recv, send)
        counts = list(packed)
        counts[self.comm.rank] = 0
        rows = self.comm.last_rows
        # next frontier = my changed vertices + every received record; its GEN units = every
        # rank's next_units (a record is a changed vertex of its sender)
        frontier = int(rows[self.comm.rank][1]) + sum(counts)
        units = int(sum(r[2] for r in rows))
        self.state.unpack_regions(rptr, counts, maxc, frontier, units)
        return sum(counts) * rec

    def install(self, buf: int, stream=None) -> int:
        """update("pull_from_upper") of this rank's owned vertices (A/agent.py:224-232): install
        staging buffer `buf` (gxb_attrs_install, owned scope), then refresh every peer's mirror
        of them before the next round. PageRank: the owned contribution slice is all-gathered;
        SSSP / CC / LP: installed values that changed joined the frontier and travel as delta
        records (a vertex already in a peer's frontier is listed once). `stream` must be the
        current torch stream (the collectives are ordered on it). Returns the bytes received."""
        self.state.attrs_install(buf, stream)
        if self.comm.world == 1:
            return 0
        if self.algo == "pagerank":
            return self._exchange_dense()
        return self._exchange_delta()

    def _on_stream(self) -> dict:
        """The library calls run on torch's current stream of this device (explicitly: the
        NCCL collectives of the round are ordered on it, and a user stream context must not
        leave the kernels on the legacy default stream)."""
        if self.device is None:
            return {}
        import torch
        if torch.device(self.device).type != "cuda":
            return {}
        return {"stream": torch.cuda.current_stream(self.device)}

    def _view(self, ptr, nbytes, dtype):
        if hasattr(self.state, "view"):
            return self.state.view(ptr, nbytes, dtype)
        return device_view(ptr, nbytes, dtype)

    def _setup_delta_peers(self) -> bool:
        """Frontier algorithms: map every peer's receive arena (CUDA IPC, handles all-gathered
        once) so the pack kernel stores each changed value only into the arenas of the peers
        whose CSC reads it; all ranks must agree or none uses it (padded all-gather then)."""
        if self._dpeers is not None:
            return self._dpeers
        self._dpeers = False
        if not (self.peer_delta and self.algo != "pagerank" and 1 < self.comm.world <= 8
                and hasattr(self.state, "delta_arena") and hasattr(self.comm.dist, "all_gather_object")):
            return False
        ok = 1
        try:
            send, _ = self.state.exchange_counts()
        except Exception:  # noqa: BLE001
            send, ok = [0] * self.comm.world, 0
        rows = [None] * self.comm.world
        self.comm.dist.all_gather_object(rows, send, group=self.comm.group)
        handle = b""
        if ok:
            try:
                handle = self.state.delta_arena(np.asarray(rows, dtype=np.uint64))
            except Exception:  # noqa: BLE001 - no IPC on this platform
                ok = 0
        handles = [None] * self.comm.world
        self.comm.dist.all_gather_object(handles, handle, group=self.comm.group)
        if ok and all(handles):
            try:
                self.state.delta_open(b"".join(handles))
            except Exception:  # noqa: BLE001
                ok = 0
        else:
            ok = 0
        if self.comm.all_min_flag(ok, self.device) != 1:
            if ok:
                self.state.delta_close()
            return False
        self._dpeers = True
        return True

    def prepare(self):
        """One-time setup outside any timed region: maps the peers' replicas (PageRank) or
        receive arenas (frontier algorithms), else allocates the delta-record buffers."""
        self._setup_peers()
        self._setup_delta_peers()
        if self.comm.world > 1 and self.algo != "pagerank" and hasattr(self.state, "buffer"):
            for which in (L.BUF_SEND, L.BUF_RECV):
                self.state.buffer(which)
        return self

    def _setup_peers(self) -> bool:
        """Map every peer's contribution buffers (CUDA IPC handles, all-gathered once) so
        PageRank's Apply writes the mirrors itself; all ranks must agree or none uses it."""
        if self._peers is not None:
            return self._peers
        self._peers = False
        if not (self.peer_writes and self.algo == "pagerank" and self.comm.world > 1
                and hasattr(self.state, "ipc_handle") and hasattr(self.comm.dist, "all_gather_object")):
            return False
        ok = 1
        try:
            mine = self.state.ipc_handle(0) + self.state.ipc_handle(1)
        except Exception:  # noqa: BLE001 - no IPC on this platform: fall back to NCCL
            mine, ok = b"", 0
        handles = [None] * self.comm.world
        self.comm.dist.all_gather_object(handles, mine, group=self.comm.group)
        if ok and all(handles):
            try:
                peers = b"".join(h for q, h in enumerate(handles) if q != self.comm.rank)
                self.state.open_peers(peers, self.comm.world - 1)
            except Exception:  # noqa: BLE001
                ok = 0
        else:
            ok = 0
        if self.comm.all_min_flag(ok, self.device) != 1:
            if ok:
                self.state.close_peers()
            return False
        # peer order on this rank = ranks ascending without me; the library writes them all
        self._peers = True
        return True

    # ---- one iteration ----------------------------------------------------
    def _tick(self, name, t0):
        if self.phase_times is not None:
            import time
            import torch
            if self.device is not None:
                torch.cuda.synchronize(self.device)
            t = time.perf_counter()
            self.phase_times[name] = self.phase_times.get(name, 0.0) + (t - t0)
            return t
        return t0

    # ---- pipeline shuffle: chunked PageRank round with the exchange overlapped ----
    def _chunk_ranges(self, q: int, k: int, K: int) -> tuple[int, int]:
        lo, hi = int(self.bounds[q]), int(self.bounds[q + 1])
        owned = hi - lo
        pw = L.get_option("xchunk_power") if hasattr(L, "get_option") else 2   # xchunk_bound (csrc/gxb_store.cu)
        b0 = owned * k ** pw // K ** pw
        b1 = owned * (k + 1) ** pw // K ** pw
        return lo + b0, lo + b1

    def _overlapped_pagerank_round(self):
        """Chunks run hubs-last (tail chunks hold many slots but few edges); chunk k's new
        contributions go to every peer while later chunks compute (A/agent.py:282-328's
        upload/compute overlap, on streams and NCCL instead of threads and queues)."""
        st = self.state
        K = self.xchunks
        ptr, nbytes = st.buffer(L.BUF_VALUES_NEXT)
        width = nbytes // max(1, int(self.bounds[-1]))
        values = self._view(ptr, nbytes, "f8" if width == 8 else "f4")
        st.iterate_begin()
        works = []
        for k in reversed(range(K)):
            st.iterate_chunk(k)
            ops = []
            for q in range(self.comm.world):
                if q == self.comm.rank:
                    continue
                a, b = self._chunk_ranges(self.comm.rank, k, K)
                if b > a:
                    ops.append(self.comm.dist.P2POp(self.comm.dist.isend, values[a:b], q, self.comm.group))
                a, b = self._chunk_ranges(q, k, K)
                if b > a:
                    ops.append(self.comm.dist.P2POp(self.comm.dist.irecv, values[a:b], q, self.comm.group))
            if ops:
                works.extend(self.comm.dist.batch_isend_irecv(ops))
        st.iterate_end()
        self._pending = works
        sizes = np.diff(self.bounds.astype(np.int64))
        return width * int(self.bounds[-1] - sizes[self.comm.rank])

    def step(self, direction: str = "auto") -> StepRecord:
        import time
        t0 = time.perf_counter() if self.phase_times is not None else 0.0
        for w in self._pending:  # the previous round's overlapped exchange
            w.wait()
        self._pending = []
        peers = self._setup_peers()
        overlapped = (not peers and self.algo == "pagerank" and self.comm.world > 1 and self.overlap
                      and self.xchunks > 1 and self._pr_remote is not None
                      and not (self.enable_skip and self._pr_remote == 0))
        moved_early = 0
        if overlapped:
            moved_early = self._overlapped_pagerank_round()
        else:
            self.state.iterate(direction, **self._on_stream())
        t0 = self._tick("iterate", t0)
        device_vote = (self.comm.world > 1 and hasattr(self.state, "stats_device")
                       and hasattr(self.comm, "vote_start_device"))
        dpeers = device_vote and self.algo != "pagerank" and self._setup_delta_peers()
        async_delta = device_vote and self.algo != "pagerank" and hasattr(self.state, "pack_async")
        # dense mirror exchange when the previous round changed most vertices (every rank
        # decides from the same global count, so all agree without a collective)
        dense = (device_vote and self.algo != "pagerank" and self.dense_frac > 0 and self._equal_blocks()
                 and self._prev_changed >= self.dense_frac * int(self.bounds[-1]))
        if device_vote:
            # the vote block goes from device stripes straight into the all-gather; the host
            # reads the round's statistics after the collective (one synchronisation per round).
            # Frontier algorithms pack their changed values first: the record count rides along.
            import torch
            if getattr(self, "_vote_buf", None) is None:
                self._vote_buf = torch.zeros(6 + (self.comm.world if dpeers else 0), dtype=torch.float64,
                                             device=self.device)
            if dense:
                if self._vote_buf.numel() > 6:
                    self._vote_buf[6:].zero_()  # no records this round
            elif dpeers:
                # split rounds (option split_overlap): the next round's local-source pass runs
                # beside this round's pack, vote and unpack (a no-op unless this was a dense pull)
                if hasattr(self.state, "iterate_local"):
                    self.state.iterate_local(**self._on_stream())
                self.state.delta_pack(self._vote_buf, **self._on_stream())
            elif async_delta:
                self.state.pack_async(**self._on_stream())
            t0 = self._tick("pack", t0)
            self.state.stats_device(self._vote_buf, **self._on_stream())
            handle = self.comm.vote_start_device(self._vote_buf)
            st = None
        else:
            st = self.state.stats()
            handle = self.comm.vote_start(
                [st["changed"], st["next_active"], st["next_units"], st["remote_active"], 0], st["max_stat"],
                self.device)
        t0 = self._tick("compute", t0)
        moved = moved_early
        early = overlapped
        if peers:  # the round's Apply already stored every owned contribution in every replica
            sizes = np.diff(self.bounds.astype(np.int64))
            ptr, nbytes = self.state.buffer(L.BUF_VALUES)
            moved = nbytes // max(1, int(self.bounds[-1])) * int(self.bounds[-1] - sizes[self.comm.rank])
            early = True
        elif not overlapped and self.algo == "pagerank" and self._pr_remote is not None and self.comm.world > 1:
            # every PageRank vertex is active every round, so the skip vote is the same each
            # round: start the dense exchange behind the vote without waiting for its result
            early = not (self.enable_skip and self._pr_remote == 0)
            if early:
                moved = self._exchange_dense()
        counts, max_stat = self.comm.vote_finish(handle)
        if st is None:
            st = self.state.stats()  # the round is complete: no wait
        t0 = self._tick("vote", t0)
        changed, next_active, next_units, remote_active, _packed = counts
        self._prev_changed = changed
        if self.algo == "pagerank":
            self._pr_remote = remote_active
        self.iteration += 1
        # skip iff no next-active vertex anywhere has a consumer on another partition
        skip = self.comm.world == 1 or (self.enable_skip and remote_active == 0)
        if not skip and not early:
            if self.algo == "pagerank":
                moved = self._exchange_dense()
            elif dense:
                moved = self._exchange_dense_mirror()
            elif dpeers:
                me = self.comm.rank
                counts_from = [0 if p == me else int(r[6 + me]) for p, r in enumerate(self.comm.last_rows)]
                self.state.delta_unpack(counts_from, **self._on_stream())
                moved = sum(counts_from) * self.state.buffer(L.BUF_RECORD_SIZE)[1]
            elif async_delta:
                moved = self._exchange_delta_async([int(r[4]) for r in self.comm.last_rows])
            else:
                moved = self._exchange_delta()
        t0 = self._tick("exchange", t0)
        if self.algo == "pagerank":
            converged = max_stat < 1e-9           # PageRank.vote (A/algorithms.py:164-165)
        else:
            converged = next_active == 0          # not next_active (A/algorithms.py:70-72)
        if skip and self.comm.world > 1 and not converged:
            self.skipped_rounds += 1
        rec = StepRecord(self.iteration, changed, next_active, st["units"], remote_active, max_stat,
                         skip and self.comm.world > 1, converged, moved, st["direction"])
        self.records.append(rec)
        return rec

    def finish(self):
        """Complete any exchange still in flight (the replica is then fully current)."""
        for w in self._pending:
            w.wait()
        self._pending = []

    def can_run_ahead(self) -> bool:
        return (self.algo == "pagerank" and hasattr(self.state, "stats_async")
                and hasattr(self.state, "stats_device") and hasattr(self.state, "rollback"))

    def run_rounds(self, n: int) -> list:
        """Up to n PageRank rounds back to back: round k+1 is launched before the host reads
        round k's vote, so the GPU never waits for the host between rounds. The vote blocks go
        from the device (all-gathered at N > 1) into a pinned ring read one round behind; when
        round k converged, the already-launched round k+1 is rolled back (its rank and
        contributions went to the next buffers only), so results and iteration counts equal
        the round-by-round loop (A/algorithms.py:318-341)."""
        import torch
        if not self.can_run_ahead() or n <= 0:
            return [self.step() for _ in range(n)]
        world = self.comm.world
        dev = self.device
        peers = self._setup_peers() if world > 1 else False
        if world > 1 and not peers:
            return [self.step() for _ in range(n)]  # the NCCL dense exchange is issued per round
        out = []
        bufs = [torch.empty(6, dtype=torch.float64, device=dev) for _ in range(2)]
        host = [torch.empty(world * 6, dtype=torch.float64).pin_memory() for _ in range(2)]
        evs = [torch.cuda.Event() for _ in range(2)]
        sizes = np.diff(self.bounds.astype(np.int64))
        ptr, nbytes = self.state.buffer(L.BUF_VALUES)
        moved = 0 if world == 1 else nbytes // max(1, int(self.bounds[-1])) * int(self.bounds[-1] - sizes[self.comm.rank])
        self.state.stats()  # settle the last synchronous round
        self.state.stats_async(True)
        try:
            launched = 0

            def launch(k):
                self.state.iterate("pull", **self._on_stream())
                self.state.stats_device(bufs[k % 2], **self._on_stream())
                rows = self.comm.vote_start_device(bufs[k % 2]) if world > 1 else bufs[k % 2]
                host[k % 2].copy_(rows, non_blocking=True)
                evs[k % 2].record()

            launch(0)
            launched = 1
            for k in range(n):
                if launched < n:
                    launch(launched)
                    launched += 1
                evs[k % 2].synchronize()
                rows = host[k % 2].view(world, 6).tolist()
                changed, next_active, next_units, remote_active = (int(sum(r[i] for r in rows)) for i in range(4))
                max_stat = max(r[5] for r in rows)
                self.iteration += 1
                self._pr_remote = remote_active
                converged = max_stat < 1e-9  # PageRank.vote (A/algorithms.py:164-165)
                skip = world == 1 or (self.enable_skip and remote_active == 0)
                units = int(rows[self.comm.rank][2])  # this rank's GEN units (every owned vertex)
                rec = StepRecord(self.iteration, changed, next_active, units, remote_active, max_stat,
                                 skip and world > 1, converged, moved, 1)
                self.records.append(rec)
                out.append(rec)
                if converged:
                    if launched > k + 1:  # round k+2 (1-based) already ran: undo it
                        torch.cuda.synchronize(dev)
                        self.state.rollback()
                    break
        finally:
            torch.cuda.synchronize(dev)
            self.state.stats_async(False)
        return out

    def run(self, max_iterations: int, direction: str = "auto") -> tuple[int, bool]:
        converged = False
        while self.iteration < max_iterations:
            if self.step(direction).converged:
                converged = True
                break
        self.finish()
        return self.iteration, converged
