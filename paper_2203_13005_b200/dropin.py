"""The B200 daemon dropped into an unmodified reference process (`accelgraph`).

GX-Plug is a plug-in: the upper graph system keeps its engine, partitions, agents,
shared regions and synchronisation rounds, and only the daemon behind the agent
interface changes. This module does exactly that for the reference system, through
the three module-attribute seams SURVEY.md §8(b) verified without editing it:

    accelgraph.agent.daemon_init     (called by Agent.connect, A/agent.py:186)
        -> gpu_daemon_init: a GpuDaemon (subclass of the reference's Daemon) whose
           persistent initialisation opens the B200 (gxb_init, once per daemon)
    accelgraph.daemon.execute_request (called by Daemon._loop, A/daemon.py:191)
        -> execute_request: runs a work item's range on the device (gxb_request /
           gxb_iterate) instead of Python triplet loops
    accelgraph.engine.Agent          (constructed by Engine._setup, A/engine.py:205)
        -> GpuAgent: the reference's Agent with the work-item construction, result
           assembly and mirror handling replaced (`_build_work_items`,
           `_absorb_results`, `_ensure_remote_attrs`, SURVEY.md §8(b) "Implication")

Everything else is the reference's own code: `Engine` and its barrier schedule, the
`SharedRegion` three-slot protocol and its trace, `Agent.request` / `_drive` (Alg. 2),
`Daemon._loop` (Alg. 1), `RunConfig`, `IterationRecord`, the CLI.

What a work item is here. The reference ships one `EdgeTriplet` per frontier out-edge
through the region (`build_blocks`, A/graph.py:215-245). A GpuAgent ships a
`DeviceRange` (an op over a range of the device-resident CSC edges or owned slots) or,
on the default fused path, one `FusedRound` (Gen -> Merge -> Apply of the partition in
one device pass); results never leave HBM.

Pull instead of push. Every GpuAgent holds the in-edges (CSC) of the destinations its
partition owns and a replica of every source value, so MSGMerge never needs remote
messages: the route step carries nothing (the reference's combiner output is empty)
and the values that cross partitions are source attributes, moved by the reference's
own synchronisation round — `publish_queries` names the remote sources this partition
reads, `serve_uploads` uploads the owned values that changed (dirty; with the cache on,
dirty and queried), and `deliver` installs the delivered values of the queried sources
into the device replica, where they become active sources of the next round
(`gxb_attrs_deliver`). The skip vote is the device's remote-active count: a round whose
next frontier has no consumer on another partition skips the exchange
(A/agent.py:533-535, A/engine.py:242-246), which is sound for pull for the same reason
it is for push (the changed set is the next frontier).

The reference package must be importable: it is found on sys.path, else in
`<repo>/baseline/_ref` (the offline install of /root/reference), else ImportError.
"""

from __future__ import annotations

import importlib
import os
import sys
import threading
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from . import _lib as L

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_REF_DIRS = (os.path.join(_REPO, "baseline", "_ref"),)


def reference():
    """Import the reference package `accelgraph` (sys.path, then baseline/_ref)."""
    try:
        return importlib.import_module("accelgraph")
    except ImportError:
        pass
    for d in _REF_DIRS:
        if os.path.isdir(os.path.join(d, "accelgraph")):
            if d not in sys.path:
                sys.path.append(d)
            return importlib.import_module("accelgraph")
    raise ImportError("the reference package 'accelgraph' is not importable (sys.path or baseline/_ref)")


_ag = reference()
_agent_mod = importlib.import_module("accelgraph.agent")
_daemon_mod = importlib.import_module("accelgraph.daemon")
_engine_mod = importlib.import_module("accelgraph.engine")
_channel_mod = importlib.import_module("accelgraph.channel")
OpKind = _channel_mod.OpKind
WorkItem = _channel_mod.WorkItem
ProtocolError = _channel_mod.ProtocolError

DEVICE_ALGOS = ("sssp", "pagerank", "lp", "cc")


@dataclass
class DropinConfig:
    """Options of the device path (the reference's RunConfig has no slot for them)."""

    device: int = 0
    fused: bool = True        # one fused Gen->Merge->Apply device pass per iteration
    direction: str = "auto"   # pull / push / auto (direction-optimising frontier rounds)


CONFIG = DropinConfig()


# --------------------------------------------------------------------------- work items

@dataclass(frozen=True)
class DeviceRange:
    """A template op over [lo, hi): GEN over owned CSC edges, MERGE / APPLY over owned slots."""

    agent: "GpuAgent"
    op: object
    lo: int
    hi: int


@dataclass(frozen=True)
class FusedRound:
    """Gen -> Merge -> Apply of the whole partition in one device pass (gxb_iterate)."""

    agent: "GpuAgent"


_OPS = {}


def _op_code(kind) -> int:
    if not _OPS:
        _OPS.update({OpKind.GEN: L.OP_GEN, OpKind.MERGE: L.OP_MERGE, OpKind.APPLY: L.OP_APPLY})
    return _OPS[kind]


def execute_request(algorithm, profile, item) -> float:
    """Drop-in for execute_request (A/daemon.py:86-130): run the item on the device, in
    situ. `item.result` stays None (results live in HBM), `result_units` counts the
    messages (GEN), merged targets (MERGE) or applied vertices (APPLY) of the range.
    Returns the simulated cost, same formula as the reference (A/daemon.py:130)."""
    payload = item.payload
    if isinstance(payload, FusedRound):
        a = payload.agent
        with a._device_lock:
            a.device_state.iterate(a.direction)
        item.result_units = item.units
    elif isinstance(payload, DeviceRange):
        a = payload.agent
        if item.kind is not payload.op:
            raise ValueError(f"work item kind {item.kind!r} does not match its range op {payload.op!r}")
        with a._device_lock:
            a.device_state.request(_op_code(payload.op), payload.lo, payload.hi)
        item.result_units = payload.hi - payload.lo
    else:
        raise TypeError("the B200 daemon executes device work items only (DeviceRange / FusedRound); "
                        f"got {type(payload).__name__} — build work items with dropin.GpuAgent")
    item.result = None
    return profile.call_overhead + profile.per_unit_cost * item.units


# --------------------------------------------------------------------------- daemon

class GpuDaemon(_daemon_mod.Daemon):
    """The reference's Daemon (lifecycle, Alg. 1 service loop, error surfacing) bound to
    one B200: `initialize()` additionally opens the device (`gxb_init`) exactly once."""

    def __init__(self, profile, algorithm, channel_key, channels, device: int = 0):
        super().__init__(profile, algorithm, channel_key, channels)
        self.device = device
        self.context = None

    def initialize(self):
        if self.state.phase is _daemon_mod.DaemonPhase.UNINITIALIZED:
            from .device import DeviceContext
            self.context = DeviceContext(self.device)  # fails loudly without a B200
        return super().initialize()  # ProtocolError on re-initialisation (A/daemon.py:148-161)

    def shutdown(self) -> None:
        super().shutdown()
        if self.context is not None:
            self.context.shutdown()
            self.context = None


def gpu_daemon_init(profile, algorithm, channel_key, channels) -> GpuDaemon:
    """Drop-in for daemon_init (A/daemon.py:207-212)."""
    daemon = GpuDaemon(profile, algorithm, channel_key, channels, device=CONFIG.device)
    daemon.initialize()
    return daemon


# --------------------------------------------------------------------------- agent

def device_algorithm(algorithm) -> str:
    name = getattr(algorithm, "name", None)
    if name not in DEVICE_ALGOS:
        raise ValueError(f"algorithm {name!r} has no device kernels (device algorithms: {DEVICE_ALGOS})")
    return name


def _edge_arrays(graph):
    """All partitions' edges as (src, dst, w) arrays; cached on the PartitionedGraph."""
    cached = getattr(graph, "_gxb_edges", None)
    if cached is not None:
        return cached
    edges = [e for p in graph.partitions for e in p.edges]
    n = len(edges)
    src = np.fromiter((e.src for e in edges), dtype=np.int64, count=n)
    dst = np.fromiter((e.dst for e in edges), dtype=np.int64, count=n)
    w = np.fromiter((e.weight for e in edges), dtype=np.float64, count=n)
    if n and (min(src.min(), dst.min()) < 0 or max(src.max(), dst.max()) >= 0xFFFFFFFF):
        raise ValueError("device vertex ids must be in [0, 2^32-1)")
    out = (src.astype(np.uint32), dst.astype(np.uint32), w)
    try:
        graph._gxb_edges = out
    except AttributeError:
        pass
    return out


class GpuAgent(_agent_mod.Agent):
    """The reference's Agent (A/agent.py:96-622) with device work items."""

    def __init__(self, *args, **kwargs):
        super().__init__(*args, **kwargs)
        self.direction = CONFIG.direction
        self.algo_name = device_algorithm(self.algorithm)
        # LP folds a label multiset, which has no materialised-message form: always fused
        self.fused = CONFIG.fused or self.algo_name == "lp"
        self.device_state = None
        self.device_graph = None
        self._device_lock = threading.Lock()
        self._seed_pass = False
        self.stats = None

    # The device holds the frontier; the upper system's frontier sets are not needed.
    @property
    def frontier(self):
        return frozenset()

    @frontier.setter
    def frontier(self, value):
        pass

    def connect(self, daemon_profiles):
        state = super().connect(daemon_profiles)
        try:
            self._build_device()
        except BaseException:
            self.shutdown()
            raise
        return state

    def _build_device(self):
        from .device import DeviceGraph, make_state
        ctx = self.daemons[0].context
        if ctx is None:
            raise ProtocolError(f"node {self.node_id}: daemon {self.daemons[0].state.channel_key} has no device "
                                "(install the drop-in: dropin.install())")
        graph, part = self.graph, self.partition
        src, dst, w = _edge_arrays(graph)
        present = np.unique(np.concatenate([src, dst])) if src.size else np.zeros(0, np.uint32)
        if present.size != graph.num_vertices:
            raise ValueError("device partitions need every vertex to appear in an edge "
                             f"({graph.num_vertices} vertices, {present.size} present in edges)")
        sizes = [len(p.vertices) for p in graph.partitions]
        algo = self.algo_name
        weights = w if algo == "sssp" else None
        self.device_graph = DeviceGraph(ctx, src, dst, weights, part=self.node_id, nparts=len(sizes),
                                        csr=algo != "pagerank", partitioning="ids", sizes=sizes)
        sources = list(self.algorithm.sources) if algo == "sssp" else None
        maxw = int(np.max(weights)) if weights is not None and weights.size else None
        self.device_state = make_state(self.device_graph, algo, sources=sources, max_weight=maxw)
        self._ids = self.device_graph.ids()
        owned = np.fromiter(sorted(part.vertices), dtype=np.int64, count=len(part.vertices))
        self._owned_pos = np.searchsorted(self._ids, owned)
        if owned.size and not np.array_equal(self._ids[self._owned_pos], owned):
            raise ValueError(f"node {self.node_id}: partition vertices are not the device partition's")
        self._owned_ids = owned
        self._snapshot = self._owned_rows()       # last values the upper system has seen
        # remote sources this partition's in-edges read (static): the pull analogue of the
        # next frontier's remote destinations (A/agent.py:542-548)
        own_mask = np.zeros(self._ids.size, dtype=bool)
        own_mask[self._owned_pos] = True
        si = np.searchsorted(self._ids, src)
        di = np.searchsorted(self._ids, dst)
        need = np.unique(si[own_mask[di] & ~own_mask[si]])
        self._needed_pos = need
        self._needed = frozenset(int(v) for v in self._ids[need])

    def shutdown(self) -> None:
        with self._device_lock:
            if self.device_state is not None:
                self.device_state.free()
                self.device_state = None
            if self.device_graph is not None:
                self.device_graph.free()
                self.device_graph = None
        super().shutdown()

    # ---- attribute conversion (device rows <-> the reference's attribute objects) ----
    def _owned_rows(self) -> np.ndarray:
        rows = self.device_state.read_attrs(owned_only=self.graph.num_nodes > 1)
        return rows[self._owned_pos]

    def _attr(self, vid: int, row: np.ndarray):
        a = self.algo_name
        if a == "sssp":
            return tuple(float(x) for x in row)
        if a == "pagerank":
            return (float(row[0]), self.algorithm.out_degree[vid])
        return int(row[0])

    def _row(self, attr) -> list[float]:
        a = self.algo_name
        if a == "sssp":
            return [float(x) for x in attr]
        if a == "pagerank":
            return [float(attr[0])]
        return [float(attr)]

    def _dirty(self):
        """Owned vertices whose value differs from what the upper system last saw."""
        rows = self._owned_rows()
        diff = np.any(rows != self._snapshot, axis=1)
        return rows, np.flatnonzero(diff)

    # ---- work items (A/agent.py:352-402) ----
    def _build_work_items(self, op_kind):
        st = self.device_state
        if self._seed_pass:
            return []
        if self.fused:
            if op_kind is not OpKind.GEN:
                return []
            units = max(1, int(self.stats["next_units"]) if self.stats else
                        int(self.device_graph.info.owned_out_edges))
            self._set_capacity(units)
            return [WorkItem(OpKind.GEN, 0, FusedRound(self), units)]
        if op_kind is OpKind.GEN:
            lo, hi = 0, int(self.device_graph.info.owned_edges)
        elif op_kind in (OpKind.MERGE, OpKind.APPLY):
            lo, hi = self.device_graph.owned
        else:
            raise ValueError(f"unknown operation kind {op_kind!r}")
        if st is None:
            raise ProtocolError(f"node {self.node_id}: no device state (connect() first)")
        b = self._plan_block_size(hi - lo)
        self._set_capacity(b)
        return [WorkItem(op_kind, i, DeviceRange(self, op_kind, s, min(hi, s + b)), min(hi, s + b) - s)
                for i, s in enumerate(range(lo, hi, b))]

    def _absorb_results(self, op_kind, done):
        if self.fused:
            if op_kind is OpKind.GEN and done:
                self._round_closed()
            return
        if op_kind is OpKind.APPLY:
            with self._device_lock:
                self.device_state.commit()
            self._round_closed()

    def _round_closed(self):
        self.stats = self.device_state.stats()
        self._applied_this_iteration = True

    def _ensure_remote_attrs(self, frontier) -> None:
        """Pull design: destination attributes are never read by any algorithm (SURVEY.md
        §8(a) a3) and source mirrors are refreshed by `deliver`; nothing to fetch."""

    def _push_updates(self) -> None:
        """Changed values stay on the device until serve_uploads / flush_all read them."""

    # ---- iteration phases (A/agent.py:469-502) ----
    def work_phase(self, iteration: int) -> dict:
        if self.model == "bsp":
            self.update("pull_from_upper")
            self.request(OpKind.GEN)
            self.request(OpKind.MERGE)
            return self._export_remote_merged()
        # GAS: the seed Gen pass of iteration 1 materialises nothing in the pull design (it
        # runs as an empty pass); an iteration k > 1 runs Gen on the values the last sync
        # round delivered, then Merge and Apply.
        if iteration > 1:
            self.update("pull_from_upper")
            self.request(OpKind.GEN)
            self.request(OpKind.MERGE)
            self.request(OpKind.APPLY)
            self.update("push_to_upper")
        else:
            self._seed_pass = True
            try:
                self.request(OpKind.GEN)
            finally:
                self._seed_pass = False
        return self._export_remote_messages()

    def _export_remote_merged(self) -> dict:
        return {}  # every merged target is owned: nothing to route

    def _export_remote_messages(self) -> dict:
        return {}

    def post_route(self, inbox: list) -> None:
        if inbox:
            raise ProtocolError(f"node {self.node_id}: the device path routes no messages, got {len(inbox)}")
        if self.model == "bsp":
            self.request(OpKind.APPLY)
            self.update("push_to_upper")

    def round_closed(self) -> bool:
        """No next-active vertex has a consumer on another partition (A/agent.py:533-535).
        Before any Apply (the GAS seed round) the next frontier is the initial one."""
        st = self.stats if self.stats is not None else self.device_state.stats()
        return st["remote_active"] == 0

    def vote(self) -> bool:
        if not self._applied_this_iteration:
            return False
        return bool(self.stats["voted"])

    # ---- synchronisation round (A/agent.py:542-611) ----
    def publish_queries(self) -> frozenset:
        self._last_queries = self._needed
        return self._needed

    def serve_uploads(self, gqq):
        rows, dirty = self._dirty()
        serve = dirty
        if self.cache is not None:  # lazy upload: dirty and queried (A/sync.py:171-198)
            ids = self._owned_ids[dirty]
            q = np.fromiter(gqq, dtype=np.int64, count=len(gqq)) if gqq else np.zeros(0, np.int64)
            serve = dirty[np.isin(ids, q)]
        uploads = self._take(rows, serve)
        self.counters.uploads += len(uploads)
        self.counters.uploads_avoided += int(dirty.size - serve.size)
        self.counters.t_upload += self.io_cost * len(uploads)
        return uploads, {}

    def _take(self, rows, idx) -> dict:
        table = self.partition.vertices
        out = {}
        for i in idx.tolist():
            vid = int(self._owned_ids[i])
            attr = self._attr(vid, rows[i])
            out[vid] = attr
            v = table[vid]
            v.attr = attr
            v.updated = False
        self._snapshot[idx] = rows[idx]
        return out

    def deliver(self, gqq, gdq) -> None:
        if not gdq:
            return
        vids = np.fromiter(gdq.keys(), dtype=np.int64, count=len(gdq))
        pos = np.searchsorted(self._ids, vids)
        pos = np.minimum(pos, max(0, self._ids.size - 1))
        ok = (self._ids[pos] == vids) & np.isin(pos, self._needed_pos)
        if not ok.any():
            return
        keep = np.flatnonzero(ok)
        vals = np.asarray([self._row(gdq[int(vids[i])]) for i in keep.tolist()], dtype=np.float64)
        with self._device_lock:
            self.device_state.deliver(pos[keep].astype(np.uint64), vals)
        self.counters.t_download += self.io_cost * int(keep.size)

    def flush_all(self) -> dict:
        rows, dirty = self._dirty()
        out = self._take(rows, dirty)
        self.counters.uploads += len(out)
        self.counters.t_upload += self.io_cost * len(out)
        return out


# --------------------------------------------------------------------------- install

_SEAMS = (
    (_agent_mod, "daemon_init", gpu_daemon_init),
    (_daemon_mod, "execute_request", execute_request),
    (_engine_mod, "Agent", GpuAgent),
)
_saved: dict = {}


def install(device: int | None = None, fused: bool | None = None, direction: str | None = None) -> None:
    """Rebind the reference's three seams to the B200 path (idempotent)."""
    if device is not None:
        CONFIG.device = int(device)
    if fused is not None:
        CONFIG.fused = bool(fused)
    if direction is not None:
        if direction not in ("auto", "pull", "push"):
            raise ValueError(f"unknown direction {direction!r}")
        CONFIG.direction = direction
    for mod, name, repl in _SEAMS:
        key = (mod.__name__, name)
        if key not in _saved:
            _saved[key] = getattr(mod, name)
        setattr(mod, name, repl)


def uninstall() -> None:
    """Restore the reference's own daemon, request executor and agent."""
    for mod, name, _ in _SEAMS:
        key = (mod.__name__, name)
        if key in _saved:
            setattr(mod, name, _saved.pop(key))


def installed_now() -> bool:
    return all(getattr(mod, name) is repl for mod, name, repl in _SEAMS)


@contextmanager
def installed(**options):
    """`with dropin.installed(): accelgraph.engine.run(...)` — the B200 path inside the block."""
    prev = (CONFIG.device, CONFIG.fused, CONFIG.direction)
    was = installed_now()
    install(**options)
    try:
        yield
    finally:
        CONFIG.device, CONFIG.fused, CONFIG.direction = prev
        if not was:
            uninstall()


def main(argv=None) -> int:
    """`python -m paper_2203_13005_b200.dropin run --graph g.txt --algo sssp ...`: the
    reference's own CLI (A/cli.py) with the B200 daemon installed."""
    cli = importlib.import_module("accelgraph.cli")
    with installed():
        return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
