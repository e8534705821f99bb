"""Upper-system driver: BSP / GAS iterations over partitioned device state.

Drop-in for the reference's `Engine` / `run` (A/engine.py:172-427). The
reference simulates m nodes as threads sharing a barrier; here the m partitions
are destination ranges of the device store (on one GPU in one process — the
multi-process / multi-GPU driver is `dist.PartitionedRun`). The per-iteration
schedule is the reference's barrier schedule (A/engine.py:226-294):

    work phase    Gen (requestGen) -> Merge (requestMerge) -> Apply (requestApply)
    route         nothing to route: the pull design merges locally, remote
                  sources are mirrored
    skip          AND over partitions of "no next-active vertex has a remote
                  consumer" (A/engine.py:242-246) when enable_skip
    sync round    mirror exchange of changed values (A/engine.py:247-266)
    verdict       AND of the votes, apply-round cap (A/engine.py:267-285)

GAS (A/agent.py:476-486) runs a seed Gen pass in iteration 1 and then
Merge -> Apply -> push -> Gen; the seed round is excluded from the cap.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .agent import GpuAgent
from .channel import trace_conforms
from .daemon import AcceleratorProfile


class EngineError(RuntimeError):
    pass


class ComputationModel(Enum):
    BSP = "bsp"
    GAS = "gas"


@dataclass
class RunConfig:
    """Same keys as the reference (A/engine.py:45-60). enable_cache / cache_* are accepted for
    compatibility: every mirror fits in HBM, so the weighted-LRU policy is moot."""

    partitions: int = 1
    daemons_per_node: int = 1
    daemon_profile: AcceleratorProfile = field(default_factory=lambda: AcceleratorProfile(lanes=4))
    node_profiles: list[AcceleratorProfile] | None = None
    block_size: int | str = 1 << 22
    enable_cache: bool = False
    cache_capacity: int = 1024
    cache_decay: float = 0.5
    cache_boost: float = 1.0
    enable_skip: bool = False
    io_cost: float = 0.01
    seed: int = 0
    max_iterations: int | None = None
    barrier_timeout: float = 60.0
    fused: bool = False          # True: one fused device pass per iteration instead of requestX passes
    direction: str = "auto"
    device: int = 0
    partitioning: str = "ids"    # "ids": contiguous ascending-id ranges like partition_graph (A/graph.py:175-212);
                                 # "edges": destination ranges balanced by in-edges (the multi-GPU default)
    sizes: list[int] | None = None  # explicit partition sizes (partition_graph's `sizes`)
    capacity: list[float] | None = None  # per-partition capacity factors (balancer.capacity_factors):
                                         # degree-sorted ranges cut in proportion (A/balancer.py:79-98)


@dataclass
class IterationRecord:
    iteration: int
    model: str
    t_download: float
    t_compute: float
    t_upload: float
    skipped: bool
    cache_hits: int
    cache_misses: int
    uploads: int
    uploads_avoided: int
    converged: bool

    def to_line(self) -> str:
        """The reference's metrics line format (A/engine.py:77-85)."""
        return (
            f"iter={self.iteration} model={self.model} "
            f"t_download={self.t_download:.6f} t_compute={self.t_compute:.6f} "
            f"t_upload={self.t_upload:.6f} skipped={str(self.skipped).lower()} "
            f"cache_hits={self.cache_hits} cache_misses={self.cache_misses} "
            f"uploads={self.uploads} uploads_avoided={self.uploads_avoided} "
            f"converged={str(self.converged).lower()}"
        )


@dataclass
class NodeStats:
    iteration: int
    node_id: int
    units: int
    blocks: int
    compute_time: float
    pipeline_time: float
    download_time: float
    upload_time: float


@dataclass
class RunMetrics:
    model: str
    records: list[IterationRecord] = field(default_factory=list)
    node_stats: list[NodeStats] = field(default_factory=list)
    converged: bool = False
    iterations: int = 0
    skipped_rounds: int = 0
    block_plans: dict[int, tuple[int, int]] = field(default_factory=dict)
    init_counts: dict[str, int] = field(default_factory=dict)
    copy_counts: dict[str, int] = field(default_factory=dict)
    traces: dict[str, list[str]] = field(default_factory=dict)
    exchanged_bytes: int = 0

    def lines(self) -> list[str]:
        return [r.to_line() for r in self.records]

    def write(self, path) -> None:
        with open(path, "w", encoding="ascii") as fh:
            for line in self.lines():
                fh.write(line + "\n")

    def protocol_conformant(self) -> bool:
        return all(trace_conforms(t) for t in self.traces.values())


def convergence_vote(votes: list) -> bool:
    """Logical AND over per-node votes; a missing vote is fatal (A/engine.py:131-136)."""
    if any(v is None for v in votes):
        missing = [i for i, v in enumerate(votes) if v is None]
        raise EngineError(f"missing convergence vote from node(s) {missing}")
    return all(votes)


def exchange_local(states, bounds) -> int:
    """Sync round between partitions that live in this process (device-to-device copies).

    PageRank: the owned slice of every partition's contribution replica is copied into all
    other replicas. Others: changed (slot, value) records are packed by the owner and
    installed by every peer (A/sync.py:171-198)."""
    from . import _lib as L
    from .dist import device_view

    m = len(states)
    if m <= 1:
        return 0
    moved = 0
    if states[0].algo == "pagerank":
        width = states[0].buffer(L.BUF_VALUES)[1] // max(1, int(bounds[-1]))
        views = [device_view(*s.buffer(L.BUF_VALUES), "f8" if width == 8 else "f4") for s in states]
        for j in range(m):
            lo, hi = int(bounds[j]), int(bounds[j + 1])
            for k in range(m):
                if k != j and hi > lo:
                    views[k][lo:hi].copy_(views[j][lo:hi])
                    moved += width * (hi - lo)
        return moved
    rec = states[0].buffer(L.BUF_RECORD_SIZE)[1]
    counts = [s.pack() for s in states]
    sends = [device_view(*s.buffer(L.BUF_SEND), "u1") for s in states]
    total = sum(counts)
    for k, s in enumerate(states):
        rptr, rbytes = s.buffer(L.BUF_RECV)
        recv = device_view(rptr, rbytes, "u1")
        off = 0
        for j in range(m):
            n = counts[j] * rec
            if n:
                recv[off:off + n].copy_(sends[j][:n])
                if j != k:
                    moved += n
            off += n
        s.unpack(rptr, total)
    return moved


class Engine:
    def __init__(self, graph, algorithm, model: ComputationModel | str, config: RunConfig):
        self.graph_input = graph
        self.algorithm = algorithm
        self.model = ComputationModel(model) if isinstance(model, str) else model
        self.config = config
        self.metrics = RunMetrics(model=self.model.value)
        self.agents: list[GpuAgent] = []
        self.states = []
        self.graphs = []

    def _edges(self):
        from .graph import EdgeArrays
        g = self.graph_input
        if isinstance(g, EdgeArrays):
            return g
        if isinstance(g, tuple) and len(g) == 2:
            return EdgeArrays.from_edges(list(g[1]))
        if hasattr(g, "partitions"):  # a reference-style PartitionedGraph
            return EdgeArrays.from_edges([e for p in g.partitions for e in p.edges])
        raise TypeError("graph must be EdgeArrays, (vertices, edges) or a PartitionedGraph")

    def _setup(self):
        from .device import DeviceContext, DeviceGraph, DeviceState
        cfg = self.config
        ea = self._edges()
        algo = self.algorithm.device_name
        self.ctx = DeviceContext(cfg.device)
        m = max(1, int(cfg.partitions))
        w = ea.weight if algo == "sssp" else None
        maxw = int(np.max(w)) if (w is not None and w.size) else 1
        for j in range(m):
            g = DeviceGraph(self.ctx, ea.src, ea.dst, w, part=j, nparts=m, csr=algo in ("sssp", "cc", "lp"),
                            partitioning=cfg.partitioning, sizes=cfg.sizes, capacity=cfg.capacity)
            s = DeviceState(g, algo, sources=getattr(self.algorithm, "sources", None) if algo == "sssp" else None,
                            max_weight=maxw if algo == "sssp" else None)
            self.graphs.append(g)
            self.states.append(s)
        self.bounds = self.graphs[0].bounds()
        for j, s in enumerate(self.states):
            agent = GpuAgent(j, s, self.algorithm, model=self.model.value, block_size=cfg.block_size,
                             io_cost=cfg.io_cost, recv_timeout=cfg.barrier_timeout, fused=cfg.fused)
            base = cfg.node_profiles[j] if cfg.node_profiles is not None else cfg.daemon_profile
            agent.connect([base] * cfg.daemons_per_node)
            self.agents.append(agent)
        self.cap = cfg.max_iterations
        if self.cap is None:
            self.cap = self.algorithm.default_iteration_cap(self.graphs[0].num_vertices)

    def run(self) -> tuple[dict[int, object], RunMetrics]:
        self._setup()
        try:
            self._loop()
        finally:
            for agent in self.agents:
                agent.shutdown()
            self._collect_instrumentation()
        attrs = self._read_attrs()
        return attrs, self.metrics

    def _loop(self):
        agents, cfg = self.agents, self.config
        gas = self.model is ComputationModel.GAS
        iteration, apply_rounds = 0, 0
        if gas:
            # seed Gen pass (A/agent.py:476-486); excluded from the cap (A/engine.py:271-275)
            iteration = 1
            for a in agents:
                a.begin_iteration()
                a.gen_phase()
                a.end_iteration()
            # the seed round still takes the skip vote on the initial frontier (A/engine.py:242-246)
            seed_skip = cfg.enable_skip and all(a.device_state.stats()["remote_active"] == 0 for a in agents)
            if seed_skip and len(agents) > 1:
                self.metrics.skipped_rounds += 1
            self._record(iteration, skipped=seed_skip and len(agents) > 1, converged=False, agents=agents)
            if self.cap <= 0:
                return
        while apply_rounds < self.cap:
            iteration += 1
            for a in agents:
                a.begin_iteration()
                if not gas:
                    a.gen_phase()
                a.merge_apply_phase()
            closed = [a.round_closed() for a in agents]
            skip = cfg.enable_skip and all(closed)
            moved = 0 if (skip or len(agents) == 1) else exchange_local(self.states, self.bounds)
            self.metrics.exchanged_bytes += moved
            converged = convergence_vote([a.vote() for a in agents])
            apply_rounds += 1
            if skip and not converged:
                self.metrics.skipped_rounds += 1
            stop = converged or apply_rounds >= self.cap
            if gas and not stop:
                for a in agents:
                    a.gen_phase()  # ... -> push -> Gen for the next iteration
            for a in agents:
                a.end_iteration()
            self._record(iteration, skip and len(agents) > 1 and cfg.enable_skip, converged, agents, moved)
            if stop:
                self.metrics.converged = converged
                self.metrics.iterations = iteration
                break

    def _record(self, iteration, skipped, converged, agents, moved=0):
        cs = [a.counters for a in agents]
        self.metrics.records.append(IterationRecord(
            iteration=iteration, model=self.model.value,
            t_download=max(c.t_download for c in cs), t_compute=max(c.t_compute for c in cs),
            t_upload=max(c.t_upload for c in cs), skipped=skipped, cache_hits=0, cache_misses=0,
            uploads=moved, uploads_avoided=0, converged=converged))
        for a in agents:
            c = a.counters
            self.metrics.node_stats.append(NodeStats(iteration, a.node_id, c.units, c.blocks, c.t_compute,
                                                     c.pipeline_time, c.t_download, c.t_upload))

    def _collect_instrumentation(self):
        for agent in self.agents:
            for daemon in agent.daemons:
                key = daemon.state.channel_key
                self.metrics.init_counts[key] = daemon.init_count
                self.metrics.copy_counts[key] = daemon.region.copy_count
                self.metrics.traces[key] = list(daemon.region.trace)

    def _read_attrs(self) -> dict[int, object]:
        ids = self.graphs[0].ids()
        rows = None
        for s in self.states:
            r = s.read_attrs(owned_only=len(self.states) > 1)
            if rows is None:
                rows = r
            else:
                mask = ~np.isnan(r[:, 0])
                rows[mask] = r[mask]
        return {int(v): self.algorithm.attr_from_row(int(v), rows[i]) for i, v in enumerate(ids)}


def run(graph, algorithm, model: ComputationModel | str, config: RunConfig) -> tuple[dict[int, object], RunMetrics]:
    """Run one algorithm over a partitioned graph; returns (attrs, metrics) (A/engine.py:422-427)."""
    return Engine(graph, algorithm, model, config).run()


def dump_attributes(attrs: dict[int, object], algorithm) -> str:
    """Diff-friendly dump: ascending vertex id, one 'id value(s)' per line (A/engine.py:430-433)."""
    lines = [f"{vid} {algorithm.format_attr(attr)}" for vid, attr in sorted(attrs.items())]
    return "\n".join(lines) + ("\n" if lines else "")
