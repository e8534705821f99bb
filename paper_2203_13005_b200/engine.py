"""Device-only BSP / GAS driver for m partitions in one process (one GPU).

The reference-compatible way to run an algorithm over partitions is the reference's
own `Engine` with the B200 daemon dropped in (`dropin.install()`, A/engine.py:172-427
unmodified). This module is the same schedule without the upper system: no Python
partition tables, agents or shared regions — each partition is a device state and the
per-iteration barrier schedule of A/engine.py:226-294 is driven directly:

    work phase    fused Gen∘Merge∘Apply (gxb_iterate), or the request path:
                  GEN / MERGE / APPLY over block ranges (gxb_request) + commit
    skip          AND over partitions of "no next-active vertex has a remote
                  consumer" (A/engine.py:242-246), when enable_skip
    sync round    mirror exchange of changed values between the partitions'
                  device replicas (`exchange_local`, device-to-device copies)
    verdict       AND of the votes (A/engine.py:131-136), apply-round cap

GAS (A/agent.py:476-486) takes a seed round in iteration 1 (no Apply, not counted
against the cap) and then Merge -> Apply -> Gen; in the pull design its Gen reads the
values the previous sync round delivered, so each later iteration is one device round.
The multi-process, multi-GPU driver with the same schedule is `dist.PartitionedRun`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .dist import StepRecord


class EngineError(RuntimeError):
    pass


MODELS = ("bsp", "gas")


@dataclass
class RunConfig:
    partitions: int = 1
    block_size: int = 1 << 22     # request-path block (range) length
    enable_skip: bool = False
    max_iterations: int | None = None
    fused: bool = True            # one fused device pass per iteration instead of GEN/MERGE/APPLY ranges
    direction: str = "auto"
    device: int = 0
    partitioning: str = "ids"     # "ids": contiguous ascending-id ranges like partition_graph (A/graph.py:175-212);
                                  # "edges": degree-sorted slots dealt to balance in-edges (the multi-GPU default)
    sizes: list[int] | None = None  # explicit partition sizes (partition_graph's `sizes`)
    capacity: list[float] | None = None  # per-partition capacity factors (balancer.capacity_factors):
                                         # degree-sorted ranges cut in proportion (A/balancer.py:79-98)
    peer_delta: bool = True       # SSSP / CC / LP: changed values go only to the partitions that read
                                  # them, stored by the pack kernel into their arenas (else: to all)

    def __post_init__(self):
        if self.partitions < 1:
            raise ValueError(f"partitions must be >= 1, got {self.partitions}")
        if self.block_size < 1:
            raise ValueError(f"block size must be >= 1, got {self.block_size}")


@dataclass
class RunMetrics:
    model: str
    records: list[StepRecord] = field(default_factory=list)
    converged: bool = False
    iterations: int = 0
    skipped_rounds: int = 0
    exchanged_bytes: int = 0
    split_passes: int = 0  # local-source passes run beside an exchange (option split_overlap)
    init_counts: dict[int, int] = field(default_factory=dict)

    def lines(self) -> list[str]:
        return [r.to_line(self.model) for r in self.records]


def convergence_vote(votes: list) -> bool:
    """Logical AND over per-partition votes; a missing vote is fatal (A/engine.py:131-136)."""
    if any(v is None for v in votes):
        missing = [i for i, v in enumerate(votes) if v is None]
        raise EngineError(f"missing convergence vote from partition(s) {missing}")
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


def setup_local_peers(states) -> list:
    """Same-process partitions for the per-peer delta exchange: every partition's receive
    arena sized from the all-partition send counts, the peers' arenas wired directly.
    Returns the per-partition vote blocks (6 + m float64 each) the pack kernel fills."""
    import torch
    m = len(states)
    try:
        caps = np.asarray([s.exchange_counts()[0] for s in states], dtype=np.uint64)
    except ValueError:  # no per-peer lists (an edgeless graph): the all-to-all round applies
        return None
    for s in states:
        s.delta_arena(caps)
    for s in states:
        s.delta_set_peers(states)
    dev = torch.device("cuda", states[0].graph.ctx.device)
    return [torch.zeros(6 + m, dtype=torch.float64, device=dev) for _ in states]


def exchange_local_peers(states, votes) -> int:
    """Sync round over the per-peer arenas (the in-process analogue of PartitionedRun's
    delta_pack -> vote -> delta_unpack): each partition receives only the changed values its
    CSC reads (A/agent.py:550-582 with a static query set)."""
    from . import _lib as L
    for s in states:  # split rounds (option split_overlap): the next round's local pass first
        s.iterate_local()
    for s, v in zip(states, votes):
        s.delta_pack(v)
    rows = [v.cpu().tolist() for v in votes]
    rec = states[0].buffer(L.BUF_RECORD_SIZE)[1]
    moved = 0
    for j, s in enumerate(states):
        counts = [0 if p == j else int(rows[p][6 + j]) for p in range(len(states))]
        s.delta_unpack(counts)
        moved += sum(counts) * rec
    return moved


def _edges(graph):
    from .graph import EdgeArrays
    if isinstance(graph, EdgeArrays):
        return graph
    if isinstance(graph, tuple) and len(graph) == 2:
        return EdgeArrays.from_edges(list(graph[1]))
    if hasattr(graph, "partitions"):  # the reference's PartitionedGraph
        return EdgeArrays.from_edges([e for p in graph.partitions for e in p.edges])
    raise TypeError("graph must be EdgeArrays, (vertices, edges) or a PartitionedGraph")


class Engine:
    def __init__(self, graph, algorithm, model: str, config: RunConfig):
        model = getattr(model, "value", model)
        if model not in MODELS:
            raise ValueError(f"unknown computation model {model!r}")
        self.edges = _edges(graph)
        self.algorithm = algorithm
        self.model = model
        self.config = config
        self.metrics = RunMetrics(model=model)
        self.states, self.graphs = [], []

    def _setup(self):
        from .device import DeviceContext, DeviceGraph, make_state
        cfg, ea = self.config, self.edges
        algo = self.algorithm.device_name
        self.ctx = DeviceContext(cfg.device)
        w = ea.weight if algo == "sssp" else None
        maxw = int(np.max(w)) if (w is not None and w.size) else 1
        for j in range(cfg.partitions):
            g = DeviceGraph(self.ctx, ea.src, ea.dst, w, part=j, nparts=cfg.partitions, csr=algo != "pagerank",
                            partitioning=cfg.partitioning, sizes=cfg.sizes, capacity=cfg.capacity)
            s = make_state(g, algo, sources=getattr(self.algorithm, "sources", None) if algo == "sssp" else None,
                           max_weight=maxw if algo == "sssp" else None)
            self.graphs.append(g)
            self.states.append(s)
        self.bounds = self.graphs[0].bounds()
        self.metrics.init_counts = {0: self.ctx.init_count}
        # SSSP with more than 4 sources: one device state per 4-lane group, exchanged per group
        lanes = getattr(self.states[0], "states", None)
        self.groups = [[st.states[k] for st in self.states] for k in range(len(lanes))] if lanes else [self.states]
        self.votes = None
        if cfg.partitions > 1 and algo != "pagerank" and cfg.peer_delta and cfg.partitions <= 8:
            votes = [setup_local_peers(grp) for grp in self.groups]
            self.votes = None if any(v is None for v in votes) else votes
        cap = cfg.max_iterations
        self.cap = self.algorithm.default_iteration_cap(self.graphs[0].num_vertices) if cap is None else cap

    def _round(self, s, g) -> dict:
        """One Gen∘Merge∘Apply round of one partition (fused, or the template ops over ranges)."""
        cfg = self.config
        if cfg.fused or s.algo == "lp":  # LP folds a label multiset: no materialised-message form
            s.iterate(cfg.direction)
        else:
            from . import _lib as L
            b = cfg.block_size
            E = int(g.info.owned_edges)
            lo, hi = g.owned
            for e0 in range(0, E, b):
                s.request(L.OP_GEN, e0, min(E, e0 + b))
            for op in (L.OP_MERGE, L.OP_APPLY):
                for v0 in range(lo, hi, b):
                    s.request(op, v0, min(hi, v0 + b))
            s.commit()
        return s.stats()

    def run(self):
        self._setup()
        try:
            self._loop()
            return self._read_attrs(), self.metrics
        finally:
            for s in self.states:
                s.free()
            for g in self.graphs:
                g.free()
            self.ctx.shutdown()

    def _loop(self):
        cfg, m = self.config, len(self.states)
        iteration, apply_rounds = 0, 0
        if self.model == "gas":
            # seed round (A/agent.py:476-486): nothing materialises in the pull design; it still
            # takes the skip vote on the initial frontier and is excluded from the cap
            iteration = 1
            stats = [s.stats() for s in self.states]
            skip = cfg.enable_skip and m > 1 and all(st["remote_active"] == 0 for st in stats)
            self.metrics.skipped_rounds += int(skip)
            self.metrics.records.append(StepRecord(1, 0, sum(st["next_active"] for st in stats), 0, 0, 0.0,
                                                   skip, False))
        while apply_rounds < self.cap:
            iteration += 1
            stats = [self._round(s, g) for s, g in zip(self.states, self.graphs)]
            skip = cfg.enable_skip and m > 1 and all(st["remote_active"] == 0 for st in stats)
            if skip or m == 1:
                moved = 0
            elif self.votes is not None:
                moved = sum(exchange_local_peers(grp, v) for grp, v in zip(self.groups, self.votes))
            else:
                moved = sum(exchange_local(grp, self.bounds) for grp in self.groups)
            self.metrics.exchanged_bytes += moved
            self.metrics.split_passes = sum(getattr(s, "local_passes", 0) for s in self.states)
            converged = convergence_vote([bool(st["voted"]) for st in stats])
            apply_rounds += 1
            if skip and not converged:
                self.metrics.skipped_rounds += 1
            self.metrics.records.append(StepRecord(
                iteration, sum(st["changed"] for st in stats), sum(st["next_active"] for st in stats),
                sum(st["units"] for st in stats), sum(st["remote_active"] for st in stats),
                max(st["max_stat"] for st in stats), skip, converged, moved))
            if converged or apply_rounds >= self.cap:
                self.metrics.converged = converged
                self.metrics.iterations = iteration
                break

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


def run(graph, algorithm, model: str, config: RunConfig) -> tuple[dict[int, object], RunMetrics]:
    """Run one algorithm over m device partitions; returns (attrs, metrics)."""
    return Engine(graph, algorithm, model, config).run()


def dump_attributes(attrs: dict[int, object], algorithm) -> str:
    """Diff-friendly dump: ascending vertex id, one 'id value(s)' per line (A/engine.py:430-433)."""
    lines = [f"{vid} {algorithm.format_attr(attr)}" for vid, attr in sorted(attrs.items())]
    return "\n".join(lines) + ("\n" if lines else "")
