"""Installing the B200 path into an unmodified reference process (`accelgraph`).

The reference's own injection seams (verified there without
editing the reference) are module attributes: `accelgraph.engine.run` /
`accelgraph.engine.Agent` (A/engine.py:205, 422-427), `accelgraph.agent.daemon_init`
(A/agent.py:186) and `accelgraph.daemon.execute_request` (A/daemon.py:191). Because
the reference's agent builds Python triplet blocks before any daemon sees them,
the drop-in replaces the engine entry point: `install(accelgraph)` rebinds
`accelgraph.engine.run` (and `accelgraph.cli`'s import of it) to a wrapper that
converts the reference's `PartitionedGraph` / `Algorithm` objects and runs the
device Engine, returning the reference's `(attrs, RunMetrics)` shape.
"""

from __future__ import annotations

from . import algorithms as A
from .engine import RunConfig, run as device_run


def to_device_algorithm(ref_algo) -> A.Algorithm:
    """A reference Algorithm instance (A/algorithms.py:81-205, or a CC plug-in) -> descriptor."""
    name = getattr(ref_algo, "name", None)
    if name == "sssp":
        return A.SsspBellmanFord(list(ref_algo.sources))
    if name == "pagerank":
        return A.PageRank(dict(ref_algo.out_degree))
    if name == "lp":
        return A.LabelPropagation()
    if name == "cc":
        return A.ConnectedComponents()
    raise ValueError(f"algorithm {name!r} has no device kernels")


def to_device_config(ref_cfg) -> RunConfig:
    """Copy the reference RunConfig fields (A/engine.py:45-60); partition sizes are kept."""
    keys = ["partitions", "daemons_per_node", "enable_cache", "cache_capacity", "cache_decay", "cache_boost",
            "enable_skip", "io_cost", "seed", "max_iterations", "barrier_timeout"]
    cfg = RunConfig(**{k: getattr(ref_cfg, k) for k in keys if hasattr(ref_cfg, k)})
    bs = getattr(ref_cfg, "block_size", None)
    if isinstance(bs, int):
        cfg.block_size = bs
    return cfg


def run_partitioned(graph, algorithm, model, config):
    """Signature-compatible replacement of accelgraph.engine.run (A/engine.py:422-427)."""
    cfg = to_device_config(config)
    if hasattr(graph, "partitions"):
        cfg.partitions = len(graph.partitions)
        cfg.sizes = [len(p.vertices) for p in graph.partitions]  # the reference's own partition sizes
    model = getattr(model, "value", model)
    return device_run(graph, to_device_algorithm(algorithm), model, cfg)


def install(accelgraph) -> None:
    """Rebind the reference's engine entry point (and the CLI's import of it) to the B200 path."""
    import importlib
    importlib.import_module(accelgraph.__name__ + ".engine").run = run_partitioned
    importlib.import_module(accelgraph.__name__ + ".cli").run = run_partitioned
