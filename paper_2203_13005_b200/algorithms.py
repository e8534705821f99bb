"""Algorithm template of the reference (`A/algorithms.py`), as device descriptors.

Each class names the same constructor arguments, constants, iteration caps,
vote rule and attribute format as the reference's `SsspBellmanFord`
(A/algorithms.py:81-122), `PageRank` (125-171) and `LabelPropagation`
(174-205), plus the CC plug-in. The per-element
`gen / merge_payloads / apply_one` bodies are not executed in Python: they are
the kernels of libgxb200 (`csrc/gxb_algo.cu` SsspOps / PrOps / CcOps,
`csrc/gxb_lp.cu`). `run_device` is the drop-in for `run_reference`
(A/algorithms.py:298-342): same inputs, same output dict.
"""

from __future__ import annotations

import math
from typing import Iterable

import numpy as np

INF = math.inf


class Algorithm:
    """Base descriptor; `device_name` selects the kernel family."""

    name = "abstract"
    device_name = ""
    applies_to_all = False
    merge_is_commutative = True  # merge must be associative and commutative (A/algorithms.py:9-10)

    def initial_attr(self, vid: int) -> object:
        raise NotImplementedError

    def initially_active(self, vid: int) -> bool:
        raise NotImplementedError

    def default_iteration_cap(self, num_vertices: int) -> int:
        raise NotImplementedError

    def vote(self, max_stat: float, next_active) -> bool:
        """Local convergence vote after an apply round (A/algorithms.py:70-72)."""
        return not next_active

    def format_attr(self, attr: object) -> str:
        raise NotImplementedError

    def attr_from_row(self, vid: int, row: np.ndarray) -> object:
        """Device row (float64) -> the reference's attribute object."""
        raise NotImplementedError

    def row_from_attr(self, attr: object) -> list[float]:
        raise NotImplementedError


class SsspBellmanFord(Algorithm):
    """Multi-source Bellman-Ford; one distance lane per source (A/algorithms.py:81-122).

    Device distances are exact 32-bit integers: weights must be integral or dyadic
    rationals (scaled to integers exactly, device.validate_weights) with
    max_w * |V| < 2^32 - 1 (checked); any number of sources (groups of 4 lanes).
    """

    name = "sssp"
    device_name = "sssp"

    def __init__(self, sources: list[int]):
        if not sources:
            raise ValueError("sssp needs at least one source vertex")
        self.sources = list(sources)
        self.arity = len(sources)

    def initial_attr(self, vid):
        return tuple(0.0 if vid == s else INF for s in self.sources)

    def initially_active(self, vid):
        return vid in self.sources

    def default_iteration_cap(self, num_vertices):
        return num_vertices + 1

    def format_attr(self, attr):
        return " ".join("inf" if math.isinf(d) else repr(d) for d in attr)

    def attr_from_row(self, vid, row):
        return tuple(float(x) for x in row[: self.arity])

    def row_from_attr(self, attr):
        return [float(x) for x in attr]


class PageRank(Algorithm):
    """Damped PageRank; attribute (rank, out_degree); dangling mass stays put (A/algorithms.py:125-171)."""

    name = "pagerank"
    device_name = "pagerank"
    applies_to_all = True
    damping = 0.85
    base = 0.15  # the literal 0.15, not 1 - 0.85 (Appendix A)
    tolerance = 1e-9

    def __init__(self, out_degree: dict[int, int]):
        self.out_degree = out_degree

    def initial_attr(self, vid):
        return (1.0, self.out_degree[vid])

    def initially_active(self, vid):
        return True

    def vote(self, max_stat, next_active):
        return max_stat < self.tolerance

    def default_iteration_cap(self, num_vertices):
        return 100

    def format_attr(self, attr):
        return repr(attr[0])

    def attr_from_row(self, vid, row):
        return (float(row[0]), self.out_degree[vid])

    def row_from_attr(self, attr):
        return [float(attr[0])]


class LabelPropagation(Algorithm):
    """Majority label of active in-neighbours, ties to the smallest label (A/algorithms.py:174-205)."""

    name = "lp"
    device_name = "lp"

    def initial_attr(self, vid):
        return vid

    def initially_active(self, vid):
        return True

    def default_iteration_cap(self, num_vertices):
        return 15

    def format_attr(self, attr):
        return str(attr)

    def attr_from_row(self, vid, row):
        return int(row[0])

    def row_from_attr(self, attr):
        return [float(attr)]


class ConnectedComponents(Algorithm):
    """Min-label propagation (build-defined plug-in)."""

    name = "cc"
    device_name = "cc"

    def initial_attr(self, vid):
        return vid

    def initially_active(self, vid):
        return True

    def default_iteration_cap(self, num_vertices):
        return num_vertices + 1

    def format_attr(self, attr):
        return str(attr)

    def attr_from_row(self, vid, row):
        return int(row[0])

    def row_from_attr(self, attr):
        return [float(attr)]


def make_algorithm(
    name: str,
    vertex_ids: Iterable[int],
    out_degree: dict[int, int] | None = None,
    sources: list[int] | None = None,
) -> Algorithm:
    """Instantiate an algorithm for a concrete graph (A/algorithms.py:208-229)."""
    if name == "sssp":
        if sources is None:
            sources = sorted(vertex_ids)[:4]
        return SsspBellmanFord(sources)
    if name == "pagerank":
        if out_degree is None:
            raise ValueError("pagerank needs the global out-degree table")
        return PageRank(out_degree)
    if name == "lp":
        return LabelPropagation()
    if name == "cc":
        return ConnectedComponents()
    raise ValueError(f"unknown algorithm {name!r}")


def _edge_arrays(vertices, edges):
    from .graph import EdgeArrays
    ea = edges if isinstance(edges, EdgeArrays) else EdgeArrays.from_edges(list(edges))
    if vertices is not None:
        vs = np.fromiter((int(v) for v in vertices), dtype=np.int64)
        present = ea.vertex_ids()
        if vs.size and not np.array_equal(np.unique(vs), present.astype(np.int64)):
            # the reference's vertex set is exactly the ids present in edges (A/graph.py:163-164)
            raise ValueError("vertex set must equal the ids present in the edge list on the device")
    return ea


def run_device(algorithm: Algorithm, vertices, edges, max_iterations: int | None = None,
               ctx=None, direction: str = "auto", return_result: bool = False):
    """Drop-in for run_reference (A/algorithms.py:298-342) on one B200.

    Returns {vid: attr} with the reference's attribute objects. With
    return_result=True also returns the DeviceRun (iterations, convergence,
    per-iteration statistics)."""
    from .device import DeviceContext, DeviceGraph, DeviceRun, make_state, run_state

    ea = _edge_arrays(vertices, edges)
    own = ctx is None
    if own:
        ctx = DeviceContext(0)
    try:
        algo = algorithm.device_name
        w = ea.weight if algo == "sssp" else None
        g = DeviceGraph(ctx, ea.src, ea.dst, w, csr=algo in ("sssp", "cc", "lp"))
        sources = getattr(algorithm, "sources", None) if algo == "sssp" else None
        maxw = int(np.max(w)) if (w is not None and w.size) else 1
        s = make_state(g, algo, sources=sources, max_weight=maxw if algo == "sssp" else None)
        it, conv, hist = run_state(s, max_iterations, direction, keep_history=return_result)
        rows = s.read_attrs()
        ids = g.ids()
        attrs = {int(v): algorithm.attr_from_row(int(v), rows[i]) for i, v in enumerate(ids)}
        if return_result:
            return attrs, DeviceRun(ids, rows, it, conv, hist)
        return attrs
    finally:
        if own:
            ctx.shutdown()
