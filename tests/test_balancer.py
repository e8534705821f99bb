"""Heterogeneous balancing (A/balancer.py): the planners' known answers from the
reference's own tests (T/test_balancer.py), and on the GPU the capacity-weighted
degree-sorted partitions (gxb_graph_build_balanced) against the oracle."""

from __future__ import annotations

import itertools
import random

import os
import sys

import numpy as np
import pytest
from conftest import assert_attrs_match

from paper_2203_13005_b200.balancer import (BalanceProblem, CalibrationError, CapacityProblem, NodeCost,
                                            balance_capacity, balance_data, calibrate, capacity_factors,
                                            makespan, real_valued_makespan)


def _costs(cs):
    return [NodeCost(c) for c in cs]


def _enumerate_optimum(total, costs):
    """Brute-force best makespan over every integer split (T/test_balancer.py's helper)."""
    best = float("inf")
    for cut in itertools.product(range(total + 1), repeat=len(costs) - 1):
        if sum(cut) <= total:
            best = min(best, makespan(list(cut) + [total - sum(cut)], costs))
    return best


def test_makespan_known_answers():
    assert makespan([1, 1], [1.0, 1.0]) == 1.0
    assert makespan([3, 1], [1.0, 3.0]) == 3.0
    with pytest.raises(ValueError):
        makespan([1, 2], [1.0])


def test_balance_data_known_answers():
    assert balance_data(BalanceProblem(100, _costs([1.0, 1.0]))) == [50, 50]
    sizes = balance_data(BalanceProblem(4, _costs([1.0, 3.0])))
    assert sizes == [3, 1] and makespan(sizes, [1.0, 3.0]) == _enumerate_optimum(4, [1.0, 3.0]) == 3.0
    sizes = balance_data(BalanceProblem(7, _costs([1.0, 2.0, 4.0])))
    assert sizes == [4, 2, 1]


def test_balance_data_sum_exact_and_near_optimal():
    rng = random.Random(5)
    for _ in range(200):
        k = rng.randint(1, 4)
        costs = [rng.uniform(0.1, 5.0) for _ in range(k)]
        total = rng.randint(1, 12 if k > 2 else 40)
        sizes = balance_data(BalanceProblem(total, _costs(costs)))
        assert sum(sizes) == total and min(sizes) >= 0
        assert makespan(sizes, costs) <= _enumerate_optimum(total, costs) + max(costs)
        want = total / sum(1.0 / c for c in costs)
        assert real_valued_makespan(BalanceProblem(total, _costs(costs))) == pytest.approx(want, rel=1e-12)


def test_balance_data_ties_go_to_lower_index():
    assert balance_data(BalanceProblem(5, _costs([1.0, 1.0]))) == [3, 2]
    assert balance_data(BalanceProblem(4, _costs([1.0, 1.0, 1.0]))) == [2, 1, 1]


def test_balance_capacity_known_answers():
    assert balance_capacity(CapacityProblem([10, 5], max_factor=1.0)) == [1.0, 0.5]
    assert balance_capacity(CapacityProblem([8, 4], max_factor=4.0)) == [4.0, 2.0]
    assert balance_capacity(CapacityProblem([6, 6, 6], max_factor=2.5)) == [2.5, 2.5, 2.5]
    with pytest.raises(ValueError):
        balance_capacity(CapacityProblem([0, 0], max_factor=1.0))
    with pytest.raises(ValueError):
        CapacityProblem([1, 1], max_factor=0.5, current_costs=_costs([1.0, 1.0]))


def test_preconditions():
    with pytest.raises(ValueError):
        NodeCost(0.0)
    with pytest.raises(ValueError):
        BalanceProblem(0, _costs([1.0]))
    with pytest.raises(ValueError):
        BalanceProblem(5, [])
    with pytest.raises(ValueError):
        capacity_factors([1.0, -2.0])
    assert capacity_factors([1.0, 4.0]) == [1.0, 0.25]


def test_calibrate():
    c, t_call = 0.25, 3.0
    obs = [(u, b, c * u + t_call * b) for u, b in [(10, 1), (20, 2), (40, 1), (80, 4)]]
    r = calibrate(obs)
    assert r.unit_cost == pytest.approx(c, rel=1e-9) and r.call_cost == pytest.approx(t_call, rel=1e-9)
    r = calibrate([(u, 2, 2.0 * u + 1.0) for u in (3, 7, 11)])
    assert r.unit_cost == pytest.approx(2.0, rel=1e-9) and r.call_cost is None
    with pytest.raises(CalibrationError):
        calibrate([(5, 1, 1.0)])
    with pytest.raises(CalibrationError):
        calibrate([(5, 1, 1.0), (5, 2, 2.0)])


def test_matches_reference_planners_when_present():
    """Cross-check against the reference's own module (this container only; skipped
    where /root/reference is absent, e.g. on the GPU box)."""
    src_dir = "/root/reference/pkg/src"
    if not os.path.isdir(src_dir):
        pytest.skip("reference not present")
    if src_dir not in sys.path:
        sys.path.append(src_dir)
    sys.dont_write_bytecode = True
    ref = pytest.importorskip("accelgraph.balancer")
    rng = random.Random(11)
    for _ in range(300):
        k = rng.randint(1, 6)
        costs = [rng.uniform(0.05, 9.0) for _ in range(k)]
        total = rng.randint(1, 10_000)
        got = balance_data(BalanceProblem(total, _costs(costs)))
        want = ref.balance_data(ref.BalanceProblem(total, [ref.NodeCost(c) for c in costs]))
        assert got == want
        sizes = [rng.randint(0, 100) for _ in range(k)]
        if any(sizes):
            assert balance_capacity(CapacityProblem(sizes, 3.0)) == ref.balance_capacity(ref.CapacityProblem(sizes, 3.0))


@pytest.mark.gpu
@pytest.mark.parametrize("algo_name", ["sssp", "pagerank", "cc", "lp"])
@pytest.mark.parametrize("capacity", [[3.0, 1.0], [1.0, 2.0, 4.0]])
def test_capacity_partitions_match_oracle(oracle_lib, algo_name, capacity):
    from paper_2203_13005_b200.algorithms import make_algorithm
    from paper_2203_13005_b200.engine import RunConfig, run
    from paper_2203_13005_b200.graph import EdgeArrays
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    p = RmatParams(scale=11, seed=71, wmax=63 if algo_name == "sssp" else 0, symmetric=algo_name == "cc")
    src, dst, w = rmat_host(p)
    ea = EdgeArrays(src, dst, None if w is None else w.astype(np.float64))
    ids = ea.vertex_ids()
    algo = make_algorithm(algo_name, [int(v) for v in ids], ea.out_degree())
    cap = 10 if algo_name == "pagerank" else None
    cfg = RunConfig(partitions=len(capacity), block_size=5000, max_iterations=cap, fused=True,
                    partitioning="ranges", capacity=capacity, enable_skip=True)
    attrs, metrics = run(ea, algo, "bsp", cfg)
    ref = oracle_lib.OracleGraph(src, dst, None if w is None else w.astype(np.float64)).run(
        algo_name, max_iterations=cap)
    got = np.array([algo.row_from_attr(attrs[int(v)]) for v in ids], dtype=np.float64)
    assert_attrs_match(algo_name, got, ref.attrs)
    assert metrics.iterations == ref.iterations


@pytest.mark.gpu
def test_capacity_cuts_cost_in_proportion():
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, _ = rmat_host(RmatParams(scale=14, seed=3))
    ctx = DeviceContext(0)
    try:
        capacity = [4.0, 1.0, 2.0]
        graphs = [DeviceGraph(ctx, src, dst, None, part=j, nparts=3, csr=False, capacity=capacity)
                  for j in range(3)]
        cost = np.array([12 * g.info.owned_edges + 64 * (g.info.owned_hi - g.info.owned_lo) for g in graphs],
                        dtype=np.float64)
        share = cost / cost.sum()
        want = np.array(capacity) / sum(capacity)
        assert np.abs(share - want).max() < 0.02
        # same bounds on every partition; partitions tile the slots
        b = [tuple(g.bounds()) for g in graphs]
        assert len(set(b)) == 1 and b[0][0] == 0 and b[0][-1] == graphs[0].info.num_slots
        with pytest.raises(Exception):
            DeviceGraph(ctx, src, dst, None, part=0, nparts=2, csr=False, capacity=[1.0, 0.0])
        with pytest.raises(ValueError):
            DeviceGraph(ctx, src, dst, None, part=0, nparts=2, csr=False, capacity=[1.0, 1.0], sizes=[1, 1])
        for g in graphs:
            g.free()
    finally:
        ctx.shutdown()



@pytest.mark.gpu
def test_observe_then_calibrate_gives_device_unit_cost():
    """Measured SSSP iterations (frontier sizes vary) identify a positive unit cost."""
    from paper_2203_13005_b200.balancer import observe
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=16, seed=9, wmax=63))
    ctx = DeviceContext(0)
    try:
        g = DeviceGraph(ctx, src, dst, w, csr=True)
        s = DeviceState(g, "sssp", max_weight=63)
        obs = observe(s, iterations=6)
        assert len(obs) == 6 and all(t > 0 for _, _, t in obs)
        assert len({u for u, _, _ in obs}) >= 2
        r = calibrate(obs)
        assert r.call_cost is None and np.isfinite(r.unit_cost)
        s.free()
        g.free()
    finally:
        ctx.shutdown()
