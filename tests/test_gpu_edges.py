"""GPU edge cases against the oracle: degenerate graphs, extreme ids, zero weights, heavy
multi-edges, partitions that own nothing, and the device limits' error behaviour."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_attrs_match

pytestmark = pytest.mark.gpu

ALGOS = ["sssp", "pagerank", "cc", "lp"]


@pytest.fixture(scope="module")
def ctx():
    from paper_2203_13005_b200.device import DeviceContext
    c = DeviceContext(0)
    yield c
    c.shutdown()


def run_both(ctx, oracle_lib, src, dst, w, algo, direction="auto", cap=None):
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState, run_state
    src = np.asarray(src, np.uint32)
    dst = np.asarray(dst, np.uint32)
    wd = None if w is None else np.asarray(w, np.float64)
    g = DeviceGraph(ctx, src, dst, wd if algo == "sssp" else None, csr=algo != "pagerank")
    s = DeviceState(g, algo)
    it, conv, hist = run_state(s, cap if algo != "pagerank" else (cap or 10), direction, keep_history=True)
    ref = oracle_lib.OracleGraph(src, dst, wd).run(algo, max_iterations=cap if algo != "pagerank" else (cap or 10))
    assert it == ref.iterations and conv == ref.converged
    np.testing.assert_array_equal(g.ids().astype(np.uint64), np.unique(np.concatenate([src, dst])).astype(np.uint64))
    assert_attrs_match(algo, s.read_attrs(), ref.attrs)
    if algo != "pagerank":
        assert [h["changed"] for h in hist] == ref.changed.tolist()
    return g, s


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("direction", ["auto", "pull", "push"])
def test_single_self_loop(ctx, oracle_lib, algo, direction):
    if direction == "push" and algo == "pagerank":
        pytest.skip("no push mode for PageRank")
    run_both(ctx, oracle_lib, [7], [7], [3], algo, direction)


@pytest.mark.parametrize("algo", ALGOS)
def test_extreme_ids(ctx, oracle_lib, algo):
    """Ids at both ends of the u32 range (0xFFFFFFFF is the device's reserved sentinel)."""
    big = 0xFFFFFFFE
    src = [0, big, big - 1, 5, big, 0]
    dst = [big, big - 1, 0, big, 5, 5]
    run_both(ctx, oracle_lib, src, dst, [1, 2, 3, 4, 5, 6], algo)


@pytest.mark.parametrize("algo", ["sssp", "cc", "lp"])
def test_heavy_multi_edges(ctx, oracle_lib, algo):
    """Parallel edges count once per edge in LP's multiset (ties to the smallest label)."""
    rng = np.random.default_rng(5)
    src = rng.integers(0, 40, 3000)
    dst = rng.integers(0, 12, 3000)
    w = rng.integers(0, 4, 3000)
    run_both(ctx, oracle_lib, src, dst, w, algo)


def test_zero_weights(ctx, oracle_lib):
    src = np.arange(0, 50)
    dst = np.arange(1, 51)
    run_both(ctx, oracle_lib, src, dst, np.zeros(50), "sssp")


@pytest.mark.parametrize("algo", ALGOS)
def test_hub_in_and_out(ctx, oracle_lib, algo):
    """One destination with ~300 K in-edges (spans hundreds of tiles, LP hub tables and the
    push hot-pair path) and one source with as many out-edges."""
    rng = np.random.default_rng(6)
    n = 300_000
    src = np.concatenate([rng.integers(1, 5000, n), np.zeros(n, np.int64), rng.integers(0, 5000, 20_000)])
    dst = np.concatenate([np.zeros(n, np.int64), rng.integers(1, 5000, n), rng.integers(0, 5000, 20_000)])
    w = rng.integers(1, 63, src.size)
    run_both(ctx, oracle_lib, src, dst, w, algo)


@pytest.mark.parametrize("algo", ALGOS)
def test_more_partitions_than_vertices(oracle_lib, algo):
    """Dealt partitioning of 3 vertices over 4 partitions: one partition owns only padding."""
    from paper_2203_13005_b200.algorithms import make_algorithm
    from paper_2203_13005_b200.engine import RunConfig, run
    from paper_2203_13005_b200.graph import EdgeArrays
    src = np.array([0, 1, 2, 2], np.uint32)
    dst = np.array([1, 2, 0, 1], np.uint32)
    w = np.array([1.0, 2.0, 3.0, 4.0])
    ea = EdgeArrays(src, dst, w)
    ids = ea.vertex_ids()
    alg = make_algorithm(algo, [int(v) for v in ids], ea.out_degree())
    cap = 10 if algo == "pagerank" else None
    attrs, metrics = run(ea, alg, "bsp", RunConfig(partitions=4, block_size=2, max_iterations=cap,
                                                   partitioning="edges", enable_skip=True))
    ref = oracle_lib.OracleGraph(src, dst, w).run(algo, max_iterations=cap)
    got = np.array([alg.row_from_attr(attrs[int(v)]) for v in ids], dtype=np.float64)
    assert_attrs_match(algo, got, ref.attrs)
    assert metrics.iterations == ref.iterations


def test_device_limits_raise(ctx):
    """Inputs the exact u32 device arithmetic cannot represent fail loudly (ValueError)."""
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState
    with pytest.raises(ValueError):  # id 0xFFFFFFFF is the reserved sentinel
        DeviceGraph(ctx, np.array([0xFFFFFFFF], np.uint32), np.array([1], np.uint32))
    with pytest.raises(ValueError):  # max_w * |V| >= 2^32 - 1: sums could saturate
        g = DeviceGraph(ctx, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32),
                        np.array([3.0e9, 1.0]))
        DeviceState(g, "sssp")
    g = DeviceGraph(ctx, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32),
                    np.array([3_000_000_000, 1], np.uint32))  # integer weights: the state checks
    with pytest.raises(ValueError):
        DeviceState(g, "sssp")


@pytest.mark.parametrize("algo", ["pagerank", "cc", "lp"])
def test_empty_graph(ctx, oracle_lib, algo):
    """No edges, no vertices: one round that converges (the oracle's / reference's loop)."""
    run_both(ctx, oracle_lib, [], [], None, algo)


def test_empty_graph_sssp(ctx):
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState, run_state
    g = DeviceGraph(ctx, np.array([], np.uint32), np.array([], np.uint32), None)
    try:
        s = DeviceState(g, "sssp")
    except ValueError:
        return  # no source vertex to start from: refused loudly
    it, conv, _ = run_state(s)
    assert conv and s.read_attrs().shape[0] == 0


# ---- SSSP inputs beyond 4 integral lanes (the reference takes any source list and float
# weights, A/algorithms.py:81-122, A/graph.py:155-162) ----

@pytest.mark.parametrize("nsrc", [5, 9, 13])
@pytest.mark.parametrize("cap", [None, 3])
def test_sssp_many_sources(ctx, oracle_lib, nsrc, cap):
    """More than 4 sources: groups of 4 lanes (SsspLanes) = the oracle's joint run."""
    from paper_2203_13005_b200.algorithms import SsspBellmanFord, run_device
    from paper_2203_13005_b200.graph import EdgeArrays
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=11, seed=90 + nsrc, wmax=40))
    ids = np.union1d(src, dst)
    rng = np.random.default_rng(nsrc)
    sources = [int(x) for x in rng.choice(ids, size=nsrc - 1, replace=False)] + [int(ids.max()) + 7]  # one absent
    algo = SsspBellmanFord(sources)
    attrs, res = run_device(algo, None, EdgeArrays(src, dst, w.astype(np.float64)), max_iterations=cap, ctx=ctx,
                            return_result=True)
    ref = oracle_lib.OracleGraph(src, dst, w.astype(np.float64)).run(
        "sssp", sources=np.array(sources, np.uint32), max_iterations=cap)
    assert res.iterations == ref.iterations and res.converged == ref.converged
    assert_attrs_match("sssp", res.attrs, ref.attrs)
    assert attrs[int(ids[0])] == tuple(float(x) for x in ref.attrs[0])


@pytest.mark.parametrize("denom", [2, 4, 64])
def test_sssp_dyadic_weights(ctx, oracle_lib, denom):
    """Non-integral dyadic weights (2.5, 0.25, ...) run exactly: scaled to u32 by 2^k."""
    from paper_2203_13005_b200.algorithms import SsspBellmanFord, run_device
    from paper_2203_13005_b200.graph import EdgeArrays
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=11, seed=95, wmax=63))
    wf = w.astype(np.float64) / denom
    ids = np.union1d(src, dst)
    algo = SsspBellmanFord([int(x) for x in ids[:4]])
    _, res = run_device(algo, None, EdgeArrays(src, dst, wf), ctx=ctx, return_result=True)
    ref = oracle_lib.OracleGraph(src, dst, wf).run("sssp")
    assert res.iterations == ref.iterations
    assert_attrs_match("sssp", res.attrs, ref.attrs)
    assert np.any(res.attrs != np.floor(res.attrs))  # fractional distances really occur


def test_sssp_non_dyadic_weights_raise(ctx):
    """Weights like 1e-3 have no exact u32 form: refused loudly, never approximated."""
    from paper_2203_13005_b200.device import DeviceGraph
    with pytest.raises(ValueError, match="dyadic"):
        DeviceGraph(ctx, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([1e-3, 1.0]))


@pytest.mark.parametrize("m", [2, 3])
def test_sssp_many_sources_partitioned(oracle_lib, m):
    """Partitioned engine with 6 sources and dyadic weights: per-group sync rounds."""
    from paper_2203_13005_b200.algorithms import SsspBellmanFord
    from paper_2203_13005_b200.engine import RunConfig, run
    from paper_2203_13005_b200.graph import EdgeArrays
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=11, seed=97, wmax=31))
    wf = w.astype(np.float64) / 8
    ids = np.union1d(src, dst)
    sources = [int(x) for x in ids[::max(1, len(ids) // 6)][:6]]
    algo = SsspBellmanFord(sources)
    attrs, met = run(EdgeArrays(src, dst, wf), algo, "bsp", RunConfig(partitions=m, partitioning="edges",
                                                                        enable_skip=True))
    ref = oracle_lib.OracleGraph(src, dst, wf).run("sssp", sources=np.array(sources, np.uint32))
    got = np.array([algo.row_from_attr(attrs[int(v)]) for v in ids])
    assert_attrs_match("sssp", got, ref.attrs)
    assert met.iterations == ref.iterations


def test_sssp_many_sources_split_rounds(oracle_lib):
    """Split rounds (option split_overlap) with lane groups (6 sources, dyadic weights,
    3 partitions, every round a dense pull): each group's states run their local-source
    passes beside the group's exchange; results equal the oracle."""
    from paper_2203_13005_b200 import _lib as L
    from paper_2203_13005_b200.algorithms import SsspBellmanFord
    from paper_2203_13005_b200.engine import RunConfig, run
    from paper_2203_13005_b200.graph import EdgeArrays
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=12, seed=98, wmax=31))
    wf = w.astype(np.float64) / 4
    ids = np.union1d(src, dst)
    sources = [int(x) for x in ids[::max(1, len(ids) // 6)][:6]]
    algo = SsspBellmanFord(sources)
    L.set_option("split_overlap", 1)
    L.set_option("pull_dense_div", 1 << 20)
    try:
        attrs, met = run(EdgeArrays(src, dst, wf), algo, "bsp",
                         RunConfig(partitions=3, enable_skip=True, direction="pull"))
    finally:
        L.set_option("split_overlap", 0)
        L.set_option("pull_dense_div", 4)
    ref = oracle_lib.OracleGraph(src, dst, wf).run("sssp", sources=np.array(sources, np.uint32))
    got = np.array([algo.row_from_attr(attrs[int(v)]) for v in ids])
    assert_attrs_match("sssp", got, ref.attrs)
    assert met.iterations == ref.iterations
    assert met.split_passes > 0
