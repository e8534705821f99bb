"""GPU tests of the package API: run_device (drop-in for run_reference) against the
reference's own golden outputs, the device-only partitioned Engine against the oracle,
attribute staging. The reference's own Engine / Agent / Daemon with the B200 daemon
dropped in is tests/test_dropin_gpu.py."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_attrs_match, golden_cases, load_golden

pytestmark = pytest.mark.gpu


def golden_dict(data, key, ids, algo, out_degree):
    rows = data[key]
    out = {}
    for i, v in enumerate(ids):
        v = int(v)
        if algo == "sssp":
            out[v] = tuple(float(x) for x in rows[i])
        elif algo == "pagerank":
            out[v] = (float(rows[i][0]), out_degree[v])
        else:
            out[v] = int(rows[i][0])
    return out


def attrs_close(got, want, algo, rel=1e-9):
    """T/conftest.py:22-30: exact for SSSP/LP/CC, relative rank tolerance for PageRank."""
    if set(got) != set(want):
        return False
    if algo == "pagerank":
        return all(abs(got[k][0] - want[k][0]) <= rel * max(1.0, abs(want[k][0])) and got[k][1] == want[k][1]
                   for k in want)
    return got == want


def _setup(tag):
    from paper_2203_13005_b200.graph import EdgeArrays
    src, dst, w, data, meta = load_golden(tag)
    ea = EdgeArrays(src, dst, w)
    ids = data["ids"]
    od = {int(v): int(c) for v, c in zip(ids, data["out_degree"])}
    return ea, ids, od, data, meta


@pytest.fixture(scope="module")
def ctx():
    from paper_2203_13005_b200.device import DeviceContext
    c = DeviceContext(0)
    yield c
    c.shutdown()


SMALL = [c["tag"] for c in golden_cases() if not c["tag"].startswith("rmat_s1")]


@pytest.mark.parametrize("tag", SMALL)
def test_run_device_is_run_reference(ctx, tag):
    from paper_2203_13005_b200.algorithms import make_algorithm, run_device
    ea, ids, od, data, meta = _setup(tag)
    for run in meta["runs"]:
        algo = make_algorithm(run["algo"], [int(v) for v in ids], od)
        got = run_device(algo, None, ea, max_iterations=run["cap"], ctx=ctx)
        want = golden_dict(data, run["key"], ids, run["algo"], od)
        assert attrs_close(got, want, run["algo"]), (tag, run["key"])


@pytest.mark.parametrize("partitioning", ["ids", "edges"])
@pytest.mark.parametrize("algo_name", ["sssp", "pagerank", "cc", "lp"])
@pytest.mark.parametrize("m", [2, 3, 4])
def test_partitioned_engine_matches_oracle(oracle_lib, algo_name, m, partitioning):
    from paper_2203_13005_b200.algorithms import make_algorithm
    from paper_2203_13005_b200.engine import RunConfig, run
    from paper_2203_13005_b200.graph import EdgeArrays
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    p = RmatParams(scale=11, seed=40 + m, wmax=63 if algo_name == "sssp" else 0, symmetric=algo_name == "cc")
    src, dst, w = rmat_host(p)
    ea = EdgeArrays(src, dst, None if w is None else w.astype(np.float64))
    ids = ea.vertex_ids()
    algo = make_algorithm(algo_name, [int(v) for v in ids], ea.out_degree())
    cap = 10 if algo_name == "pagerank" else None
    for fused in (False, True):
        cfg = RunConfig(partitions=m, block_size=5000, max_iterations=cap, fused=fused, partitioning=partitioning,
                        enable_skip=True)
        attrs, metrics = run(ea, algo, "bsp", cfg)
        ref = oracle_lib.OracleGraph(src, dst, None if w is None else w.astype(np.float64)).run(
            algo_name, max_iterations=cap)
        got = np.array([algo.row_from_attr(attrs[int(v)]) for v in ids], dtype=np.float64)
        assert_attrs_match(algo_name, got, ref.attrs)
        assert metrics.iterations == ref.iterations


def test_dump_attributes_format(ctx):
    from paper_2203_13005_b200.algorithms import make_algorithm, run_device
    from paper_2203_13005_b200.engine import dump_attributes
    from paper_2203_13005_b200.graph import EdgeArrays
    ea = EdgeArrays.from_edges([(0, 1, 2.0), (1, 2, 3.0)])
    algo = make_algorithm("sssp", [0, 1, 2], None)
    text = dump_attributes(run_device(algo, None, ea, ctx=ctx), algo)
    assert text == "0 0.0 inf inf\n1 2.0 0.0 inf\n2 5.0 3.0 0.0\n"


def test_write_attrs_round_trip(ctx):
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=10, seed=3, wmax=9))
    for algo in ("pagerank", "sssp", "cc"):
        g = DeviceGraph(ctx, src, dst, w if algo == "sssp" else None)
        s = DeviceState(g, algo)
        s.iterate()
        s.stats()
        a = s.read_attrs()
        s2 = DeviceState(g, algo)
        s2.write_attrs(a)
        np.testing.assert_array_equal(s2.read_attrs(), a)
        if algo != "pagerank":
            bad = a.copy()
            bad[0, 0] = 0.5
            with pytest.raises(ValueError):
                s2.write_attrs(bad)


def test_owned_scope_staging(ctx):
    """Owned-scope async staging moves exactly this partition's vertices, ascending ids."""
    import torch
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=11, seed=74, wmax=9))
    for part in range(3):
        for algo in ("pagerank", "sssp", "cc"):
            g = DeviceGraph(ctx, src, dst, w if algo == "sssp" else None, part=part, nparts=3, csr=False)
            s = DeviceState(g, algo)
            s.iterate("pull")
            s.stats()
            full = s.read_attrs()                       # every vertex, ascending ids
            ids = g.ids()
            own = g.owned_ids()
            assert np.all(np.diff(own.astype(np.int64)) > 0)
            lo, hi = g.owned
            pos = np.searchsorted(ids, own)
            st = torch.cuda.current_stream()
            s.attrs_scope(True)
            out = torch.empty(len(own) * s.arity, dtype=torch.float64).pin_memory()
            s.attrs_extract(0, st)
            s.attrs_d2h(out, 0, st)
            st.synchronize()
            np.testing.assert_array_equal(out.numpy().reshape(len(own), s.arity), full[pos])
            # install modified owned values and read them back through the full view
            new = full[pos].copy()
            new[:, 0] = np.where(np.isinf(new[:, 0]), new[:, 0], new[:, 0] + (1 if algo != "pagerank" else 0.5))
            hin = torch.from_numpy(new.reshape(-1).copy()).pin_memory()
            s.attrs_h2d(hin, 1, st)
            s.attrs_install(1, st)
            st.synchronize()
            np.testing.assert_array_equal(s.read_attrs()[pos], new)
            s.attrs_scope(False)
