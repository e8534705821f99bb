"""The CPU oracle (oracle/gx_oracle.c) against the reference's own outputs.

Every golden vector was produced by running the reference (run_reference and
Engine, tests/golden/make_golden.py). The oracle restates run_reference with the
same per-target fold order, so every algorithm — PageRank included — must match
bit for bit. This pins the oracle before any GPU result is compared with it."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import golden_cases, golden_runs, load_golden, parse_run_key


@pytest.mark.parametrize("tag,key", golden_runs())
def test_oracle_matches_reference_run(oracle_lib, tag, key):
    src, dst, w, data, meta = load_golden(tag)
    algo, cap = parse_run_key(key)
    g = oracle_lib.OracleGraph(src, dst, w)
    np.testing.assert_array_equal(g.ids().astype(np.uint64), data["ids"])
    np.testing.assert_array_equal(g.out_degree().astype(np.uint64), data["out_degree"])
    r = g.run(algo, max_iterations=cap)
    np.testing.assert_array_equal(r.attrs, data[key])  # bit-exact, PageRank included


def engine_runs():
    out = []
    for case in golden_cases():
        for key in case["engine"]:
            out.append((case["tag"], key))
    return out


@pytest.mark.parametrize("tag,key", engine_runs())
def test_reference_engine_equals_run_reference(tag, key):
    """The reference's Engine (partitioned, pipelined) agrees with its own oracle; the
    fixture also records the Engine's iteration counts / skip counts used by GPU tests."""
    src, dst, w, data, meta = load_golden(tag)
    algo = key.split("__")[1]
    ref_key = f"{algo}__capnone"
    got, want = data[key], data[ref_key]
    if algo == "pagerank":
        assert np.allclose(got, want, rtol=1e-9, atol=0)
    else:
        np.testing.assert_array_equal(got, want)
    em = [e for e in meta["engine"] if e["key"] == key][0]
    assert em["protocol_conformant"] and em["init_counts"] == [1] and em["copy_counts"] == [0]


def test_rmat_fixture_digests():
    """The shared generator (include/gxb_rmat.h) reproduces the streams the fixtures were built on."""
    seen = 0
    for case in golden_cases():
        src, dst, w, data, meta = load_golden(case["tag"])
        if "rmat" not in meta:
            continue
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(src, dtype=np.uint32).tobytes())
        h.update(np.ascontiguousarray(dst, dtype=np.uint32).tobytes())
        if w is not None:
            h.update(np.ascontiguousarray(w, dtype=np.float64).tobytes())
        assert h.hexdigest() == meta["edge_sha256"], case["tag"]
        seen += 1
    assert seen >= 5


def test_oracle_pagerank_iteration_trace(oracle_lib):
    """PR: every vertex active every round, units == |E| (A/algorithms.py:144-145)."""
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, _ = rmat_host(RmatParams(scale=9, seed=3))
    r = oracle_lib.OracleGraph(src, dst).run("pagerank", max_iterations=5)
    assert r.iterations == 5 and (r.units == len(src)).all()


def test_oracle_threads_do_not_change_results(oracle_lib):
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, w = rmat_host(RmatParams(scale=11, seed=8, wmax=63))
    g = oracle_lib.OracleGraph(src, dst, w.astype(np.float64))
    for algo in ("pagerank", "sssp", "lp", "cc"):
        a = g.run(algo, max_iterations=6, nthreads=1).attrs
        b = g.run(algo, max_iterations=6, nthreads=4).attrs
        np.testing.assert_array_equal(a, b)
