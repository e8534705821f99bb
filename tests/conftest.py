"""Shared fixtures. `gpu` tests need a B200 (sm_100) and the in-tree libgxb200.so;
everything else runs on the CPU (the oracle, golden vectors, host logic, ABI
exports, gloo multi-process paths)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and libgxb200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden_cases():
    with open(os.path.join(GOLDEN, "index.json")) as fh:
        return json.load(fh)


def load_golden(tag):
    """(src, dst, w|None, data dict, meta dict) of a golden fixture; R-MAT edges regenerated."""
    z = np.load(os.path.join(GOLDEN, f"{tag}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    data = {k: z[k] for k in z.files if k != "meta"}
    if "rmat" in meta:
        from paper_2203_13005_b200.rmat import RmatParams, rmat_host
        p = RmatParams(**meta["rmat"])
        src, dst, w = rmat_host(p)
        w = None if w is None else w.astype(np.float64)
    else:
        src, dst = data["src"].astype(np.uint32), data["dst"].astype(np.uint32)
        w = data.get("w")
    return src, dst, w, data, meta


def golden_runs():
    out = []
    for case in golden_cases():
        for key in case["runs"]:
            out.append((case["tag"], key))
    return out


def parse_run_key(key):
    """'<algo>__cap<N|none>' -> (algo, cap)."""
    algo, cap = key.split("__cap")
    return algo, (None if cap == "none" else int(cap))


def assert_attrs_match(algo, got, want, rel=1e-9):
    """SSSP/LP/CC bit-exact; PageRank within `rel` relative per vertex
    (the north star's bar is 1e-5; T/conftest.py:22-30 uses 1e-9)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    if algo == "pagerank":
        err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
        assert float(err.max(initial=0.0)) <= rel, f"max rel err {err.max()}"
    else:
        eq = (got == want)
        assert eq.all(), f"{(~eq).sum()} mismatching entries, first at {np.argwhere(~eq)[:5].tolist()}"


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle
    oracle.lib()
    return oracle
