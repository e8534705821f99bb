"""CPU-only tests of the host layer: generator, loader, algorithm descriptors, the
drop-in into the reference's own Engine / Agent / Daemon / SharedRegion (seams,
request protocol and error surfacing over a recording fake device state), and the
C-ABI surface of libgxb200.so (symbols only; no compute without a GPU)."""

from __future__ import annotations

import ctypes
import json
import os
import re
import threading

import numpy as np
import pytest

from conftest import GOLDEN, REPO

from paper_2203_13005_b200.algorithms import (ConnectedComponents, LabelPropagation, PageRank,
                                              SsspBellmanFord, make_algorithm)
from paper_2203_13005_b200.graph import EdgeArrays, GraphParseError, read_edge_text
from paper_2203_13005_b200.rmat import RmatParams, rmat_host


# ---------------------------------------------------------------- generator
@pytest.mark.parametrize("kw", [dict(scale=7), dict(scale=9, wmax=63, seed=4),
                                dict(scale=10, symmetric=True, seed=2),
                                dict(scale=8, a=0.65, b=0.15, c=0.15, scramble=False)])
def test_rmat_host_matches_c_generator(oracle_lib, kw):
    p = RmatParams(**kw)
    s, d, w = rmat_host(p)
    s2, d2, w2 = oracle_lib.rmat(p.scale, p.edge_factor, p.seed, p.a, p.b, p.c, p.wmax, p.scramble, p.symmetric)
    np.testing.assert_array_equal(s, s2)
    np.testing.assert_array_equal(d, d2)
    assert (w is None and w2 is None) or np.array_equal(w, w2)


def test_rmat_properties():
    p = RmatParams(scale=12, seed=9, wmax=63)
    s, d, w = rmat_host(p)
    assert s.size == 16 << 12 and s.max() < 4096 and d.max() < 4096
    assert w.min() >= 1 and w.max() <= 63
    with pytest.raises(ValueError):
        RmatParams(scale=0)
    with pytest.raises(ValueError):
        RmatParams(scale=10, a=0.6, b=0.3, c=0.2)


# ---------------------------------------------------------------- loader
def test_load_edge_list_matches_reference(tmp_path):
    with open(os.path.join(GOLDEN, "edge_lists.json")) as fh:
        cases = json.load(fh)
    for name, case in cases.items():
        p = tmp_path / f"{name}.txt"
        p.write_bytes(case["text"].encode("ascii"))
        if case["ok"]:
            ea = read_edge_text(p)
            assert ea.vertex_ids().tolist() == case["vertices"], name
            w = ea.weight.tolist() if ea.weight is not None else [1.0] * len(ea)
            assert [[int(a), int(b), x] for a, b, x in zip(ea.src, ea.dst, w)] == case["edges"], name
        else:
            with pytest.raises(GraphParseError) as exc:
                read_edge_text(p)
            assert exc.value.lineno == case["lineno"], name
            assert str(exc.value) == case["message"], name


def test_binary_edge_format_round_trip(tmp_path):
    """Binary ingest (GXEDGE01) == the reference text loader on every golden edge list."""
    from paper_2203_13005_b200.graph import edge_list_to_binary, read_edge_binary, write_edge_binary
    with open(os.path.join(GOLDEN, "edge_lists.json")) as fh:
        cases = json.load(fh)
    for name, case in cases.items():
        if not case["ok"]:
            continue
        t = tmp_path / f"{name}.txt"
        t.write_bytes(case["text"].encode("ascii"))
        b = tmp_path / f"{name}.gxe"
        n = edge_list_to_binary(t, b)
        ea = read_edge_binary(b)
        assert n == len(ea) == len(case["edges"])
        assert [[int(s), int(d)] for s, d in zip(ea.src, ea.dst)] == [[e[0], e[1]] for e in case["edges"]]
        ws = [e[2] for e in case["edges"]]
        if ea.weight is None:
            assert all(w == 1.0 for w in ws)
        else:
            assert ea.weight.tolist() == ws
    rng = np.random.default_rng(1)
    big = EdgeArrays(rng.integers(0, 1 << 31, 100_000), rng.integers(0, 1 << 31, 100_000),
                     rng.integers(1, 64, 100_000).astype(np.float64))
    write_edge_binary(tmp_path / "big.gxe", big)
    back = read_edge_binary(tmp_path / "big.gxe")
    assert np.array_equal(back.src, big.src) and np.array_equal(back.dst, big.dst)
    assert np.array_equal(back.weight, big.weight)
    (tmp_path / "bad.gxe").write_bytes(b"GXEDGE01" + b"\0" * 30)
    with pytest.raises(GraphParseError):
        read_edge_binary(tmp_path / "bad.gxe")


def test_edge_arrays():
    ea = EdgeArrays.from_edges([(5, 7), (7, 5, 2.0), (5, 5)])
    assert ea.vertex_ids().tolist() == [5, 7]
    assert ea.out_degree() == {5: 2, 7: 1}
    assert ea.weight is not None and ea.weight.tolist() == [1.0, 2.0, 1.0]


# ---------------------------------------------------------------- algorithms
def test_make_algorithm_semantics():
    a = make_algorithm("sssp", {5, 9, 2, 14, 30}, None)
    assert isinstance(a, SsspBellmanFord) and a.sources == [2, 5, 9, 14]
    assert make_algorithm("sssp", {3, 1}, None).sources == [1, 3]
    with pytest.raises(ValueError, match="pagerank needs the global out-degree table"):
        make_algorithm("pagerank", {1}, None)
    with pytest.raises(ValueError, match="unknown algorithm"):
        make_algorithm("bfs", {1}, {})
    with pytest.raises(ValueError, match="at least one source"):
        SsspBellmanFord([])
    pr = make_algorithm("pagerank", {0, 1}, {0: 1, 1: 0})
    assert isinstance(pr, PageRank) and pr.base == 0.15 and pr.damping == 0.85
    assert pr.initial_attr(0) == (1.0, 1) and pr.default_iteration_cap(5) == 100
    assert pr.vote(1e-10, set()) and not pr.vote(1e-8, set())
    assert isinstance(make_algorithm("lp", {1}), LabelPropagation)
    assert isinstance(make_algorithm("cc", {1}), ConnectedComponents)
    s = SsspBellmanFord([0, 3])
    assert s.initial_attr(3) == (float("inf"), 0.0) and s.format_attr((1.0, float("inf"))) == "1.0 inf"


# ---------------------------------------------------------------- drop-in (reference seams)
dropin = pytest.importorskip("paper_2203_13005_b200.dropin", reason="reference package not importable")


class FakeDeviceState:
    """Records the device calls the drop-in makes (no GPU)."""

    def __init__(self, fail_on=None):
        self.calls = []
        self.fail_on = fail_on
        self.commits = 0

    def request(self, op, lo, hi):
        if self.fail_on is not None and op == self.fail_on:
            raise ValueError("apply targets vertex 99 not owned by this node")
        self.calls.append((op, lo, hi))

    def commit(self):
        self.commits += 1

    def iterate(self, direction="auto"):
        self.calls.append(("fused", direction))

    def stats(self):
        return {"remote_active": 0, "voted": 1, "changed": 0, "next_active": 0, "next_units": 5}

    def free(self):
        pass


def test_dropin_seams_install_and_restore():
    import accelgraph.agent as A
    import accelgraph.daemon as D
    import accelgraph.engine as E
    orig = (A.daemon_init, D.execute_request, E.Agent)
    with dropin.installed(fused=False, direction="pull"):
        assert (A.daemon_init, D.execute_request, E.Agent) == \
            (dropin.gpu_daemon_init, dropin.execute_request, dropin.GpuAgent)
        assert dropin.CONFIG.fused is False and dropin.CONFIG.direction == "pull"
        with dropin.installed():          # nested: stays installed on exit
            pass
        assert dropin.installed_now()
    assert (A.daemon_init, D.execute_request, E.Agent) == orig
    assert dropin.CONFIG.fused is True
    with pytest.raises(ValueError):
        dropin.install(direction="sideways")
    assert not dropin.installed_now()


def test_execute_request_runs_device_items_only():
    from accelgraph.channel import OpKind, WorkItem
    from accelgraph.daemon import AcceleratorProfile
    st = FakeDeviceState()
    agent = type("A", (), {})()
    agent.device_state, agent._device_lock, agent.direction = st, threading.Lock(), "push"
    prof = AcceleratorProfile(4, 2.0, 3.0)
    item = WorkItem(OpKind.MERGE, 0, dropin.DeviceRange(agent, OpKind.MERGE, 10, 18), 8)
    assert dropin.execute_request(None, prof, item) == 3.0 + 2.0 * 8
    assert st.calls == [(1, 10, 18)] and item.result_units == 8 and item.result is None
    item = WorkItem(OpKind.GEN, 0, dropin.FusedRound(agent), 5)
    dropin.execute_request(None, prof, item)
    assert st.calls[-1] == ("fused", "push")
    with pytest.raises(TypeError, match="device work items only"):
        dropin.execute_request(None, prof, WorkItem(OpKind.GEN, 0, ("triplets",), 1))
    with pytest.raises(ValueError, match="does not match"):
        dropin.execute_request(None, prof, WorkItem(OpKind.GEN, 0, dropin.DeviceRange(agent, OpKind.APPLY, 0, 1), 1))


def test_gpu_daemon_fails_loudly_without_a_device():
    import torch
    from accelgraph.channel import SharedRegion
    from accelgraph.daemon import AcceleratorProfile
    if torch.cuda.is_available():
        pytest.skip("needs a host without a GPU")
    regions = {"r0": SharedRegion("r0", 8)}
    with pytest.raises(KeyError):
        dropin.GpuDaemon(AcceleratorProfile(4), None, "nope", regions)
    with pytest.raises(Exception, match="(?i)cuda|device|sm_100"):
        dropin.gpu_daemon_init(AcceleratorProfile(4), None, "r0", regions)


def _fake_device(monkeypatch, fail_on=None):
    """GpuDaemon without gxb_init and GpuAgent over a recording fake device state."""
    states = []

    def init(self):
        return super(dropin.GpuDaemon, self).initialize()

    def build(self):
        st = FakeDeviceState(fail_on)
        states.append(st)
        self.device_state = st
        lo = 100 * self.node_id
        self.device_graph = type("G", (), {"owned": (lo, lo + 40), "free": lambda _s: None,
                                           "info": type("I", (), {"owned_edges": 100, "owned_out_edges": 7})()})()
        self._needed = frozenset()

    monkeypatch.setattr(dropin.GpuDaemon, "initialize", init)
    monkeypatch.setattr(dropin.GpuAgent, "_build_device", build)
    monkeypatch.setattr(dropin.GpuAgent, "serve_uploads", lambda self, gqq: ({}, {}))
    monkeypatch.setattr(dropin.GpuAgent, "flush_all", lambda self: {})
    return states


@pytest.mark.parametrize("fused", [False, True])
def test_reference_engine_drives_gpu_agents(monkeypatch, fused):
    """The reference's own Engine / Agent.request / _drive / SharedRegion / Daemon._loop run
    device range items (round-robin over two daemons per node): every GEN edge range and
    MERGE / APPLY slot range covered once, conformant traces, no content copies."""
    from accelgraph.channel import trace_conforms
    from accelgraph.engine import RunConfig, run
    from accelgraph.graph import Edge, even_sizes, partition_graph
    states = _fake_device(monkeypatch)
    edges = [Edge(i, (i + 1) % 6, 1.0) for i in range(6)]
    graph = partition_graph(set(range(6)), edges, even_sizes(6, 2))
    from accelgraph.algorithms import make_algorithm
    algo = make_algorithm("lp" if fused else "sssp", set(range(6)), graph.out_degree)
    with dropin.installed(fused=fused):
        attrs, metrics = run(graph, algo, "bsp", RunConfig(partitions=2, daemons_per_node=2, block_size=16))
    assert metrics.iterations == 1 and metrics.converged
    assert metrics.protocol_conformant() and all(trace_conforms(t) for t in metrics.traces.values())
    assert set(metrics.init_counts.values()) == {1} and set(metrics.copy_counts.values()) == {0}
    for j, st in enumerate(states):
        if fused:
            assert st.calls == [("fused", "auto")]
            continue
        gens = sorted(c[1:] for c in st.calls if c[0] == 0)
        assert gens[0] == (0, 16) and gens[-1] == (96, 100) and len(gens) == 7
        for op in (1, 2):
            rs = sorted(c[1:] for c in st.calls if c[0] == op)
            assert rs[0][0] == 100 * j and rs[-1][1] == 100 * j + 40
            assert sum(h - lo for lo, h in rs) == 40
        assert st.commits == 1


def test_device_error_surfaces_through_the_reference_region(monkeypatch):
    from accelgraph.engine import EngineError, RunConfig, run
    from accelgraph.graph import Edge, partition_graph
    from accelgraph.algorithms import make_algorithm
    _fake_device(monkeypatch, fail_on=2)
    edges = [Edge(0, 1, 1.0), Edge(1, 0, 1.0)]
    graph = partition_graph({0, 1}, edges, [1, 1])
    algo = make_algorithm("sssp", {0, 1}, graph.out_degree)
    with dropin.installed(fused=False), pytest.raises(EngineError, match="not owned"):
        run(graph, algo, "bsp", RunConfig(partitions=2, block_size=64, barrier_timeout=10.0))


# ---------------------------------------------------------------- C ABI surface
def test_abi_exports_every_declared_symbol():
    """libgxb200.so loads on a CPU-only host and exports each function of include/gxb.h."""
    from paper_2203_13005_b200 import _lib as L
    with open(os.path.join(REPO, "include", "gxb.h")) as fh:
        text = fh.read()
    names = sorted(set(re.findall(r"^\s*(?:const\s+char\*|int|void)\s+(gxb_\w+)\s*\(", text, re.M)))
    assert len(names) >= 25
    lib = ctypes.CDLL(L.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert L.lib().gxb_version().startswith(b"gxb200")
    # no GPU here: gxb_init reports an error instead of crashing
    import torch
    if not torch.cuda.is_available():
        h = ctypes.c_void_p()
        assert L.lib().gxb_init(0, ctypes.byref(h)) != 0
        assert L.lib().gxb_last_error()


def test_options_roundtrip():
    from paper_2203_13005_b200 import _lib as L
    old = L.get_option("push_alpha")
    L.set_option("push_alpha", 13)
    assert L.get_option("push_alpha") == 13
    L.set_option("push_alpha", old)
    with pytest.raises(ValueError):
        L.set_option("no_such_knob", 1)
    with pytest.raises(ValueError):
        L.set_option("tile_minblocks", 3)
    # split rounds: off by default (measured slower), 0/1 only; reserve 0..140 SMs
    assert L.get_option("split_overlap") == 0
    assert L.get_option("push_alpha") == 10
    for name, bad in (("split_overlap", 2), ("split_reserve_sms", 141), ("split_reserve_sms", -1)):
        with pytest.raises(ValueError):
            L.set_option(name, bad)
    old = L.get_option("split_reserve_sms")
    L.set_option("split_reserve_sms", 32)
    assert L.get_option("split_reserve_sms") == 32
    L.set_option("split_reserve_sms", old)


# ---------------------------------------------------------------- device weight encoding
def test_validate_weights_dyadic_scaling():
    """Integral weights keep shift 0; dyadic rationals scale exactly by the smallest 2^k;
    anything inexact or out of range raises (device.validate_weights)."""
    from paper_2203_13005_b200.device import validate_weights
    w, k = validate_weights(np.array([1.0, 2.0, 63.0]))
    assert k == 0 and w.dtype == np.uint32 and w.tolist() == [1, 2, 63]
    w, k = validate_weights(np.array([2.5, 0.25, 1.0]))
    assert k == 2 and w.tolist() == [10, 1, 4]
    assert np.array_equal(np.ldexp(w.astype(np.float64), -k), [2.5, 0.25, 1.0])
    w, k = validate_weights(np.array([3, 4], dtype=np.int64))
    assert k == 0 and w.tolist() == [3, 4]
    assert validate_weights(None) == (None, 0)
    for bad in ([1e-3], [0.1, 1.0], [-1.0], [np.inf], [np.nan]):
        with pytest.raises(ValueError):
            validate_weights(np.array(bad))
    with pytest.raises(ValueError):  # exact, but sums over |V| vertices could reach 2^32 - 1
        validate_weights(np.array([2.0 ** 30 + 0.5]), num_vertices=8)
    with pytest.raises(ValueError):
        validate_weights(np.array([-3], dtype=np.int64))


def test_engine_config_validation():
    from paper_2203_13005_b200.engine import RunConfig, convergence_vote, EngineError
    with pytest.raises(ValueError):
        RunConfig(partitions=0)
    with pytest.raises(ValueError):
        RunConfig(block_size=0)
    assert convergence_vote([True, True]) and not convergence_vote([True, False])
    with pytest.raises(EngineError, match="missing convergence vote"):
        convergence_vote([True, None])


def test_protocol_errors_are_the_reference_type():
    """With the reference loaded, a library protocol error is both this package's and the
    reference's ProtocolError (A/channel.py), so the reference's handlers catch it."""
    import accelgraph.channel as ch
    from paper_2203_13005_b200 import _lib as L
    with pytest.raises(ch.ProtocolError) as exc:
        L.check(L.GXB_EPROTO)
    assert isinstance(exc.value, L.ProtocolError)
    with pytest.raises(ValueError):
        L.check(L.GXB_EINVAL)
    with pytest.raises(MemoryError):
        L.check(L.GXB_ENOMEM)


def test_oracle_thread_control(oracle_lib):
    oracle_lib.set_threads(2)
    assert oracle_lib.max_threads() == 2
    oracle_lib.set_threads(os.cpu_count() or 1)
