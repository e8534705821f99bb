"""The B200 daemon inside the UNMODIFIED reference (`accelgraph`, installed offline into
baseline/_ref or importable from sys.path): the reference's own Engine, Agent.request /
_drive, SharedRegion protocol, Daemon loop and CLI run, with the three seams of
SURVEY.md §8(b) rebound by `dropin.install()` — `accelgraph.agent.daemon_init`
(A/agent.py:186), `accelgraph.daemon.execute_request` (A/daemon.py:191) and
`accelgraph.engine.Agent` (A/engine.py:205).

Checked against the golden Engine runs the reference itself produced
(tests/golden/make_golden.py): attributes, iteration count, convergence, skipped
rounds, per-iteration metrics lines (iter / model / skipped / converged, and the
upload counts of the integer algorithms), protocol-trace conformance, init_count == 1
and copy_count == 0 — for the fused path (default) and the request path
(GEN / MERGE / APPLY range items), one and two daemons per node.
"""

from __future__ import annotations

import io
import math
import os
from contextlib import redirect_stdout

import numpy as np
import pytest

from conftest import golden_cases, load_golden

pytestmark = pytest.mark.gpu

ag = pytest.importorskip("paper_2203_13005_b200.dropin", reason="reference package not importable")


def _cc_class():
    from accelgraph.algorithms import Algorithm, Message

    class ConnectedComponents(Algorithm):
        """Min-label propagation plug-in, as in make_golden.py."""

        name = "cc"

        def initial_attr(self, vid):
            return vid

        def initially_active(self, vid):
            return True

        def gen(self, triplet):
            return Message(triplet.edge.dst, triplet.src_attr)

        def merge_payloads(self, a, b):
            return min(a, b)

        def zero_payload(self):
            return math.inf

        def apply_one(self, vid, old_attr, payload):
            new = min(old_attr, payload)
            return new, new != old_attr

        def default_iteration_cap(self, num_vertices):
            return num_vertices + 1

        def format_attr(self, attr):
            return str(attr)

    return ConnectedComponents


def _ref_graph(tag, m):
    from accelgraph.graph import Edge, even_sizes, partition_graph
    src, dst, w, data, meta = load_golden(tag)
    ww = np.ones(len(src)) if w is None else w
    edges = [Edge(int(a), int(b), float(x)) for a, b, x in zip(src, dst, ww)]
    vertices = {v for e in edges for v in (e.src, e.dst)}
    graph = partition_graph(vertices, edges, even_sizes(len(vertices), m))
    return graph, vertices, data, meta


def _algo(name, vertices, graph):
    from accelgraph.algorithms import make_algorithm
    if name == "cc":
        return _cc_class()()
    return make_algorithm(name, vertices, graph.out_degree)


def _golden_attrs(data, key, algo, out_degree):
    rows, ids = data[key], data["ids"]
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


def _close(got, want, algo, rel=1e-9):
    assert set(got) == set(want)
    if algo == "pagerank":
        for k in want:
            assert got[k][1] == want[k][1]
            assert abs(got[k][0] - want[k][0]) <= rel * max(1.0, abs(want[k][0])), (k, got[k], want[k])
    else:
        assert got == want


def _fields(line, keys):
    kv = dict(tok.split("=", 1) for tok in line.split())
    return {k: kv[k] for k in keys}


def engine_cases():
    return [(c["tag"], key) for c in golden_cases() for key in c["engine"]]


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "request"])
@pytest.mark.parametrize("tag,key", engine_cases())
def test_reference_engine_on_b200(tag, key, fused):
    from accelgraph.channel import trace_conforms
    from accelgraph.engine import RunConfig, run
    meta0 = load_golden(tag)[4]
    em = [e for e in meta0["engine"] if e["key"] == key][0]
    graph, vertices, data, meta = _ref_graph(tag, em["m"])
    want = _golden_attrs(data, key, em["algo"], graph.out_degree)
    for daemons in ((1, 2) if not fused else (1,)):
        graph, vertices, _, _ = _ref_graph(tag, em["m"])
        algo = _algo(em["algo"], vertices, graph)
        cfg = RunConfig(partitions=em["m"], daemons_per_node=daemons, block_size=7 if not fused else 256,
                        enable_skip=em["enable_skip"])
        with ag.installed(fused=fused):
            attrs, metrics = run(graph, algo, em["model"], cfg)
        _close(attrs, want, em["algo"])
        assert metrics.iterations == em["iterations"] and metrics.converged == em["converged"]
        assert metrics.skipped_rounds == em["skipped_rounds"]
        assert metrics.protocol_conformant() and all(trace_conforms(t) for t in metrics.traces.values())
        assert set(metrics.init_counts.values()) == {1} and set(metrics.copy_counts.values()) == {0}
        assert len(metrics.traces) == em["m"] * daemons
        keys = ["iter", "model", "skipped", "converged"] + (["uploads"] if em["algo"] != "pagerank" else [])
        got_lines = [_fields(x, keys) for x in metrics.lines()]
        want_lines = [_fields(x, keys) for x in em["lines"]]
        assert got_lines == want_lines
    assert not ag.installed_now()


def test_seams_are_the_reference_modules():
    import accelgraph.agent as A
    import accelgraph.daemon as D
    import accelgraph.engine as E
    orig = (A.daemon_init, D.execute_request, E.Agent)
    with ag.installed():
        assert A.daemon_init is ag.gpu_daemon_init
        assert D.execute_request is ag.execute_request
        assert E.Agent is ag.GpuAgent and issubclass(ag.GpuAgent, A.Agent)
        assert issubclass(ag.GpuDaemon, D.Daemon)
    assert (A.daemon_init, D.execute_request, E.Agent) == orig


def _write_edges(path, tag):
    src, dst, w, _, _ = load_golden(tag)
    with open(path, "w", encoding="ascii") as fh:
        for i in range(len(src)):
            fh.write(f"{src[i]} {dst[i]}" + ("" if w is None else f" {float(w[i])!r}") + "\n")


def _cli(argv):
    from accelgraph import cli
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


@pytest.mark.parametrize("algo,extra", [("sssp", []), ("lp", []), ("sssp", ["--model", "gas"]),
                                         ("pagerank", ["--max-iterations", "10"]),
                                         ("sssp", ["--enable-skip", "--block-size", "auto"])])
def test_reference_cli_on_b200(tmp_path, algo, extra):
    """`accelgraph run` (A/cli.py:142-251) prints the same dump with the drop-in installed."""
    path = os.path.join(tmp_path, "g.txt")
    _write_edges(path, "random20w")
    argv = ["run", "--graph", path, "--algo", algo, "--partitions", "2", *extra]
    rc_ref, out_ref = _cli(argv)
    with ag.installed():
        rc, out = _cli(argv)
    assert rc == rc_ref and rc in (0, 2)  # 2 = not converged within --max-iterations (A/cli.py:251)
    assert out and not out.startswith("error")
    if algo == "pagerank":
        a = [line.split() for line in out.splitlines()]
        b = [line.split() for line in out_ref.splitlines()]
        assert [x[0] for x in a] == [x[0] for x in b]
        for x, y in zip(a, b):
            assert abs(float(x[1]) - float(y[1])) <= 1e-9 * max(1.0, abs(float(y[1])))
    else:
        assert out == out_ref


def test_dropin_module_cli(tmp_path):
    """`python -m paper_2203_13005_b200.dropin run ...` = the reference CLI on the B200."""
    path = os.path.join(tmp_path, "g.txt")
    _write_edges(path, "gen_components40")
    argv = ["run", "--graph", path, "--algo", "sssp", "--partitions", "3", "--enable-skip"]
    rc_ref, out_ref = _cli(argv)
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = ag.main(argv)
    assert (rc, buf.getvalue()) == (rc_ref, out_ref) and rc == 0 and out_ref
    assert not ag.installed_now()


def test_device_errors_surface_through_the_region():
    """A failing device request reaches the agent the reference's way (region.error re-raised
    by recv_agent, A/daemon.py:188-196, A/channel.py:122-126) and the engine reports it."""
    from accelgraph.engine import EngineError, RunConfig, run
    graph, vertices, _, _ = _ref_graph("random20w", 2)
    algo = _algo("sssp", vertices, graph)
    cfg = RunConfig(partitions=2, block_size=4, barrier_timeout=20.0)
    from paper_2203_13005_b200.device import DeviceState
    saved = DeviceState.request

    def broken(self, op, lo, hi, stream=None):
        return saved(self, op, lo, hi + 10 ** 9, stream)   # out-of-range range -> ValueError

    DeviceState.request = broken
    try:
        with ag.installed(fused=False), pytest.raises(EngineError, match="range|out of"):
            run(graph, algo, "bsp", cfg)
    finally:
        DeviceState.request = saved


def test_isolated_vertices_rejected():
    from accelgraph.engine import RunConfig, run
    from accelgraph.graph import Edge, partition_graph
    edges = [Edge(0, 1, 1.0), Edge(1, 2, 1.0)]
    graph = partition_graph({0, 1, 2, 3}, edges, [2, 2])
    algo = _algo("lp", {0, 1, 2, 3}, graph)
    with ag.installed(), pytest.raises(ValueError, match="appear in an edge"):
        run(graph, algo, "bsp", RunConfig(partitions=2))


def test_reference_cli_sources_and_float_weights(tmp_path):
    """`accelgraph run --sources` with 6 sources over a weighted file with 2.5-style weights."""
    path = os.path.join(tmp_path, "g.txt")
    src, dst, w, _, _ = load_golden("random20w")
    with open(path, "w", encoding="ascii") as fh:
        for i in range(len(src)):
            fh.write(f"{src[i]} {dst[i]} {float(w[i]) / 2!r}\n")
    ids = sorted(set(src.tolist()) | set(dst.tolist()))
    argv = ["run", "--graph", path, "--algo", "sssp", "--partitions", "2",
            "--sources", ",".join(str(v) for v in ids[:6])]
    rc_ref, out_ref = _cli(argv)
    with ag.installed():
        rc, out = _cli(argv)
    assert rc == rc_ref == 0 and out == out_ref
    assert ".5" in out


@pytest.mark.parametrize("algo_name", ["sssp", "pagerank", "lp", "cc"])
@pytest.mark.parametrize("model", ["bsp", "gas"])
def test_reference_engine_cache_and_auto_blocks(algo_name, model):
    """RunConfig(enable_cache=True, block_size="auto") on three partitions: the lazy upload
    serves dirty and queried values, the rest is flushed at the end (A/agent.py:550-611);
    attributes equal the reference's own run of the same configuration."""
    from accelgraph.engine import RunConfig, run
    cfg = dict(partitions=3, enable_cache=True, cache_capacity=8, block_size="auto", enable_skip=True)
    graph, vertices, _, _ = _ref_graph("gen_random40", 3)
    want, wmet = run(graph, _algo(algo_name, vertices, graph), model, RunConfig(**cfg))
    graph, vertices, _, _ = _ref_graph("gen_random40", 3)
    with ag.installed(fused=algo_name != "sssp"):
        got, met = run(graph, _algo(algo_name, vertices, graph), model, RunConfig(**cfg))
    _close(got, want, algo_name)
    assert met.iterations == wmet.iterations and met.converged == wmet.converged
    assert met.skipped_rounds == wmet.skipped_rounds and met.protocol_conformant()
