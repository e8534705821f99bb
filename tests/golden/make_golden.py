"""Generate golden vectors by running the REFERENCE itself (this container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports the reference read-only from /root/reference/pkg/src and records, for a
set of graphs x algorithms x iteration caps, the attributes that
``run_reference`` (``A/algorithms.py:298-342``) returns, plus ``Engine`` runs
(``A/engine.py:422-427``) with their iteration/convergence/skip metrics. CC is
not a reference algorithm; it is defined here as a plug-in subclass of the
reference's own ``Algorithm`` base and run through the
reference's own loop and engine, so its golden vectors are produced by
reference code too.

The fixtures travel with the repo; /root/reference does not (nothing at test
time reads it). R-MAT cases store the generator parameters plus a SHA-256 of the
generated edge stream instead of the edges, keeping the fixtures small.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from accelgraph import generators as G  # noqa: E402
from accelgraph.algorithms import Algorithm, Message, make_algorithm, run_reference  # noqa: E402
from accelgraph.engine import RunConfig, run as engine_run  # noqa: E402
from accelgraph.graph import Edge, GraphParseError, even_sizes, load_edge_list, partition_graph  # noqa: E402

from oracle.oracle import rmat  # noqa: E402  (deterministic input stream only)


class ConnectedComponents(Algorithm):
    """Min-label propagation plug-in."""

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


def algo_for(name, vertices, out_degree, sources=None):
    if name == "cc":
        return ConnectedComponents()
    return make_algorithm(name, vertices, out_degree, sources)


def edge_digest(src, dst, w):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(src, dtype=np.uint32).tobytes())
    h.update(np.ascontiguousarray(dst, dtype=np.uint32).tobytes())
    if w is not None:
        h.update(np.ascontiguousarray(w, dtype=np.float64).tobytes())
    return h.hexdigest()


def attrs_matrix(name, ids, attrs):
    if name == "sssp":
        return np.array([attrs[v] for v in ids], dtype=np.float64)
    if name == "pagerank":
        return np.array([[attrs[v][0]] for v in ids], dtype=np.float64)
    return np.array([[attrs[v]] for v in ids], dtype=np.float64)


CASES = []


def add_case(tag, src, dst, w, algos, caps=(None,), rmat_params=None, engine=(), sources=None):
    CASES.append(dict(tag=tag, src=np.asarray(src, dtype=np.uint32),
                      dst=np.asarray(dst, dtype=np.uint32),
                      w=None if w is None else np.asarray(w, dtype=np.float64),
                      algos=algos, caps=caps, rmat=rmat_params, engine=engine, sources=sources))


def pairs(edge_pairs):
    s = [a for a, _ in edge_pairs]
    d = [b for _, b in edge_pairs]
    return s, d


def build_cases():
    ALL = ("sssp", "pagerank", "lp", "cc")
    # graphs from the reference's own tests (T/test_algorithms.py:140-195)
    add_case("path3", *pairs([(0, 1), (1, 2)]), None, ALL, caps=(None, 1, 2),
             engine=[dict(m=2, model="bsp"), dict(m=2, model="gas")])
    add_case("two_cycle", *pairs([(0, 1), (1, 0)]), None, ALL, caps=(None, 1, 2, 3))
    tri = [(a, b) for a in (1, 2, 3) for b in (1, 2, 3) if a != b]
    add_case("triangle", *pairs(tri), None, ALL)
    ring = [(i, (i + 1) % 12) for i in range(12)] + [(i, (i + 5) % 12) for i in range(12)]
    add_case("ring12", *pairs(ring), None, ALL, caps=(None, 1, 3))
    rng = random.Random(11)
    r20 = [(rng.randrange(20), rng.randrange(20), rng.choice([1.0, 2.0, 5.0])) for _ in range(60)]
    add_case("random20w", [e[0] for e in r20], [e[1] for e in r20], [e[2] for e in r20], ALL,
             caps=tuple([None] + list(range(1, 8))),
             engine=[dict(m=2, model="bsp"), dict(m=3, model="gas", block_size=4)])
    add_case("star5", *pairs([(0, i) for i in range(1, 5)]), None, ALL)
    # reference corpus generators (A/generators.py)
    add_case("gen_path10", *pairs(G.generate("path", 10)), None, ALL)
    add_case("gen_cycle10", *pairs(G.generate("cycle", 10)), None, ALL)
    add_case("gen_star10", *pairs(G.generate("star", 10)), None, ALL)
    add_case("gen_random40", *pairs(G.generate("random", 40, p=0.1, seed=3)), None, ALL,
             caps=(None, 1, 2, 3, 5),
             engine=[dict(m=4, model="bsp", enable_skip=True), dict(m=2, model="gas")])
    comp = G.generate("components", 40, k=2, p=0.1, seed=5)
    add_case("gen_components40", *pairs(comp), None, ALL,
             engine=[dict(m=2, model="bsp", enable_skip=True), dict(m=2, model="gas", enable_skip=True)])
    # sparse ids with self loops and duplicates
    sp = [(1000, 7), (7, 1000), (7, 7), (7, 7), (42, 1000), (99999, 42), (42, 99999), (5, 5)]
    add_case("sparse_ids_dups", *pairs(sp), None, ALL, caps=(None, 1, 2))
    # R-MAT (include/gxb_rmat.h); weights integral in [1, 63] for SSSP
    for scale, a, b, c, seed, algos, caps in (
        (6, 0.57, 0.19, 0.19, 1, ALL, (None, 1, 2, 3, 5)),
        (8, 0.57, 0.19, 0.19, 2, ALL, (None, 2)),
        (10, 0.57, 0.19, 0.19, 3, ("sssp", "pagerank", "lp"), (None, 3)),
        (10, 0.65, 0.15, 0.15, 4, ("lp", "sssp"), (None,)),
    ):
        s, d, w = rmat(scale, seed=seed, a=a, b=b, c=c, wmax=63)
        params = dict(scale=scale, edge_factor=16, seed=seed, a=a, b=b, c=c, wmax=63,
                      scramble=True, symmetric=False)
        add_case(f"rmat_s{scale}_a{round(a * 100)}", s, d, w.astype(np.float64), algos, caps,
                 rmat_params=params,
                 engine=[dict(m=2, model="bsp")] if scale <= 8 else [])
    for scale, seed in ((8, 5), (10, 6)):
        s, d, _ = rmat(scale, seed=seed, symmetric=True)
        params = dict(scale=scale, edge_factor=16, seed=seed, a=0.57, b=0.19, c=0.19, wmax=0,
                      scramble=True, symmetric=True)
        add_case(f"rmat_sym_s{scale}", s, d, None, ("cc",), (None, 2), rmat_params=params)
    # larger single-run cases: SURVEY.md §6 config 1 (PR 10 iterations at S16), LP at S12
    s, d, _ = rmat(16, seed=1)
    add_case("rmat_s16_pr10", s, d, None, ("pagerank",), caps=(10,),
             rmat_params=dict(scale=16, edge_factor=16, seed=1, a=0.57, b=0.19, c=0.19, wmax=0,
                              scramble=True, symmetric=False))
    s, d, w = rmat(12, seed=7, wmax=63)
    add_case("rmat_s12", s, d, w.astype(np.float64), ("lp", "sssp", "cc"), caps=(None,),
             rmat_params=dict(scale=12, edge_factor=16, seed=7, a=0.57, b=0.19, c=0.19, wmax=63,
                              scramble=True, symmetric=False))


def run_case(case):
    src, dst, w = case["src"], case["dst"], case["w"]
    edges = [Edge(int(a), int(b), 1.0 if w is None else float(x))
             for a, b, x in zip(src, dst, (w if w is not None else [1.0] * len(src)))]
    vertices = {v for e in edges for v in (e.src, e.dst)}
    ids = sorted(vertices)
    out_degree = {v: 0 for v in ids}
    for e in edges:
        out_degree[e.src] += 1
    arrays = {}
    meta = {"tag": case["tag"], "runs": [], "engine": []}
    if case["rmat"] is None:
        arrays["src"], arrays["dst"] = src, dst
        if w is not None:
            arrays["w"] = w
    else:
        meta["rmat"] = case["rmat"]
        meta["edge_sha256"] = edge_digest(src, dst, w)
        meta["num_edges"] = int(len(src))
    arrays["ids"] = np.array(ids, dtype=np.uint64)
    arrays["out_degree"] = np.array([out_degree[v] for v in ids], dtype=np.uint64)
    for name in case["algos"]:
        for cap in case["caps"]:
            algo = algo_for(name, vertices, out_degree)
            t = time.time()
            attrs = run_reference(algo, vertices, edges, max_iterations=cap)
            key = f"{name}__cap{cap if cap is not None else 'none'}"
            arrays[key] = attrs_matrix(name, ids, attrs)
            meta["runs"].append(dict(algo=name, cap=cap, key=key, seconds=round(time.time() - t, 3),
                                     sources=list(getattr(algo, "sources", [])) or None))
    for eng in case["engine"]:
        m = eng["m"]
        if len(ids) < m:
            continue
        for name in case["algos"]:
            graph = partition_graph(vertices, edges, even_sizes(len(ids), m))
            algo = algo_for(name, vertices, graph.out_degree)
            cfg = RunConfig(partitions=m, block_size=eng.get("block_size", 256),
                            enable_skip=eng.get("enable_skip", False),
                            max_iterations=eng.get("cap"))
            attrs, metrics = engine_run(graph, algo, eng["model"], cfg)
            key = f"engine__{name}__m{m}__{eng['model']}__skip{int(eng.get('enable_skip', False))}"
            arrays[key] = attrs_matrix(name, ids, attrs)
            meta["engine"].append(dict(algo=name, m=m, model=eng["model"], key=key,
                                       enable_skip=eng.get("enable_skip", False),
                                       iterations=metrics.iterations, converged=metrics.converged,
                                       skipped_rounds=metrics.skipped_rounds,
                                       protocol_conformant=metrics.protocol_conformant(),
                                       init_counts=sorted(set(metrics.init_counts.values())),
                                       copy_counts=sorted(set(metrics.copy_counts.values())),
                                       lines=metrics.lines()))
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, f"{case['tag']}.npz"), **arrays)
    return meta


def edge_list_fixtures():
    """Parser behaviour of load_edge_list (A/graph.py:131-166), incl. errors."""
    texts = {
        "ok_mixed": "# comment\n0 1\n1 2 2.5\r\n\n  3 4   \n4 0 0\n# trailing\n2 2\n2 2\n",
        "ok_weights": "10 20 1.5\n20 30 1e-3\n30 10 7\n",
        "err_fields": "0 1\n1 2 3 4\n",
        "err_nonint": "0 1\nx 2\n",
        "err_negid": "0 1\n-1 2\n",
        "err_weight": "0 1 abc\n",
        "err_negw": "0 1\n1 2 -0.5\n",
        "err_float_id": "0 1.0\n",
        "empty": "# nothing\n\n",
    }
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in texts.items():
            p = os.path.join(tmp, name + ".txt")
            with open(p, "w", encoding="ascii", newline="") as fh:
                fh.write(text)
            try:
                vertices, edges = load_edge_list(p)
                out[name] = dict(text=text, ok=True, vertices=sorted(vertices),
                                 edges=[[e.src, e.dst, e.weight] for e in edges])
            except GraphParseError as exc:
                out[name] = dict(text=text, ok=False, lineno=exc.lineno, message=str(exc))
    with open(os.path.join(HERE, "edge_lists.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def main():
    build_cases()
    index = []
    for case in CASES:
        t = time.time()
        meta = run_case(case)
        index.append(dict(tag=case["tag"], runs=[r["key"] for r in meta["runs"]],
                          engine=[e["key"] for e in meta["engine"]]))
        print(f"{case['tag']}: {time.time() - t:.1f}s", flush=True)
    edge_list_fixtures()
    with open(os.path.join(HERE, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1)


if __name__ == "__main__":
    main()
