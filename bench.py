"""Benchmark: GTEPS per BSP iteration of GX-Plug's MSGGen -> MSGMerge -> MSGApply
path (+ mirror exchange) on synthetic R-MAT graphs, on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload pr-s26]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference        # CPU restatement of the reference path

One step = one BSP iteration over the whole graph: Gen∘Merge∘Apply on every
partition, the skip vote, the mirror exchange and the convergence verdict.
value = edges processed per second by the whole job (GTEPS_E = E * K / time),
timed with CUDA events on the launching stream, max over ranks. The graph
(R-MAT, Graph500 parameters, edge factor 16, scrambled ids) is generated on the
device from a fixed seed; its CSC (4.3 GB at scale 26) is far larger than L2,
so no L2 flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "GTEPS/iteration (PageRank, SSSP, R-MAT) at 1/2/4/8 B200; % of HBM roofline"

WORKLOADS = {
    # name: (algo, scale, rmat overrides, iterations-per-run cap, config text)
    "pr-s26": ("pagerank", 26, {}, None, "PageRank on R-MAT scale-26 (~1B edges) edge-partitioned over N B200"),
    "sssp-s26": ("sssp", 26, {"wmax": 63}, None, "SSSP (Bellman-Ford, int weights 1..63) on R-MAT scale-26"),
    "sssp-s22": ("sssp", 22, {"wmax": 63}, None, "SSSP (Bellman-Ford, int weights) on R-MAT scale-22 on 1 B200"),
    "cc-s24": ("cc", 24, {"symmetric": True}, None, "Connected components (min-label) on R-MAT scale-24"),
    "lp-s22": ("lp", 22, {"a": 0.65, "b": 0.15, "c": 0.15}, 15, "Label propagation on skewed R-MAT (a=0.65)"),
    "pr-s16": ("pagerank", 16, {}, 10, "PageRank 10 iters on R-MAT scale-16 (config 1)"),
}


def load_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_first(self, timeout=10.0):
        t = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t < timeout:
            time.sleep(0.01)

    def mark(self, start: bool):
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        inside = [ln for ts, ln in self.lines if t0 - 0.025 <= ts <= t1 + 0.025]
        if not inside and self.lines:  # region shorter than the sampling period: nearest sample
            mid = 0.5 * (t0 + t1)
            inside = [min(self.lines, key=lambda x: abs(x[0] - mid))[1]]
        for ln in inside:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- CPU arm

_CPU_GRAPHS = {}


def cpu_graph(algo, scale, over, seed=1):
    """R-MAT sample graph for the CPU restatement (cached per process)."""
    key = (algo, scale, tuple(sorted(over.items())), seed)
    if key not in _CPU_GRAPHS:
        from oracle import oracle
        from paper_2203_13005_b200.rmat import RmatParams
        p = RmatParams(scale=scale, seed=seed, **over)
        src, dst, w = oracle.rmat(p.scale, p.edge_factor, p.seed, p.a, p.b, p.c, p.wmax, p.scramble, p.symmetric)
        _CPU_GRAPHS[key] = oracle.OracleGraph(src, dst, None if w is None else w.astype("float64"))
    return _CPU_GRAPHS[key]


def host_threads() -> int:
    """Every host core this process may run on (torchrun sets OMP_NUM_THREADS=1 for its
    ranks; the CPU baseline still uses the whole host)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample(algo, scale, over, iters, threads=0, seed=1):
    """Time the CPU restatement of run_reference (oracle/, OpenMP, all host threads)."""
    from oracle import oracle
    g = cpu_graph(algo, scale, over, seed)
    t = time.perf_counter()
    r = g.run(algo, max_iterations=iters, nthreads=threads)
    dt = time.perf_counter() - t
    units = int(r.units.sum())
    return dict(seconds=dt, iterations=r.iterations, edges=g.num_edges, units=units,
                gteps=g.num_edges * r.iterations / dt / 1e9, threads=threads or oracle.max_threads(),
                result=r, graph=g)


def python_reference_sample():
    """The reference itself (pure Python, `accelgraph` from baseline/_ref or sys.path) on
    config C1 — PageRank on R-MAT scale-16 — for one BSP iteration each of `run_reference`
    (A/algorithms.py:298-342) and the `Engine` with one partition (A/engine.py:422-427,
    RunConfig defaults). One core: the reference is GIL-bound."""
    try:
        from paper_2203_13005_b200.dropin import reference
        reference()
        from accelgraph.algorithms import make_algorithm, run_reference
        from accelgraph.engine import RunConfig, run
        from accelgraph.graph import Edge, partition_graph
        from oracle import oracle
    except Exception as exc:  # noqa: BLE001
        return {"available": False, "why": f"{type(exc).__name__}: {exc}"}
    src, dst, _ = oracle.rmat(16, 16, 1, 0.57, 0.19, 0.19, 0, True, False)
    edges = [Edge(a, b) for a, b in zip(src.tolist(), dst.tolist())]
    vertices = set(src.tolist()) | set(dst.tolist())
    out = {"available": True, "config": "C1: PageRank on R-MAT scale-16 (1,048,576 edges), one BSP iteration",
           "cores": 1, "cores_note": f"1 of {os.cpu_count()} cores (GIL)"}
    graph = partition_graph(vertices, edges, [len(vertices)])
    t = time.perf_counter()
    run_reference(make_algorithm("pagerank", vertices, graph.out_degree), vertices, edges, max_iterations=1)
    dt = time.perf_counter() - t
    out["run_reference"] = {"seconds": round(dt, 3), "gteps": round(len(edges) / dt / 1e9, 7)}
    t = time.perf_counter()
    run(graph, make_algorithm("pagerank", vertices, graph.out_degree), "bsp", RunConfig(partitions=1, max_iterations=1))
    dt = time.perf_counter() - t
    out["engine_bsp_m1"] = {"seconds": round(dt, 3), "gteps": round(len(edges) / dt / 1e9, 7)}
    return out


def run_dropin_bench(args):
    """End to end through the reference's own public API: `accelgraph.engine.run` (unmodified
    Engine, agents, shared regions, sync rounds, A/engine.py:422-427) with the B200 daemon
    dropped in (dropin.install), PageRank for `--steps` iterations on R-MAT `--scale`
    (default 18) — wall clock around the call, the graph already in the reference's
    PartitionedGraph. Beside it the reference's own CPU daemon for one iteration of the same
    run (a bounded sample). One process, one GPU."""
    from paper_2203_13005_b200 import dropin  # finds the reference (sys.path or baseline/_ref)
    from accelgraph.algorithms import make_algorithm
    from accelgraph.engine import RunConfig, run
    from accelgraph.graph import Edge, even_sizes, partition_graph

    from oracle import oracle
    scale = args.scale or 18
    m = max(1, args.partitions)
    src, dst, _ = oracle.rmat(scale, 16, 1, 0.57, 0.19, 0.19, 0, True, False)
    t = time.perf_counter()
    edges = [Edge(a, b) for a, b in zip(src.tolist(), dst.tolist())]
    vertices = set(src.tolist()) | set(dst.tolist())
    graph = partition_graph(vertices, edges, even_sizes(len(vertices), m))
    t_build = time.perf_counter() - t
    iters = args.steps

    def one(n, gpu):
        g2 = partition_graph(vertices, edges, even_sizes(len(vertices), m))
        algo = make_algorithm("pagerank", vertices, g2.out_degree)
        cfg = RunConfig(partitions=m, max_iterations=n)
        t0 = time.perf_counter()
        if gpu:
            with dropin.installed():
                attrs, met = run(g2, algo, "bsp", cfg)
        else:
            attrs, met = run(g2, algo, "bsp", cfg)
        return time.perf_counter() - t0, attrs, met

    one(1, True)  # warm-up: context, allocations
    dt, attrs, met = one(iters, True)
    rt, rattrs, _ = one(1, False)
    err = max(abs(attrs[v][0] - rattrs[v][0]) for v in vertices) if iters == 1 else None
    E = len(edges)
    line = {
        "metric": METRIC, "mode": "dropin", "value": round(E * met.iterations / dt / 1e9, 5), "unit": "GTEPS",
        "n_gpus": 1, "steps": iters, "ms_per_step": round(1e3 * dt / max(1, met.iterations), 2),
        "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"dropin-pr-s{scale}", "rmat_scale": scale, "num_edges": E,
                   "num_vertices": len(vertices), "partitions": m,
                   "path": "accelgraph.engine.run (unmodified reference Engine / Agent.request / SharedRegion / "
                           "Daemon loop / gqq-gdq sync round) with dropin.install(): GpuDaemon + GpuAgent, fused rounds"},
        "iterations": met.iterations, "protocol_conformant": met.protocol_conformant(),
        "reference_cpu_daemon": {"iterations": 1, "seconds": round(rt, 3),
                                 "gteps": round(E / rt / 1e9, 7), "cores": 1,
                                 "note": "the same Engine with the reference's own daemon (pure Python, GIL-bound)"},
        "graph_build_s": round(t_build, 1),
    }
    if err is not None:
        line["max_abs_diff_vs_reference"] = err
    emit(line)
    return 0


def run_reference_arm(args):
    """The reference's CPU path on the box's host cores, on the same workload and scale as
    the GPU arm: oracle/gx_oracle.c (run_reference restated in C, OpenMP on every host
    thread) over the same R-MAT graph; a step is one BSP iteration (PageRank) or one run to
    convergence (frontier algorithms), the graph built once before the warm-up. The pure
    Python reference is timed beside it on config C1 (python_reference)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    algo, scale, over, cap, text = WORKLOADS[args.workload]
    if args.scale:
        scale = args.scale
    threads = host_threads()
    from oracle import oracle
    oracle.set_threads(threads)
    t_build = time.perf_counter()
    g = cpu_graph(algo, scale, over)
    t_build = time.perf_counter() - t_build
    t_total, done, edges = 0.0, 0, 0
    if algo == "pagerank":
        # K consecutive BSP iterations of one run (the warm-up run has W): a step = one iteration
        g.run(algo, max_iterations=args.warmup, nthreads=threads)
        t = time.perf_counter()
        r = g.run(algo, max_iterations=args.steps, nthreads=threads)
        t_total = time.perf_counter() - t
        done = r.iterations
        edges = g.num_edges * r.iterations
    else:
        g.run(algo, max_iterations=cap, nthreads=threads)
        for _ in range(args.steps):
            t = time.perf_counter()
            r = g.run(algo, max_iterations=cap, nthreads=threads)
            t_total += time.perf_counter() - t
            done += 1
            edges += g.num_edges * r.iterations
            if t_total > 120.0:
                break
    v = edges / t_total / 1e9
    sample = (f"{done} step(s) of {'1 PageRank BSP iteration' if algo == 'pagerank' else 'one ' + algo + ' run'} "
              f"on the workload's own graph (R-MAT scale-{scale}, {g.num_edges} edges, same generator and seed; "
              f"host graph built once in {t_build:.0f} s, untimed); oracle/gx_oracle.c = run_reference "
              "(A/algorithms.py:298-342) restated in C, OpenMP")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GTEPS",
        "n_gpus": args.gpus, "steps": args.steps, "steps_timed": done, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t_total / done, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if algo == "pagerank" else "u32",
        "data": "synthetic",
        "config": {"workload": args.workload, "description": text, "rmat_scale": scale,
                   "edge_factor": 16, "seed": 1, "parallelism": f"cpu x{threads}"},
        "cpu_baseline": {"value": round(v, 4), "unit": "GTEPS", "cores": threads, "kind": "port", "sample": sample,
                         "same_config": True},
        "e2e": {"value": round(v, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_python_reference:
        line["python_reference"] = python_reference_sample()
    emit(line)
    return 0


# --------------------------------------------------------------------------- GPU arm

def algorithmic_bytes(algo, E, V, units=None, nz=None):
    """PR 12E + 32V; SSSP 24 E_scanned + 36V; CC/LP 8 E_scanned + 12V."""
    if algo == "pagerank":
        return 12 * E + 32 * V
    if algo == "sssp":
        return 24 * (units if units is not None else E) + 36 * V
    return 8 * (units if units is not None else E) + 12 * V


def time_frontier_run(ctx, comm, dev, stream, name, algo, params, cap, peak=None, parity=False):
    """One full run (to convergence or cap) of a frontier algorithm; the first run warms
    allocations, the second is timed per iteration with CUDA events."""
    import torch
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import PartitionedRun
    s, d, w = ctx.rmat(params, stream)
    g = DeviceGraph(ctx, s, d, w, csr=algo in ("sssp", "cc", "lp"), stream=stream)
    del s, d, w
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    limit = cap if cap is not None else g.num_vertices + 1
    for _rep in range(2):
        st = DeviceState(g, algo)
        r = PartitionedRun(st, g.bounds(), comm, device=dev)
        per_iter = []
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        while r.iteration < limit:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rec = r.step()
            b.record(stream)
            per_iter.append((a, b, rec))
            if rec.converged:
                break
        t1.record(stream)
        t1.synchronize()
        ms = t0.elapsed_time(t1)
        attrs = st.read_attrs() if parity and _rep == 1 else None
        st.free()
    scanned = sum(x.units for x in r.records)
    out = {"workload": name, "num_edges": g.num_edges, "num_vertices": g.num_vertices,
           "iterations": r.iteration, "converged": r.records[-1].converged, "total_ms": round(ms, 3),
           "gteps_e": round(g.num_edges * r.iteration / (ms * 1e-3) / 1e9, 2),
           "gteps_ref": round(scanned / (ms * 1e-3) / 1e9, 2),
           "iteration_ms": [round(a.elapsed_time(b), 3) for a, b, _ in per_iter],
           "directions": ["push" if x.direction == 2 else "pull" for _, _, x in per_iter],
           "note": "GTEPS_ref counts the reference's GEN units (out-edges of active vertices)"}
    # a pull round scans every in-edge: its algorithmic bytes (E_scanned = E)
    # over the round's device time, against the measured HBM peak
    pull_ms = sorted(a.elapsed_time(b) for a, b, x in per_iter if x.direction != 2)
    if pull_ms and peak:
        med = pull_ms[len(pull_ms) // 2]
        gbs = algorithmic_bytes(algo, g.num_edges, g.num_vertices) / (med * 1e-3) / 1e9
        out["pull_round_roofline"] = {"bytes": algorithmic_bytes(algo, g.num_edges, g.num_vertices),
                                      "median_ms": round(med, 3), "achieved": round(gbs, 1), "peak": peak,
                                      "unit": "GB/s", "frac": round(gbs / peak, 4)}
    g.free()
    if attrs is not None:  # outside the timed runs: the oracle on the host copy of the stream
        out["parity"] = oracle_parity(algo, params, r.iteration, attrs,
                                      [x.changed for x in r.records], [x.units for x in r.records], cap)
    return out


def oracle_parity(algo, params, iterations, attrs, changed=None, units=None, cap=None, keep=None):
    """Compare a device run with the CPU oracle (oracle/gx_oracle.c, run_reference restated,
    A/algorithms.py:298-342) on the same R-MAT stream: SSSP / CC / LP bit-exact with equal
    per-iteration changed / GEN-unit traces, PageRank within 1e-5 relative per vertex."""
    import numpy as np
    t0 = time.perf_counter()
    try:
        from oracle import oracle
        oracle.set_threads(host_threads())  # every host core (torchrun's ranks default to one)
        src, dst, w = oracle.rmat(params.scale, params.edge_factor, params.seed, params.a, params.b, params.c,
                                  params.wmax if algo == "sssp" else 0, params.scramble, params.symmetric)
        og = oracle.OracleGraph(src, dst, None if w is None else w.astype(np.float64))
        del src, dst, w
        ref = og.run(algo, max_iterations=cap if cap is not None else (iterations if algo == "pagerank" else None))
        want = ref.attrs
        out = {"oracle": "oracle/gx_oracle.c (run_reference restated, A/algorithms.py:298-342)",
               "iterations": iterations, "oracle_iterations": ref.iterations,
               "iterations_equal": iterations == ref.iterations, "vertices": int(want.shape[0])}
        if algo == "pagerank":
            err = np.abs(attrs - want) / np.maximum(1.0, np.abs(want))
            out.update(max_rel_err=float(err.max(initial=0.0)), tolerance=1e-5,
                       ok=bool(out["iterations_equal"] and float(err.max(initial=0.0)) <= 1e-5))
        else:
            mism = int((attrs != want).sum())
            traces = (changed is None or list(changed) == ref.changed.tolist()) and \
                (units is None or list(units) == ref.units.tolist())
            out.update(mismatches=mism, bit_exact=mism == 0, traces_equal=bool(traces),
                       ok=bool(out["iterations_equal"] and mism == 0 and traces))
        out.update(oracle_threads=oracle.max_threads(), seconds=round(time.perf_counter() - t0, 1))
        if keep is not None:
            keep.append(og)  # the host graph of the same workload, reused by the CPU baseline
        del og
        return out
    except Exception as exc:  # noqa: BLE001
        return {"ok": False, "error": f"{type(exc).__name__}: {exc}"}


def check_parity(snap, algo, params, world, rank, dev, keep=None):
    """The timed run's attributes against the oracle for the same number of iterations.
    N > 1: each rank contributes its owned vertices (a sum all-reduce over NaN-masked rows)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rounds, attrs = snap
    if world > 1:
        t = torch.from_numpy(np.nan_to_num(attrs, nan=0.0, posinf=np.inf)).to(dev)
        dist.all_reduce(t)
        attrs = t.cpu().numpy()
        if rank != 0:
            return None
    return oracle_parity(algo, params, rounds, attrs, keep=keep)


_STDOUT_FD = None


def emit(line: dict):
    sys.stdout.flush()
    if _STDOUT_FD is not None:
        os.dup2(_STDOUT_FD, 1)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gxb", choices=["gxb", "reference"])
    ap.add_argument("--workload", default="pr-s26", choices=sorted(WORKLOADS))
    ap.add_argument("--scale", type=int, default=None, help="override the R-MAT scale")
    ap.add_argument("--cpu-scale", type=int, default=22)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed run")
    ap.add_argument("--no-python-reference", action="store_true", help="skip timing the pure-Python reference (C1)")
    ap.add_argument("--no-run-ahead", action="store_true", help="PageRank: wait for every vote before the next round")
    ap.add_argument("--dropin", action="store_true",
                    help="time the unmodified reference Engine with the B200 daemon dropped in (PageRank, "
                         "--scale default 18, --partitions)")
    ap.add_argument("--partitions", type=int, default=1)
    ap.add_argument("--dense-frac", type=float, default=0.0,
                    help="SSSP/CC/LP at N>1: dense mirror exchange after rounds changing this slot fraction (0 = off)")
    args = ap.parse_args()
    # stdout carries exactly one JSON line: library banners (NCCL prints its version when a
    # communicator is created) go to stderr until the line is printed
    global _STDOUT_FD
    sys.stdout.flush()
    _STDOUT_FD = os.dup(1)
    os.dup2(2, 1)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.dropin:
        return run_dropin_bench(args)

    import torch
    import torch.distributed as dist

    from paper_2203_13005_b200 import _lib as L
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams

    world, rank, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"  # the version banner would precede the JSON line on stdout
        dist.init_process_group("nccl", device_id=dev)
    comm = Collective()
    algo, scale, over, cap, text = WORKLOADS[args.workload]
    if args.scale:
        scale = args.scale
    params = RmatParams(scale=scale, seed=1, **over)
    ctx = DeviceContext(local)
    stream = torch.cuda.current_stream(dev)

    # graph: same device-generated edge stream on every rank, own destination range kept
    src, dst, w = ctx.rmat(params, stream)
    graph = DeviceGraph(ctx, src, dst, w, part=rank, nparts=world, csr=algo in ("sssp", "cc", "lp"), stream=stream)
    del src, dst, w
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    E, V = graph.num_edges, graph.num_vertices
    bounds = graph.bounds()

    def new_run():
        st = DeviceState(graph, algo)
        return PartitionedRun(st, bounds, comm, enable_skip=True, device=dev, dense_frac=args.dense_frac).prepare()

    # ---- device-timed steps ----
    clocks = ClockSampler(local).__enter__()
    run = new_run()
    run.state.profile(enable=True, reset=True)
    ahead = algo == "pagerank" and not args.no_run_ahead and run.can_run_ahead() and \
        (world == 1 or bool(run._peers))
    if ahead:
        run.run_rounds(args.warmup)
    for _ in range(0 if ahead else args.warmup):
        run.step()
    if algo != "pagerank":
        # frontier algorithms: time whole runs (a step = one iteration of a fresh run)
        run = new_run()
        run.state.profile(enable=True, reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    run.state.profile(reset=True)
    launches = 0
    step_ms = []
    units = 0
    xbytes = 0
    clocks.wait_first()
    clocks.mark(True)
    t_wall = time.perf_counter()
    if ahead:
        # PageRank: the K rounds run back to back (round k+1 launched before the host reads
        # vote k), timed as one block on the launching stream
        ev0.record(stream)
        recs = run.run_rounds(args.steps)
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        if len(recs) != args.steps:  # converged inside the block: time only the rounds kept
            raise SystemExit(f"run-ahead block converged after {len(recs)} of {args.steps} rounds; "
                             "lower --steps/--warmup")
        units += sum(r.units for r in recs)
        xbytes += sum(r.exchanged_bytes for r in recs)
    for _ in range(0 if ahead else args.steps):
        ev0.record(stream)
        rec = run.step()
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        units += rec.units
        xbytes += rec.exchanged_bytes
        if rec.converged and algo != "pagerank":
            launches += run.state.profile()["kernels_launched"]
            run = new_run()
            run.state.profile(enable=True, reset=True)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    clocks.mark(False)
    # attributes of the timed run, checked against the oracle after everything else (parity)
    snap = None
    if algo == "pagerank" and not args.no_parity:
        snap = (run.iteration, run.state.read_attrs(owned_only=world > 1))
    time.sleep(0.05)
    clocks.__exit__(None, None, None)
    prof = run.state.profile()
    launches += prof["kernels_launched"]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    gteps = E * args.steps / (total_ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (the fused warp-tile Gen∘Merge) ----
    peak, peak_kind = load_peaks()
    lo, hi = graph.owned
    owned_E = int(graph.info.owned_edges)
    kern_ms = prof["main_kernel_ms"] / max(1, prof["main_kernel_launches"])
    if algo == "pagerank":
        kbytes = 12 * owned_E + 8 * (hi - lo)          # idx + gathered contribution per edge, sums out
    elif algo == "sssp":
        kbytes = 24 * owned_E + 16 * (hi - lo)
    else:
        kbytes = 8 * owned_E + 4 * (hi - lo)
    achieved = kbytes / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else None
    it_bytes = algorithmic_bytes(algo, E, V)
    kname = "k_tile_a" if L.get_option("tile_async") else "k_tile_t"
    traffic = None
    try:  # dram bytes per launch of the same kernel from the committed ncu --set full capture
        tr = None
        for name in ("r02_traffic.json", "r01_traffic.json"):  # the latest capture that has it
            path = os.path.join(HERE, "profiles", name)
            if os.path.exists(path) and tr is None:
                with open(path) as fh:
                    tr = json.load(fh).get(f"{algo}-s{scale}", {}).get(kname)
        if tr and world == 1:
            traffic = int(tr["dram_read_bytes"] + tr["dram_write_bytes"])
    except Exception:  # noqa: BLE001
        traffic = None
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4) if achieved else None, "traffic": traffic,
        "kernel": f"{kname} (fused MSGGen+MSGMerge warp tiles)", "kernel_ms": round(kern_ms, 4),
        "algorithmic_bytes_per_launch": kbytes, "peak_kind": peak_kind,
        # whole-job iteration bytes (every rank streams its own slice) over the job's peak
        "iteration_frac": round(it_bytes / (ms_per_step * 1e-3) / 1e9 / (peak * world), 4)
        if algo == "pagerank" else None,
    }

    # ---- e2e through the public API with host buffers (agent pull/push per step) ----
    # Every step installs the attributes from pinned host memory (the agent's
    # pull_from_upper), runs the round, and reads the result back (push_to_upper).
    # The copies run on a copy stream, double-buffered, so step t+1's upload and step t's
    # download overlap the rounds (A/agent.py:282-328's stage tasks beside the compute).
    e2e = None
    if not args.no_e2e:
        st = run.state
        arity = st.arity
        # one agent per partition moves its own vertices (N = 1: all of them)
        st.attrs_scope(world > 1)
        nv = len(graph.owned_ids()) if world > 1 else V
        host_in = [torch.empty(nv * arity, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        host_out = [torch.empty(nv * arity, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        st.attrs_extract(0, stream)
        st.attrs_d2h(host_in[0], 0, stream)
        torch.cuda.synchronize()
        host_in[1].copy_(host_in[0])
        e2e_run = PartitionedRun(st, bounds, comm, enable_skip=True, device=dev).prepare()
        copy = torch.cuda.Stream(dev)       # host -> device
        copy_out = torch.cuda.Stream(dev)   # device -> host (the link is full duplex)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        ev_in, ev_inst, ev_out, ev_d2h = ([ev(), ev()] for _ in range(4))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.attrs_h2d(host_in[0], 0, copy)
        ev_in[0].record(copy)
        for t in range(args.steps):
            b, nb = t % 2, (t + 1) % 2
            stream.wait_event(ev_in[b])
            e2e_run.install(b, stream)                        # update("pull_from_upper") + peer mirrors
            ev_inst[b].record(stream)
            if t + 1 < args.steps:
                if t >= 1:
                    copy.wait_event(ev_inst[nb])              # staging buffer nb was installed at t-1
                st.attrs_h2d(host_in[nb], nb, copy)
                ev_in[nb].record(copy)
            e2e_run.step()                                    # requestGen/Merge/Apply + sync round
            if t >= 2:
                stream.wait_event(ev_d2h[b])                  # output buffer b drained at t-2
            st.attrs_extract(b, stream)                       # update("push_to_upper")
            ev_out[b].record(stream)
            copy_out.wait_event(ev_out[b])
            st.attrs_d2h(host_out[b], b, copy_out)
            ev_d2h[b].record(copy_out)
        copy.synchronize()
        copy_out.synchronize()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e_run.finish()
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        # whole-job bytes: the owned sets partition the vertices
        e2e = {"value": round(E * args.steps / e2e_s / 1e9, 3), "unit": "GTEPS",
               "h2d_bytes_per_step": 8 * V * arity, "d2h_bytes_per_step": 8 * V * arity,
               "path": "gxb_attrs_h2d/install (pull_from_upper) -> round -> gxb_attrs_extract/d2h "
                       "(push_to_upper), pinned host buffers, double-buffered, one copy stream per direction"}

    # ---- secondary workload (SSSP on the same scale) and CPU baseline, rank 0 / N = 1 ----
    skipped_rounds = run.skipped_rounds
    secondary = None
    if world == 1 and not args.no_secondary and algo == "pagerank":
        del run
        graph.free()
        torch.cuda.empty_cache()
        secondary = []
        for wname, walgo, wparams, wcap in (
                ("sssp-s26", "sssp", RmatParams(scale=scale, seed=1, wmax=63), None),
                ("cc-s24", "cc", RmatParams(scale=min(scale, 24), seed=1, symmetric=True), None),
                ("lp-s24-a65", "lp", RmatParams(scale=min(scale, 24), seed=1, a=0.65, b=0.15, c=0.15), 15)):
            secondary.append(time_frontier_run(ctx, comm, dev, stream, wname, walgo, wparams, wcap, peak,
                                               # the SSSP S26 run is checked here; CC S24 and LP S24
                                               # a=0.65 at the same scales by tests/test_gpu_scale.py
                                               parity=not args.no_parity and walgo == "sssp"))
            torch.cuda.empty_cache()

    parity, kept = None, []
    if snap is not None:
        parity = check_parity(snap, algo, params, world, rank, dev, keep=kept if world == 1 else None)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            threads = host_threads()
            if kept:
                # the same graph as the GPU run (built for the parity check): ~cpu_seconds of iterations
                og = kept[0]
                t = time.perf_counter()
                og.run(algo, max_iterations=1, nthreads=threads)
                t1 = time.perf_counter() - t
                iters = max(1, min(200, int(args.cpu_seconds / max(t1, 1e-6))))
                t = time.perf_counter()
                rr = og.run(algo, max_iterations=iters, nthreads=threads)
                dt = time.perf_counter() - t
                cpu = {"value": round(og.num_edges * rr.iterations / dt / 1e9, 4), "unit": "GTEPS", "cores": threads,
                       "kind": "port", "same_config": True,
                       "sample": f"{rr.iterations} {algo} BSP iterations on the same R-MAT scale-{scale} graph "
                                 f"({og.num_edges} edges, {dt:.1f} s), oracle/gx_oracle.c OpenMP restatement of "
                                 "run_reference on every host core"}
            else:
                # a bounded sample of about args.cpu_seconds of CPU work: one timed iteration sizes it
                cs = min(scale, args.cpu_scale)
                r1 = cpu_sample(algo, cs, over, 1, threads)
                iters = max(1, min(2000, int(args.cpu_seconds / max(r1["seconds"], 1e-6))))
                r = cpu_sample(algo, cs, over, iters, threads)
                cpu = {"value": round(r["gteps"], 4), "unit": "GTEPS", "cores": r["threads"], "kind": "port",
                       "same_config": cs == scale,
                       "sample": f"{r['iterations']} {algo} BSP iterations on R-MAT scale-{cs} "
                                 f"({r['edges']} edges, {r['seconds']:.1f} s), oracle/gx_oracle.c OpenMP "
                                 "restatement of run_reference on every host core"}
            if not args.no_python_reference:
                cpu["python_reference"] = python_reference_sample()
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GTEPS", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}
    kept.clear()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gteps, 3), "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if algo == "pagerank" else "u32", "data": "synthetic",
            "config": {"workload": args.workload, "description": text, "rmat_scale": scale,
                       "rmat_abc": [params.a, params.b, params.c], "edge_factor": 16, "seed": 1,
                       "scramble": True, "num_edges": E, "num_vertices": V,
                       "parallelism": f"dst-range partition x{world}" if world > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (CSC 4 B/edge), no flush"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(), "wall_s": round(t_wall, 3),
            "step_ms": [round(x, 4) for x in step_ms] if len(step_ms) <= 64 else None,
            "skipped_rounds": skipped_rounds,
        }
        if world > 1:  # mirror-exchange bytes each GPU receives per round, against NVLink 5
            per = xbytes / max(1, args.steps)
            line["exchange"] = {
                "bytes_per_gpu_per_step": int(per), "gbs_per_gpu": round(per / (ms_per_step * 1e-3) / 1e9, 1),
                "link_peak_gbs": 900, "peer_writes": bool(getattr(run, "_peers", False)),
                "mechanism": "Apply stores into IPC-mapped peer replicas over NVLink (pipelined chunks)"
                if getattr(run, "_peers", False) else "NCCL in-place all-gather"}
        if secondary:
            line["secondary"] = secondary
        if parity is not None:
            line["parity"] = parity
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
