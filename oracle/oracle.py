"""TEST INFRASTRUCTURE ONLY — the CPU parity oracle, never the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module. It wraps
``liboracle.so`` (``gx_oracle.c``), a C restatement of the reference's
``run_reference`` (``pkg/src/accelgraph/algorithms.py:298-342``) that is pinned
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``; checked by ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ALGOS = {"sssp": 0, "pagerank": 1, "lp": 2, "cc": 3}


def build(force: bool = False) -> str:
    """Compile liboracle.so in place (gcc; OpenMP when the toolchain has it)."""
    src = os.path.join(_HERE, "gx_oracle.c")
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "gx_oracle.h")),
        os.path.getmtime(os.path.join(_HERE, "..", "include", "gxb_rmat.h"))):
        return _LIB_PATH
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    base = [cc, "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"]
    try:
        subprocess.run(base[:1] + ["-fopenmp"] + base[1:], check=True, capture_output=True)
    except subprocess.CalledProcessError:
        subprocess.run(base, check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.gxo_graph_new.restype = P
        L.gxo_graph_new.argtypes = [ctypes.c_uint64, P, P, P]
        L.gxo_graph_free.argtypes = [P]
        L.gxo_graph_num_vertices.restype = ctypes.c_uint64
        L.gxo_graph_num_vertices.argtypes = [P]
        L.gxo_graph_num_edges.restype = ctypes.c_uint64
        L.gxo_graph_num_edges.argtypes = [P]
        L.gxo_graph_ids.argtypes = [P, P]
        L.gxo_graph_out_degree.argtypes = [P, P]
        L.gxo_run.restype = ctypes.c_int
        L.gxo_run.argtypes = [P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, ctypes.c_int,
                              P, P, P, P, P, P, P, ctypes.c_int64]
        L.gxo_rmat.restype = ctypes.c_int
        L.gxo_rmat.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                               ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                               ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, P, P, P]
        L.gxo_max_threads.restype = ctypes.c_int
        L.gxo_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class OracleResult:
    ids: np.ndarray          # ascending present ids (uint32)
    attrs: np.ndarray        # (V, arity) float64; SSSP inf = unreachable
    iterations: int
    converged: bool
    units: np.ndarray        # per-iteration GEN units (frontier out-edges)
    changed: np.ndarray      # per-iteration changed-vertex counts
    max_stat: np.ndarray     # per-iteration convergence statistic


class OracleGraph:
    """CSC over present ids, in-edges ordered (source asc, file order)."""

    def __init__(self, src, dst, w=None):
        self.src = np.ascontiguousarray(src, dtype=np.uint32)
        self.dst = np.ascontiguousarray(dst, dtype=np.uint32)
        if self.src.shape != self.dst.shape:
            raise ValueError("src/dst length mismatch")
        self.w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        L = lib()
        self._h = L.gxo_graph_new(len(self.src), _ptr(self.src), _ptr(self.dst), _ptr(self.w))
        if not self._h:
            raise MemoryError("oracle graph allocation failed")
        self.num_vertices = int(L.gxo_graph_num_vertices(self._h))
        self.num_edges = int(L.gxo_graph_num_edges(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().gxo_graph_free(h)
            self._h = None

    def ids(self) -> np.ndarray:
        out = np.empty(self.num_vertices, dtype=np.uint32)
        lib().gxo_graph_ids(self._h, _ptr(out))
        return out

    def out_degree(self) -> np.ndarray:
        out = np.empty(self.num_vertices, dtype=np.uint32)
        lib().gxo_graph_out_degree(self._h, _ptr(out))
        return out

    def run(self, algo: str, sources=None, max_iterations=None, nthreads: int = 0,
            trace_cap: int = 4096) -> OracleResult:
        V = self.num_vertices
        srcs = None if sources is None else np.ascontiguousarray(sources, dtype=np.uint32)
        nsrc = 0 if srcs is None else len(srcs)
        arity_guess = max(nsrc, 4) if algo == "sssp" else 1
        attrs = np.empty(max(V, 1) * arity_guess, dtype=np.float64)
        arity = ctypes.c_int(0)
        iters = ctypes.c_int64(0)
        conv = ctypes.c_int(0)
        tu = np.zeros(trace_cap, dtype=np.int64)
        tc = np.zeros(trace_cap, dtype=np.int64)
        tm = np.zeros(trace_cap, dtype=np.float64)
        rc = lib().gxo_run(self._h, ALGOS[algo], nsrc, _ptr(srcs),
                           -1 if max_iterations is None else int(max_iterations), int(nthreads),
                           _ptr(attrs), ctypes.byref(arity), ctypes.byref(iters), ctypes.byref(conv),
                           _ptr(tu), _ptr(tc), _ptr(tm), trace_cap)
        if rc != 0:
            raise ValueError(f"oracle run failed ({rc})")
        a = arity.value
        n = min(iters.value, trace_cap)
        return OracleResult(self.ids(), attrs[: V * a].reshape(V, a).copy(), int(iters.value),
                            bool(conv.value), tu[:n].copy(), tc[:n].copy(), tm[:n].copy())


def rmat(scale, edge_factor=16, seed=1, a=0.57, b=0.19, c=0.19, wmax=0, scramble=True,
         symmetric=False):
    """Host R-MAT stream (include/gxb_rmat.h); returns (src, dst, w or None)."""
    m = edge_factor << scale
    n = 2 * m if symmetric else m
    src = np.empty(n, dtype=np.uint32)
    dst = np.empty(n, dtype=np.uint32)
    w = np.empty(n, dtype=np.uint32) if wmax else None
    ta, tb, tc = (int(p * 2 ** 32) for p in (a, b, c))
    rc = lib().gxo_rmat(scale, edge_factor, seed, ta, tb, tc, wmax, int(scramble), int(symmetric),
                        _ptr(src), _ptr(dst), _ptr(w))
    if rc != 0:
        raise ValueError("bad rmat parameters")
    return src, dst, w


def max_threads() -> int:
    return int(lib().gxo_max_threads())


def set_threads(n: int) -> None:
    """OpenMP threads for the oracle's later calls (torchrun ranks default to 1)."""
    lib().gxo_set_threads(int(n))
