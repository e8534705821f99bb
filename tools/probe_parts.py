"""m device partitions of one graph in one process (the engine's in-process sync round:
k_pack / k_unpack between the partitions' replicas) — a profiling target, not the bench."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2203_13005_b200.algorithms import make_algorithm  # noqa: E402
from paper_2203_13005_b200.engine import RunConfig, run  # noqa: E402
from paper_2203_13005_b200.graph import EdgeArrays  # noqa: E402
from paper_2203_13005_b200.rmat import RmatParams, rmat_host  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--algo", default="cc")
    ap.add_argument("--parts", type=int, default=2)
    args = ap.parse_args()
    p = RmatParams(scale=args.scale, seed=1, wmax=63 if args.algo == "sssp" else 0, symmetric=args.algo == "cc")
    src, dst, w = rmat_host(p)
    ea = EdgeArrays(src, dst, None if w is None else w.astype("float64"))
    algo = make_algorithm(args.algo, [], ea.out_degree() if args.algo == "pagerank" else None) \
        if args.algo != "sssp" else make_algorithm("sssp", ea.vertex_ids().tolist()[:4], None)
    t = time.time()
    _, m = run(ea, algo, "bsp", RunConfig(partitions=args.parts, partitioning="edges", enable_skip=True))
    print(json.dumps(dict(algo=args.algo, scale=args.scale, parts=args.parts, iterations=m.iterations,
                          exchanged=m.exchanged_bytes, seconds=round(time.time() - t, 2))))


if __name__ == "__main__":
    main()
