"""Quick device timing probe (development aid, not the bench contract)."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState  # noqa: E402
from paper_2203_13005_b200.rmat import RmatParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--algo", default="pagerank")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--a", type=float, default=0.57)
    args = ap.parse_args()
    ctx = DeviceContext(0)
    b = c = (1 - args.a - 0.05) / 2
    p = RmatParams(scale=args.scale, seed=1, a=args.a, b=b, c=c, wmax=63 if args.algo == "sssp" else 0,
                   symmetric=args.algo == "cc")
    t0 = time.time()
    src, dst, w = ctx.rmat(p)
    torch.cuda.synchronize()
    t1 = time.time()
    g = DeviceGraph(ctx, src, dst, w, csr=args.algo in ("sssp", "cc", "lp"))
    torch.cuda.synchronize()
    t2 = time.time()
    del src, dst, w
    torch.cuda.empty_cache()
    s = DeviceState(g, args.algo)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times, hist = [], []
    it = 0
    while it < args.iters:
        ev[0].record()
        s.iterate("auto", torch.cuda.current_stream())
        ev[1].record()
        st = s.stats()
        times.append(ev[0].elapsed_time(ev[1]))
        hist.append((st["units"], st["changed"], st["direction"]))
        it += 1
        if st["voted"]:
            break
    E = g.num_edges
    import subprocess
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    out = dict(clocks=clk, scale=args.scale, algo=args.algo, V=g.num_vertices, E=E, gen_s=t1 - t0, build_s=t2 - t1,
               iters=it, ms=[round(x, 4) for x in times], hist=hist[:40],
               gteps_e=[round(E / (x * 1e-3) / 1e9, 2) for x in times][:12])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
