"""A/B the tuning knobs of the pull merge in one process (development aid)."""

from __future__ import annotations

import argparse
import itertools
import json
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2203_13005_b200 import _lib as L  # noqa: E402
from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState  # noqa: E402
from paper_2203_13005_b200.rmat import RmatParams  # noqa: E402


def smi():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                               "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout.strip()
    except Exception as exc:  # noqa: BLE001
        return str(exc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--algo", default="pagerank")
    ap.add_argument("--grid", default='{"tile_minblocks": [0, 4, 6], "l2_hot_mb": [64]}')
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--direction", default="pull")
    args = ap.parse_args()
    grid = json.loads(args.grid)
    ctx = DeviceContext(0)
    p = RmatParams(scale=args.scale, seed=1, wmax=63 if args.algo == "sssp" else 0, symmetric=args.algo == "cc")
    src, dst, w = ctx.rmat(p)
    g = DeviceGraph(ctx, src, dst, w, csr=args.algo in ("sssp", "cc", "lp"))
    del src, dst, w
    torch.cuda.empty_cache()
    keys = list(grid)
    combos = list(itertools.product(*[grid[k] for k in keys]))
    res = {c: [] for c in combos}
    kern = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    print("clocks before:", smi(), flush=True)
    for _ in range(args.rounds):
        for c in combos:
            for k, v in zip(keys, c):
                L.set_option(k, v)
            s = DeviceState(g, args.algo)
            # SSSP: warm to a dense frontier first
            if args.algo == "sssp":
                for _ in range(3):
                    s.iterate("auto")
                    s.stats()
            s.profile(enable=True, reset=True)
            for _ in range(args.iters):
                ev[0].record()
                s.iterate(args.direction)
                ev[1].record()
                s.stats()
                res[c].append(ev[0].elapsed_time(ev[1]))
            pr = s.profile()
            kern.setdefault(c, []).append((pr["main_kernel_ms"] / max(1, pr["main_kernel_launches"]),
                                           pr["rest_ms"] / max(1, pr["main_kernel_launches"])))
            s.free()
    print("clocks after:", smi(), flush=True)
    for c in combos:
        print(json.dumps({"opts": dict(zip(keys, c)), "median_ms": round(statistics.median(res[c]), 4),
                          "min_ms": round(min(res[c]), 4),
                          "kernel_ms": round(statistics.median(k for k, _ in kern.get(c, [(0, 0)])), 4),
                          "rest_ms": round(statistics.median(r for _, r in kern.get(c, [(0, 0)])), 4)}))


if __name__ == "__main__":
    main()
