"""Per-partition kernel times of a partitioned frontier run in ONE process on one GPU (the
in-process sync round), against the one-partition run: shows how the round's main kernel
scales with the partition's share of in-edges, without NCCL / NVLink in the way."""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState  # noqa: E402
from paper_2203_13005_b200.engine import exchange_local_peers, setup_local_peers  # noqa: E402
from paper_2203_13005_b200.rmat import RmatParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--algo", default="sssp")
    ap.add_argument("--parts", type=int, default=4)
    args = ap.parse_args()
    ctx = DeviceContext(0)
    p = RmatParams(scale=args.scale, seed=1, wmax=63 if args.algo == "sssp" else 0, symmetric=args.algo == "cc")
    out = {}
    for m in (1, args.parts):
        src, dst, w = ctx.rmat(p)
        gs = [DeviceGraph(ctx, src, dst, w, part=j, nparts=m, csr=True) for j in range(m)]
        del src, dst, w
        torch.cuda.empty_cache()
        sts = [DeviceState(g, args.algo) for g in gs]
        votes = setup_local_peers(sts) if m > 1 else None
        rounds = []
        for _ in range(60):
            ms, dirs = [], []
            for s in sts:
                s.profile(enable=True, reset=True)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                s.iterate()
                b.record()
                b.synchronize()
                st = s.stats()
                pr = s.profile()
                ms.append((round(a.elapsed_time(b), 3), round(pr["main_kernel_ms"], 3)))
                dirs.append(st["direction"])
            x = 0
            if m > 1:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                exchange_local_peers(sts, votes)
                b.record()
                b.synchronize()
                x = round(a.elapsed_time(b), 3)
            rounds.append({"round_ms": ms, "dir": dirs, "exchange_ms": x})
            if all(s.stats()["voted"] for s in sts):
                break
        out[m] = rounds
        for s in sts:
            s.free()
        for g in gs:
            g.free()
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
