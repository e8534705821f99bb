"""Probe: how much of a PageRank S26 pull round do the edges from the top-H sources cost?

Builds the full graph and the graph without the edges whose source is among the H
highest out-degree sources, and times pull rounds of both with CUDA events. The
difference bounds what a separate shared-memory hub pass could save.

    python tools/hub_split_probe.py --scale 26 --hubs 28672,57344
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def time_pr(ctx, s, d, iters=10):
    from paper_2203_13005_b200.device import DeviceGraph, DeviceState
    g = DeviceGraph(ctx, s, d, None, csr=False)
    st = DeviceState(g, "pagerank")
    for _ in range(3):
        st.iterate(direction="pull")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        st.iterate(direction="pull")
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / iters
    st.free()
    g.free()
    torch.cuda.empty_cache()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--hubs", default="28672,57344")
    args = ap.parse_args()
    from paper_2203_13005_b200.device import DeviceContext
    from paper_2203_13005_b200.rmat import RmatParams
    ctx = DeviceContext(0)
    s, d, _ = ctx.rmat(RmatParams(scale=args.scale, seed=1))
    E = s.numel()
    out = {"scale": args.scale, "edges": E, "full_ms": time_pr(ctx, s, d)}
    od = torch.bincount(s.long(), minlength=1 << args.scale)
    order = torch.argsort(od, descending=True)
    for h in [int(x) for x in args.hubs.split(",")]:
        hub = torch.zeros(1 << args.scale, dtype=torch.bool, device=s.device)
        hub[order[:h]] = True
        keep = ~hub[s.long()]
        s2, d2 = s[keep].contiguous(), d[keep].contiguous()
        frac = 1.0 - s2.numel() / E
        out[f"hubs_{h}"] = {"hub_edge_frac": round(frac, 4), "cold_ms": time_pr(ctx, s2, d2)}
        del s2, d2, keep, hub
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
