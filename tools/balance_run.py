"""Heterogeneous balancing end to end (run under torchrun): every rank measures its own
unit cost on the same workload (the whole graph, the run's own direction schedule;
`balancer.observe`: CUDA-event-timed rounds) in the graph store's cost units, the costs are
all-gathered, and every rank rebuilds its partition with the same capacity factors
(`DeviceGraph(capacity=...)` -> gxb_graph_build_balanced) and checks the run against
the CPU oracle.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29541 tools/balance_run.py --scale 18 [--slow-rank 1]

`--slow-rank r` doubles rank r's measured times, standing in for a device of half the
speed so the plan is visibly uneven.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=18)
    ap.add_argument("--algo", default="sssp")
    ap.add_argument("--slow-rank", type=int, default=-1)
    ap.add_argument("--calib-rounds", type=int, default=8)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2203_13005_b200.balancer import capacity_factors, observe
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    ctx = DeviceContext(local)
    comm = Collective()
    over = {"sssp": dict(wmax=63), "cc": dict(symmetric=True)}.get(args.algo, {})
    src, dst, w = rmat_host(RmatParams(scale=args.scale, seed=91, **over))
    csr = args.algo in ("sssp", "cc", "lp")

    # 1. measure every device on the SAME workload — the whole graph as one partition, with the
    #    direction schedule the run uses — in the store's cost units (12 B per in-edge + 64 B per
    #    vertex, the cost line gxb_graph_build_balanced cuts), so the factors compare devices,
    #    not the contents of their partitions
    g = DeviceGraph(ctx, src, dst, w, part=0, nparts=1, csr=csr)
    s = DeviceState(g, args.algo)
    observe(s, iterations=2, direction="auto")   # warm-up (allocations, L2)
    s.free()
    s = DeviceState(g, args.algo)
    obs = observe(s, iterations=args.calib_rounds, direction="auto")
    if rank == args.slow_rank:
        obs = [(u, b, 2.0 * t) for u, b, t in obs]
    cost_line = 12 * int(g.info.owned_edges) + 64 * int(g.num_vertices)
    unit = sum(t for _, _, t in obs) / (len(obs) * cost_line)
    s.free()
    g.free()
    costs = [None] * world
    dist.all_gather_object(costs, unit)
    cap = capacity_factors([max(c, 1e-15) for c in costs])

    # 2. rebuild with the plan and run against the oracle
    g = DeviceGraph(ctx, src, dst, w, part=rank, nparts=world, csr=csr, capacity=cap)
    s = DeviceState(g, args.algo)
    run = PartitionedRun(s, g.bounds(), comm, enable_skip=True, device=dev)
    limit = {"pagerank": 10, "lp": 15}.get(args.algo, g.num_vertices + 1)
    it, conv = run.run(limit)
    mine = s.read_attrs(owned_only=True)  # non-owned rows are NaN
    gathered = [torch.empty_like(torch.from_numpy(mine)).to(dev) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(mine).to(dev))
    edges = [None] * world
    dist.all_gather_object(edges, int(g.info.owned_edges))
    ok = None
    if rank == 0:
        from oracle import oracle  # test infrastructure: the checker, never the measured path
        full = gathered[0].cpu().numpy()
        for gt in gathered[1:]:
            r = gt.cpu().numpy()
            m = ~np.isnan(r[:, 0])
            full[m] = r[m]
        ref = oracle.OracleGraph(src, dst, None if w is None else w.astype(np.float64)).run(
            args.algo, max_iterations=limit if args.algo in ("pagerank", "lp") else None)
        if args.algo == "pagerank":
            ok = bool(np.allclose(full, ref.attrs, rtol=1e-9, atol=0)) and it == ref.iterations
        else:
            ok = bool(np.array_equal(full, ref.attrs)) and it == ref.iterations
        print(json.dumps({"world": world, "algo": args.algo, "scale": args.scale, "unit_costs_s": costs,
                          "capacity": cap, "owned_edges": edges,
                          "edge_share": [round(e / sum(edges), 4) for e in edges],
                          "iterations": it, "oracle_ok": ok}))
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
