"""Multi-GPU parity check (run under torchrun): partitioned device runs vs the CPU oracle.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tools/mgpu_check.py --scale 18
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=18)
    ap.add_argument("--algos", default="pagerank,sssp,cc,lp")
    ap.add_argument("--partitioning", default="edges")
    ap.add_argument("--capacity", default=None, help="comma-separated capacity factors (one per rank)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-side collectives, several ranks may share a GPU (functional check of "
                         "N ranks on fewer devices: IPC peer replicas / arenas work within one device)")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams
    ctx = DeviceContext(local)
    comm = Collective()
    report = {}
    for algo in args.algos.split(","):
        over = {"sssp": dict(wmax=63), "cc": dict(symmetric=True), "lp": dict(a=0.65, b=0.15, c=0.15)}.get(algo, {})
        p = RmatParams(scale=args.scale, seed=77, **over)
        src, dst, w = ctx.rmat(p)
        g = DeviceGraph(ctx, src, dst, w, part=rank, nparts=world, csr=algo in ("sssp", "cc", "lp"),
                        partitioning=args.partitioning,
                        capacity=None if args.capacity is None else [float(x) for x in args.capacity.split(",")])
        st = DeviceState(g, algo)
        run = PartitionedRun(st, g.bounds(), comm, enable_skip=True, device=dev)
        cap = {"pagerank": 10, "lp": 15}.get(algo, g.num_vertices + 1)
        torch.cuda.synchronize()
        t = time.perf_counter()
        it, conv = run.run(cap)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        mine = st.read_attrs(owned_only=True)
        gdev = dev if args.backend == "nccl" else torch.device("cpu")
        gathered = [torch.empty_like(torch.from_numpy(mine)).to(gdev) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine).to(gdev))
        if rank == 0:
            from oracle import oracle
            rows = gathered[0].cpu().numpy()
            for gt in gathered[1:]:
                r = gt.cpu().numpy()
                m = ~np.isnan(r[:, 0])
                rows[m] = r[m]
            hs, hd, hw = src.cpu().numpy().view(np.uint32), dst.cpu().numpy().view(np.uint32), None
            if w is not None:
                hw = w.cpu().numpy().view(np.uint32).astype(np.float64)
            ref = oracle.OracleGraph(hs, hd, hw).run(algo, max_iterations=cap)
            if algo == "pagerank":
                err = float((np.abs(rows - ref.attrs) / np.maximum(1.0, np.abs(ref.attrs))).max())
                ok = err <= 1e-9
            else:
                err = int((rows != ref.attrs).sum())
                ok = err == 0
            report[algo] = dict(ok=bool(ok and it == ref.iterations), iterations=it, ref_iterations=ref.iterations,
                                peer_path=bool(run._peers if algo == "pagerank" else run._dpeers),
                                err=err, seconds=round(dt, 4), skipped=run.skipped_rounds,
                                exchanged_mb=round(sum(r.exchanged_bytes for r in run.records) / 2 ** 20, 2))
        del st, g
    if rank == 0:
        print(json.dumps({"world": world, "devices": torch.cuda.device_count(), "backend": args.backend,
                          "scale": args.scale, "partitioning": args.partitioning, **report}))
        bad = [a for a, r in report.items() if not r["ok"]]
        if bad:
            print("MISMATCH", bad)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
