"""Per-phase timing (totals and per round) of partitioned frontier-algorithm runs under
torchrun (development aid).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29512 tools/mgpu_rounds.py cc 24
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    algo = sys.argv[1] if len(sys.argv) > 1 else "cc"
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams
    ctx = DeviceContext(local)
    p = RmatParams(scale=scale, seed=1, wmax=63 if algo == "sssp" else 0, symmetric=algo == "cc",
                   **({"a": 0.65, "b": 0.15, "c": 0.15} if algo == "lp" else {}))
    src, dst, w = ctx.rmat(p)
    g = DeviceGraph(ctx, src, dst, w, part=rank, nparts=world, csr=True)
    del src, dst, w
    torch.cuda.empty_cache()
    cap = 15 if algo == "lp" else g.num_vertices + 1
    for rep in range(2):
        st = DeviceState(g, algo)
        run = PartitionedRun(st, g.bounds(), Collective(), device=dev).prepare()
        if rep:
            run.phase_times = {}
        dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        per_round = []
        while run.iteration < cap:
            before = dict(run.phase_times or {})
            rec = run.step()
            if rep:
                now = run.phase_times
                per_round.append({"dir": rec.direction, "changed": rec.changed, "units": rec.units,
                                  "next_active": rec.next_active,
                                  **{k: round(1e3 * (now.get(k, 0.0) - before.get(k, 0.0)), 3) for k in now}})
            if rec.converged:
                break
        run.finish()
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        st.free()
    out = {"rank": rank, "algo": algo, "iterations": run.iteration, "ms_total": round(1e3 * el, 3),
           **{k: round(1e3 * v, 3) for k, v in (run.phase_times or {}).items()}, "rounds": per_round}
    allv = [None] * world
    dist.all_gather_object(allv, out)
    if rank == 0:
        for o in allv:
            print(json.dumps(o))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
