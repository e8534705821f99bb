"""Per-phase timing of partitioned PageRank steps under torchrun (development aid)."""
from __future__ import annotations
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local); dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    ctx = DeviceContext(local)
    src, dst, w = ctx.rmat(RmatParams(scale=scale, seed=1))
    g = DeviceGraph(ctx, src, dst, None, part=rank, nparts=world, csr=False)
    del src, dst; torch.cuda.empty_cache()
    st = DeviceState(g, "pagerank"); st.profile(enable=True, reset=True)
    run = PartitionedRun(st, g.bounds(), Collective(), device=dev,
                         peer_writes=os.environ.get("GXB_PEER_WRITES", "1") == "1")
    for _ in range(3): run.step()
    if os.environ.get("GXB_PHASES", "1") == "1":
        run.phase_times = {}
    st.profile(reset=True)
    n = 10
    t = time.perf_counter()
    for _ in range(n): run.step()
    torch.cuda.synchronize(); el = time.perf_counter() - t
    prof = st.profile()
    lo, hi = g.owned
    out = {"rank": rank, "owned_slots": hi - lo, "owned_edges": int(g.info.owned_edges),
           "ms_per_step": round(1e3 * el / n, 3), "kernel_ms": round(prof["main_kernel_ms"] / max(1, prof["main_kernel_launches"]), 3),
           "rest_ms": round(prof["rest_ms"] / max(1, prof["main_kernel_launches"]), 3),
           **{k: round(1e3 * v / n, 3) for k, v in (run.phase_times or {}).items()}}
    allv = [None] * world
    dist.all_gather_object(allv, out)
    if rank == 0:
        for o in allv: print(json.dumps(o))
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    main()
