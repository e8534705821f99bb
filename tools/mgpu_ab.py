"""A/B of the multi-GPU PageRank step variants under torchrun (development aid)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local); dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2203_13005_b200 import _lib as L
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    ctx = DeviceContext(local)
    out = []
    for chunks in (1,):
        L.set_option("exchange_chunks", chunks)
        src, dst, _ = ctx.rmat(RmatParams(scale=scale, seed=1))
        g = DeviceGraph(ctx, src, dst, None, part=rank, nparts=world, csr=False)
        del src, dst; torch.cuda.empty_cache()
        for needed, bits in ((False, 64), (True, 64), (False, 32), (True, 32)):
            L.set_option("pr_message_bits", bits)
            reserve, overlap = 0, False
            st = DeviceState(g, "pagerank")
            run = PartitionedRun(st, g.bounds(), Collective(), device=dev, overlap=False, needed_only=needed)
            for _ in range(3): run.step()
            run.finish(); torch.cuda.synchronize(); dist.barrier()
            t = time.perf_counter()
            for _ in range(10): run.step()
            run.finish(); torch.cuda.synchronize()
            el = torch.tensor([time.perf_counter() - t], device=dev)
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
            cnt = st.sparse_counts()
            out.append({"needed_only": needed, "bits": bits, "sparse_used": bool(run._sparse),
                        "recv_frac": round(sum(cnt[1]) / max(1, int(g.bounds()[-1]) - (g.owned[1] - g.owned[0])), 3) if cnt else None,
                        "ms_per_step": round(el.item() * 100, 3)})
            st.free()
        g.free()
    if rank == 0:
        for o in out: print(json.dumps({"world": world, **o}))
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    main()
