"""NCCL bandwidth probe under torchrun: in-place all-gather vs grouped P2P all-gather-v."""
import os, time, json
import torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps

res = {}
for mb in (16, 64):
    blk = mb * 2**20 // 8
    buf = torch.zeros(blk * world, dtype=torch.float64, device=dev)
    mine = buf[rank * blk:(rank + 1) * blk]
    ag = timeit(lambda: dist.all_gather_into_tensor(buf, mine))
    def p2p(nchunks=1):
        c = blk // nchunks
        for k in range(nchunks):
            ops = []
            for q in range(world):
                if q == rank: continue
                ops.append(dist.P2POp(dist.isend, buf[rank * blk + k * c: rank * blk + (k + 1) * c], q))
                ops.append(dist.P2POp(dist.irecv, buf[q * blk + k * c: q * blk + (k + 1) * c], q))
            for r in dist.batch_isend_irecv(ops): r.wait()
    pp = timeit(lambda: p2p(1))
    pp4 = timeit(lambda: p2p(4))
    gb = (world - 1) * blk * 8 / 1e9
    res[mb] = {"allgather_ms": round(ag, 3), "p2p_ms": round(pp, 3), "p2p_4chunks_ms": round(pp4, 3),
               "allgather_GBs": round(gb / (ag * 1e-3), 1), "p2p_GBs": round(gb / (pp * 1e-3), 1)}
if rank == 0: print(json.dumps({"world": world, **res}))
dist.destroy_process_group()
