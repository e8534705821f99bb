"""NCCL all-gather bandwidth probe (in place, equal blocks) under torchrun."""
import os, sys, time, json
import torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
res = {}
for mb in (16, 64, 128, 256):
    blk = mb * 2**20 // 8
    buf = torch.zeros(blk * world, dtype=torch.float64, device=dev)
    mine = buf[rank * blk:(rank + 1) * blk]
    for _ in range(3): dist.all_gather_into_tensor(buf, mine)
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): dist.all_gather_into_tensor(buf, mine)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[mb] = {"ms": round(ms, 3), "busbw_GBs": round((world - 1) * blk * 8 / (ms * 1e-3) / 1e9, 1)}
    # small all_gather latency (vote)
t = torch.zeros(5, dtype=torch.float64, device=dev); o = torch.empty(5 * world, dtype=torch.float64, device=dev)
for _ in range(5): dist.all_gather_into_tensor(o, t)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    dist.all_gather_into_tensor(o, t); o.cpu()
lat = (time.perf_counter() - t0) / 100 * 1e3
if rank == 0: print(json.dumps({"world": world, "allgather": res, "vote_roundtrip_ms": round(lat, 4)}))
dist.destroy_process_group()
