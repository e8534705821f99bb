import torch, sys, os
sys.path.insert(0, "/root/repo")
from paper_2203_13005_b200.device import DeviceContext
from paper_2203_13005_b200.rmat import RmatParams
ctx = DeviceContext(0)
for scale in (24, 26):
    src, dst, w = ctx.rmat(RmatParams(scale=scale, seed=1))
    V = 1 << scale
    indeg = torch.bincount(dst.to(torch.int64), minlength=V)
    order = torch.argsort(-indeg, stable=True)
    rank = torch.empty(V, dtype=torch.int64, device=indeg.device)
    rank[order] = torch.arange(V, device=indeg.device)
    r = rank[src.to(torch.int64)]
    E = src.numel()
    out = {k: round(float((r < k).sum().item()) / E, 4) for k in (1024, 2048, 4096, 8192, 12288, 16384, 32768, 65536)}
    print(scale, E, out, flush=True)
    del src, dst, indeg, order, rank, r
    torch.cuda.empty_cache()
