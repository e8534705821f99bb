"""Two processes on one B200 through the multi-process path of PartitionedRun: CUDA IPC
peer replicas (PageRank: Apply stores into the other process's replica), per-peer delta
arenas (SSSP / CC / LP: the pack kernel stores into the other process's arena), the
device vote and the run-ahead rollback — the paths tools/mgpu_check.py drives under
torchrun on several GPUs, here with a gloo group for the host-side collectives so it runs
on the single GPU of the test box. Results are compared with the CPU oracle."""

from __future__ import annotations

import json
import os
import socket
import sys

import numpy as np
import pytest

from conftest import REPO, assert_attrs_match

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, algo, out_path, split=False):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    from paper_2203_13005_b200.device import DeviceContext, DeviceGraph, DeviceState
    from paper_2203_13005_b200.dist import Collective, PartitionedRun
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    if split:  # split rounds: the local-source pass beside the cross-process exchange
        from paper_2203_13005_b200 import _lib as L
        L.set_option("split_overlap", 1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = RmatParams(scale=12, seed=77, wmax=63 if algo == "sssp" else 0, symmetric=algo == "cc")
        src, dst, w = rmat_host(p)
        ctx = DeviceContext(0)
        g = DeviceGraph(ctx, src, dst, w, part=rank, nparts=world, csr=algo != "pagerank")
        st = DeviceState(g, algo)
        run = PartitionedRun(st, g.bounds(), Collective(), enable_skip=True, device=dev).prepare()
        cap = {"pagerank": 12, "lp": 15}.get(algo, g.num_vertices + 1)
        if algo == "pagerank":
            recs = run.run_rounds(cap)
            it = run.iteration
            ok_path = bool(run._peers)
        else:
            it, _ = run.run(cap)
            recs = run.records
            ok_path = bool(run._dpeers)
        mine = torch.from_numpy(np.nan_to_num(st.read_attrs(owned_only=True), nan=0.0, posinf=np.inf)).to(dev).cpu()
        dist.all_reduce(mine)
        if rank == 0:
            with open(out_path, "w") as fh:
                json.dump({"iterations": it, "attrs": mine.numpy().tolist(), "ipc": ok_path,
                           "moved": int(sum(r.exchanged_bytes for r in recs))}, fh)
        st.free()
        g.free()
        ctx.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo,split", [("pagerank", False), ("sssp", False), ("cc", False), ("lp", False),
                                        ("sssp", True), ("cc", True)])
def test_two_processes_ipc_paths(tmp_path, oracle_lib, algo, split):
    import multiprocessing as mp
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    port = _free_port()
    out = os.path.join(tmp_path, "out.json")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, algo, out, split)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    codes = [p.exitcode for p in procs]
    if any(c is None for c in codes):
        for p in procs:
            p.kill()
        pytest.fail("worker timed out")
    assert codes == [0, 0], codes
    res = json.load(open(out))
    assert res["ipc"], "the IPC path was not taken"
    p = RmatParams(scale=12, seed=77, wmax=63 if algo == "sssp" else 0, symmetric=algo == "cc")
    src, dst, w = rmat_host(p)
    cap = {"pagerank": 12, "lp": 15}.get(algo)
    ref = oracle_lib.OracleGraph(src, dst, None if w is None else w.astype(np.float64)).run(algo, max_iterations=cap)
    assert res["iterations"] == ref.iterations
    assert_attrs_match(algo, np.asarray(res["attrs"]), ref.attrs)
