"""Multi-process (world_size 2, gloo, CPU) tests of the partitioned driver.

`dist.PartitionedRun` — the skip vote, the dense and delta mirror exchanges,
the convergence verdict — runs unchanged over torch.distributed/gloo; the
device state is replaced by a numpy partition with the same surface (iterate /
stats / buffer / pack / unpack / view), so the host protocol of the N > 1 path is
exercised without a GPU and checked against the CPU oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_13005_b200 import _lib as L


class NumpyPartition:
    """Destination-range partition over dense ids with full-length value replicas."""

    def __init__(self, src, dst, algo, part, nparts):
        self.algo = algo
        ids = np.union1d(src, dst)
        self.ids = ids
        V = ids.size
        s = np.searchsorted(ids, src)
        d = np.searchsorted(ids, dst)
        self.V = V
        b = self._cut(V, nparts, d)
        self.bounds = np.array(b, dtype=np.uint64)
        self.lo, self.hi = b[part], b[part + 1]
        owner = np.searchsorted(np.array(b[1:]), np.arange(V), side="right")
        mine = (d >= self.lo) & (d < self.hi)
        self.es, self.ed = s[mine], d[mine]
        self.outdeg = np.bincount(s, minlength=V)
        self.remote = np.zeros(V, dtype=bool)
        cross = owner[s] != owner[d]
        self.remote[s[cross]] = True
        self.iteration = 0
        if algo == "pagerank":
            self.rank = np.ones(V)
            self.contrib = np.where(self.outdeg > 0, 1.0 / np.maximum(self.outdeg, 1), 0.0)
        else:
            self.label = ids.astype(np.int64).copy()
            self.active = np.ones(V, dtype=bool)
        self.rec = 8
        self.send = np.zeros(self.rec * (V + 1), dtype=np.uint8)
        self.recv = np.zeros(self.rec * (V + 1), dtype=np.uint8)
        self._arrays = {}
        self._last = None
        self.changed_slots = np.zeros(0, dtype=np.int64)

    def _cut(self, V, nparts, d):
        return [V * p // nparts for p in range(nparts + 1)]

    def _ptr(self, a):
        self._arrays[a.ctypes.data] = a
        return a.ctypes.data

    def view(self, ptr, nbytes, dtype):
        a = self._arrays[ptr]
        t = torch.from_numpy(a.view(np.uint8)[:nbytes])
        return t.view(torch.float64) if dtype == "f8" else t

    def buffer(self, which):
        if which == L.BUF_VALUES:
            return self._ptr(self.contrib), self.contrib.nbytes
        if which == L.BUF_SEND:
            return self._ptr(self.send), self.send.nbytes
        if which == L.BUF_RECV:
            return self._ptr(self.recv), self.recv.nbytes
        return 0, self.rec

    def iterate(self, direction="auto"):
        lo, hi = self.lo, self.hi
        if self.algo == "pagerank":
            acc = np.zeros(self.V)
            # the device fold order differs from the oracle's: compare with a tolerance
            np.add.at(acc, self.ed, self.contrib[self.es])
            new = 0.15 + 0.85 * acc[lo:hi]
            old = self.rank[lo:hi]
            diff = new != old
            self.max_stat = float(np.max(np.abs(new - old)[diff])) if diff.any() else 0.0
            self.rank[lo:hi] = new
            self.contrib[lo:hi] = np.where(self.outdeg[lo:hi] > 0, new / np.maximum(self.outdeg[lo:hi], 1), 0.0)
            self.n_changed = int(diff.sum())
            self.next_active = hi - lo
            self.remote_active = int(self.remote[lo:hi].sum())
            self.units = int(self.outdeg[lo:hi].sum())
        else:
            m = np.full(self.V, np.iinfo(np.int64).max)
            act = self.active[self.es]
            np.minimum.at(m, self.ed[act], self.label[self.es[act]])
            new = np.minimum(self.label[lo:hi], m[lo:hi])
            ch = np.nonzero(new != self.label[lo:hi])[0] + lo
            self.label[lo:hi] = new
            self.units = int(self.outdeg[self.active].sum())
            self.active[:] = False
            self.active[ch] = True
            self.changed_slots = ch
            self.n_changed = int(ch.size)
            self.next_active = int(ch.size)
            self.remote_active = int(self.remote[ch].sum())
            self.max_stat = 1.0 if ch.size else 0.0
        self.iteration += 1

    def stats(self):
        voted = (self.max_stat < 1e-9) if self.algo == "pagerank" else (self.next_active == 0)
        return {"changed": self.n_changed, "next_active": self.next_active, "next_units": 0,
                "remote_active": self.remote_active, "max_stat": self.max_stat, "voted": int(voted),
                "units": self.units, "direction": 1}

    def pack(self):
        ch = self.changed_slots
        r = np.zeros((ch.size, 2), dtype=np.uint32)
        r[:, 0] = ch
        r[:, 1] = self.label[ch]
        self.send[: r.nbytes] = r.view(np.uint8).ravel()
        return int(ch.size)

    def unpack(self, ptr, count):
        r = self.recv[: 8 * count].view(np.uint32).reshape(count, 2)
        for slot, lab in r:
            if self.lo <= slot < self.hi:
                continue
            self.label[slot] = lab
            self.active[slot] = True


class AsyncNumpyPartition(NumpyPartition):
    """Adds the asynchronous delta surface (stats_device / pack_async / unpack_regions):
    the record count rides in the vote block and records move in one padded all-gather."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.recv = np.zeros(self.rec * 2 * (self.V + 1), dtype=np.uint8)
        self._packed = 0

    def pack_async(self):
        self._packed = self.pack()

    def stats_device(self, out):
        st = self.stats()
        out.copy_(torch.tensor([st["changed"], st["next_active"], st["next_units"], st["remote_active"],
                                self._packed, st["max_stat"]], dtype=torch.float64))
        self._packed = 0

    def unpack_regions(self, ptr, counts, block, frontier_after=None, units_after=None):
        for q, n in enumerate(counts):
            if not n:
                continue
            r = self.recv[8 * q * block: 8 * (q * block + n)].view(np.uint32).reshape(n, 2)
            for slot, lab in r:
                if self.lo <= slot < self.hi:
                    continue
                self.label[slot] = lab
                self.active[slot] = True


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, algo, src, dst, cap, out_q, enable_skip, cls=None, run_kw=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_13005_b200.dist import Collective, PartitionedRun
        st = (cls or NumpyPartition)(src, dst, algo, rank, world)
        run = PartitionedRun(st, st.bounds, Collective(), enable_skip=enable_skip, device=None, **(run_kw or {}))
        it, conv = run.run(cap)
        vals = st.rank if algo == "pagerank" else st.label.astype(np.float64)
        lo, hi = st.lo, st.hi
        out_q.put((rank, it, conv, run.skipped_rounds, lo, hi, vals[lo:hi].copy(),
                   [r.skipped for r in run.records], getattr(st, "dense_rounds", 0)))
    finally:
        dist.destroy_process_group()


def _run(algo, src, dst, cap, enable_skip=True, world=2, cls=None, run_kw=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, algo, src, dst, cap, q, enable_skip, cls, run_kw))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    out = np.concatenate([r[6] for r in res])
    return res, out


@pytest.mark.timeout(300)
def test_pagerank_dense_exchange_matches_oracle(oracle_lib):
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, _ = rmat_host(RmatParams(scale=9, seed=21))
    res, got = _run("pagerank", src, dst, 10)
    ref = oracle_lib.OracleGraph(src, dst).run("pagerank", max_iterations=10)
    assert all(r[1] == ref.iterations for r in res)
    assert np.allclose(got, ref.attrs[:, 0], rtol=1e-12, atol=0)
    assert all(r[3] == 0 for r in res)  # R-MAT: never closed, never skipped


@pytest.mark.timeout(300)
def test_cc_delta_exchange_matches_oracle(oracle_lib):
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, _ = rmat_host(RmatParams(scale=9, seed=22, symmetric=True))
    res, got = _run("cc", src, dst, 1000)
    ref = oracle_lib.OracleGraph(src, dst).run("cc")
    assert all(r[1] == ref.iterations and r[2] == ref.converged for r in res)
    np.testing.assert_array_equal(got, ref.attrs[:, 0])


@pytest.mark.timeout(300)
def test_skip_on_component_aligned_partitions(oracle_lib):
    """SPEC acceptance #7: components aligned with the partition boundary
    skip every intermediate sync round, without changing results."""
    import json
    from conftest import load_golden
    src, dst, w, data, meta = load_golden("gen_components40")
    res, got = _run("cc", src, dst, 1000, enable_skip=True)
    ref = oracle_lib.OracleGraph(src, dst).run("cc")
    np.testing.assert_array_equal(got, ref.attrs[:, 0])
    skipped = res[0][7]
    assert all(skipped[:-1]) and res[0][3] == len(skipped) - 1
    # and nothing is skipped when the option is off
    res2, got2 = _run("cc", src, dst, 1000, enable_skip=False)
    np.testing.assert_array_equal(got2, ref.attrs[:, 0])
    assert res2[0][3] == 0


@pytest.mark.timeout(300)
def test_cc_async_delta_exchange_matches_oracle(oracle_lib):
    """The device-vote path: record counts from the vote rows, one padded all-gather,
    per-peer block unpack (what PartitionedRun runs on B200 for SSSP / CC / LP)."""
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, _ = rmat_host(RmatParams(scale=9, seed=23, symmetric=True))
    res, got = _run("cc", src, dst, 1000, cls=AsyncNumpyPartition)
    ref = oracle_lib.OracleGraph(src, dst).run("cc")
    assert all(r[1] == ref.iterations and r[2] == ref.converged for r in res)
    np.testing.assert_array_equal(got, ref.attrs[:, 0])


class DenseNumpyPartition(AsyncNumpyPartition):
    """Adds the dense mirror exchange surface: the next-value replica (GXB_BUF_VALUES_NEXT,
    owned block = current values) all-gathered in place, then dense_install."""

    dense_rounds = 0

    def buffer(self, which):
        if which == L.BUF_VALUES_NEXT:
            self.nxt = self.label.astype(np.uint32)
            return self._ptr(self.nxt), self.nxt.nbytes
        return super().buffer(which)

    def dense_install(self):
        self.dense_rounds += 1
        for slot in range(self.V):
            if self.lo <= slot < self.hi:
                continue
            if self.nxt[slot] != self.label[slot]:
                self.label[slot] = self.nxt[slot]
                self.active[slot] = True


@pytest.mark.timeout(300)
def test_cc_dense_mirror_exchange_matches_oracle(oracle_lib):
    """Rounds after one that changed most vertices exchange whole value blocks (in-place
    all-gather of the next-value replica + install of the changed mirrors); the rest use
    records — same labels and iteration count as the oracle."""
    rng = np.random.default_rng(5)
    n = 512  # every vertex present, V divisible by the 2 ranks: equal blocks
    a = np.concatenate([np.arange(n), rng.integers(0, n, 3 * n)]).astype(np.uint32)
    b = np.concatenate([(np.arange(n) + 1) % n, rng.integers(0, n, 3 * n)]).astype(np.uint32)
    src, dst = np.concatenate([a, b]), np.concatenate([b, a])
    res, got = _run("cc", src, dst, 1000, cls=DenseNumpyPartition, run_kw={"dense_frac": 0.25})
    ref = oracle_lib.OracleGraph(src, dst).run("cc")
    assert all(r[1] == ref.iterations and r[2] == ref.converged for r in res)
    np.testing.assert_array_equal(got, ref.attrs[:, 0])
    assert all(r[8] > 0 for r in res)  # the dense exchange really ran


class CapacityNumpyPartition(NumpyPartition):
    """Uneven partitions as gxb_graph_build_balanced cuts them: contiguous ranges whose
    cost (12 B per in-edge + 64 B per vertex) is split 3 : 1 (balancer capacity factors)."""

    CAPACITY = (3.0, 1.0)

    def _cut(self, V, nparts, d):
        cost = 12 * np.bincount(d, minlength=V).astype(np.float64) + 64
        cum = np.concatenate([[0.0], np.cumsum(cost)])
        share = np.cumsum([0.0] + list(self.CAPACITY[:nparts]))
        share /= share[-1]
        return [int(np.searchsorted(cum, cum[-1] * f, side="left")) if 0 < f < 1 else (0 if f == 0 else V)
                for f in share]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("algo", ["pagerank", "cc"])
def test_capacity_weighted_partitions_match_oracle(oracle_lib, algo):
    """Uneven owned slices (heterogeneous balancing): the dense all-gather with unequal
    sizes (PageRank) and the delta exchange (CC) still give the oracle's results."""
    from paper_2203_13005_b200.rmat import RmatParams, rmat_host
    src, dst, _ = rmat_host(RmatParams(scale=9, seed=24, symmetric=algo == "cc"))
    cap = 10 if algo == "pagerank" else 1000
    res, got = _run(algo, src, dst, cap, cls=CapacityNumpyPartition)
    sizes = [r[5] - r[4] for r in res]
    assert sizes[0] > 2 * sizes[1]  # really uneven
    ref = oracle_lib.OracleGraph(src, dst).run(algo, max_iterations=cap if algo == "pagerank" else None)
    assert all(r[1] == ref.iterations for r in res)
    if algo == "pagerank":
        assert np.allclose(got, ref.attrs[:, 0], rtol=1e-12, atol=0)
    else:
        np.testing.assert_array_equal(got, ref.attrs[:, 0])
