"""The agent: per-partition bridge between the upper system and its GPU daemons.

Drop-in for the reference's `Agent` operation-interface kit (A/agent.py:96-622):
`connect / disconnect / shutdown / transfer / update / request`, the Alg. 2
pipeline driver over three-slot SharedRegions, round-robin dispatch across
daemons, and the per-iteration phases (`begin_iteration`, `work_phase`,
`post_route`, `round_closed`, `vote`, `end_iteration`).

What changes is the unit of work. The reference materialises one Python
`EdgeTriplet` per frontier out-edge (`build_blocks`, A/graph.py:215-245 — 58% of
a PageRank iteration) and ships it through the region; here a work item is a
RangeDescriptor over the device-resident CSC (GEN: owned edge ranges) or over
owned destination slots (MERGE / APPLY), and every result stays in HBM. The
region protocol, the trace and `copy_count == 0` are unchanged.
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from enum import Enum

from .channel import MsgKind, OpKind, ProtocolError, RangeDescriptor, Role, SharedRegion, WorkItem
from .daemon import AcceleratorProfile, GpuDaemon, daemon_init


class AgentPhase(Enum):
    DISCONNECTED = "disconnected"
    CONNECTED = "connected"
    IN_ITERATION = "in_iteration"


@dataclass
class AgentState:
    node_id: int
    daemons: list[str]
    phase: AgentPhase


@dataclass
class IterationCounters:
    """Per-iteration bookkeeping (A/agent.py:41-54); times are the simulated clock."""

    t_download: float = 0.0
    t_compute: float = 0.0
    t_upload: float = 0.0
    pipeline_time: float = 0.0
    units: int = 0
    blocks: int = 0
    cache_hits: int = 0
    cache_misses: int = 0
    uploads: int = 0
    uploads_avoided: int = 0


class GpuAgent:
    """Bridge for one destination partition held by one GPU daemon set."""

    def __init__(self, node_id: int, device_state, algorithm, *, model: str = "bsp",
                 block_size: int = 1 << 22, io_cost: float = 0.0, recv_timeout: float | None = 60.0,
                 fused: bool = False):
        if model not in ("bsp", "gas"):
            raise ValueError(f"unknown computation model {model!r}")
        if isinstance(block_size, int) and block_size < 1:
            raise ValueError(f"block size must be >= 1, got {block_size}")
        self.node_id = node_id
        self.device_state = device_state
        self.algorithm = algorithm
        self.model = model
        self.block_size = block_size if isinstance(block_size, int) else 1 << 22
        self.io_cost = io_cost
        self.recv_timeout = recv_timeout
        # LP folds a multiset, which has no materialised-message form: it runs fused
        self.fused = fused or getattr(algorithm, "device_name", "") == "lp"
        self.phase = AgentPhase.DISCONNECTED
        self.daemons: list[GpuDaemon] = []
        self.regions: dict[str, SharedRegion] = {}
        self._stage_pool: ThreadPoolExecutor | None = None
        self._device_lock = threading.Lock()  # calls on one device state are serialised
        self._pass_seq = 0
        self.counters = IterationCounters()
        self.stats: dict | None = None
        self._applied_this_iteration = False
        graph = device_state.graph
        self.owned = graph.owned
        self.owned_edges = int(graph.info.owned_edges)

    # ---- operation-interface kit (A/agent.py:176-276) ---------------------
    @property
    def state(self) -> AgentState:
        return AgentState(self.node_id, list(self.regions), self.phase)

    def connect(self, daemon_profiles: list[AcceleratorProfile]) -> AgentState:
        if self.phase is not AgentPhase.DISCONNECTED:
            raise ProtocolError(f"node {self.node_id}: connect() while {self.phase.value}")
        if not daemon_profiles:
            raise ValueError("connect() needs at least one daemon profile")
        for i, profile in enumerate(daemon_profiles):
            key = f"node{self.node_id}-daemon{i}"
            self.regions[key] = SharedRegion(key, capacity=self.block_size)
            self.daemons.append(daemon_init(profile, self.algorithm, key, self.regions, self.device_state,
                                            self._device_lock))
        self._stage_pool = ThreadPoolExecutor(max_workers=2 * len(daemon_profiles),
                                              thread_name_prefix=f"node{self.node_id}-stage")
        self.phase = AgentPhase.CONNECTED
        return self.state

    def disconnect(self) -> None:
        if self.phase is AgentPhase.DISCONNECTED:
            raise ProtocolError(f"node {self.node_id}: disconnect() while disconnected")
        self.phase = AgentPhase.DISCONNECTED

    def shutdown(self) -> None:
        for daemon in self.daemons:
            daemon.shutdown()
        if self._stage_pool is not None:
            self._stage_pool.shutdown(wait=False)
            self._stage_pool = None
        self.phase = AgentPhase.DISCONNECTED

    def transfer(self, item: WorkItem, region_key: str) -> None:
        """Place a work item into a region's New-role slot, in situ (A/agent.py:208-222)."""
        if self.phase is AgentPhase.DISCONNECTED:
            raise ProtocolError(f"node {self.node_id}: transfer() while disconnected")
        region = self.regions.get(region_key)
        if region is None:
            raise KeyError(f"unknown region key {region_key!r}")
        if item.units > region.capacity:
            raise ValueError(f"block of {item.units} units exceeds slot capacity {region.capacity}")
        slot = region.slot(Role.NEW)
        if slot.item is not None:
            raise ProtocolError(f"region {region_key}: New buffer already occupied")
        slot.item = item

    def update(self, direction: str) -> None:
        """pull_from_upper / push_to_upper (A/agent.py:224-232). Mirrors are HBM-resident and
        refreshed by the engine's sync round, so there is nothing to move per call."""
        if self.phase is AgentPhase.DISCONNECTED:
            raise ProtocolError(f"node {self.node_id}: update() while disconnected")
        if direction not in ("pull_from_upper", "push_to_upper"):
            raise ValueError(f"unknown update direction {direction!r}")

    def request(self, op_kind: OpKind) -> None:
        """Drive one pipelined pass of op_kind across all daemons (A/agent.py:234-276)."""
        if self.phase is AgentPhase.DISCONNECTED:
            raise ProtocolError(f"node {self.node_id}: request() while disconnected")
        items = self._build_work_items(op_kind)
        self._pass_seq += 1
        seq = self._pass_seq
        k = len(self.daemons)
        shares = [items[i::k] for i in range(k)]
        collected: list[list[WorkItem]] = [[] for _ in range(k)]
        if k == 1:
            collected[0] = self._drive(self.daemons[0].region, shares[0], seq)
        else:
            failures: list[BaseException] = []

            def driver(i: int):
                try:
                    collected[i] = self._drive(self.daemons[i].region, shares[i], seq)
                except BaseException as exc:  # noqa: BLE001
                    failures.append(exc)

            threads = [threading.Thread(target=driver, args=(i,), daemon=True) for i in range(k)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
            if failures:
                raise failures[0]
        done = sorted((it for per in collected for it in per), key=lambda it: it.index)
        self.counters.units += sum(it.units for it in done)
        self.counters.blocks += len(done)
        self.counters.t_compute += sum(d.region.last_compute_time for d in self.daemons)

    def _drive(self, region: SharedRegion, items: list[WorkItem], seq: int) -> list[WorkItem]:
        """Agent side of Alg. 2 (A/agent.py:282-328)."""
        cursor = {"next": 0}
        collected: list[WorkItem] = []

        def download():
            i = cursor["next"]
            if i < len(items):
                cursor["next"] = i + 1
                self.transfer(items[i], region.key)

        def upload():
            slot = region.slot(Role.UPLOAD)
            if slot.item is not None:
                collected.append(slot.item)
                slot.item = None

        download()
        region.send_to_daemon(MsgKind.EXCHANGE_FINISHED, seq)
        up = dl = None
        while True:
            msg = region.recv_agent(timeout=self.recv_timeout)
            if msg.kind is MsgKind.ROTATE_FINISHED:
                up = self._stage_pool.submit(upload) if region.slot(Role.UPLOAD).item is not None else None
                dl = self._stage_pool.submit(download) if cursor["next"] < len(items) else None
            elif msg.kind in (MsgKind.COMPUTE_FINISHED, MsgKind.COMPUTE_ALL_FINISHED):
                for fut in (up, dl):
                    if fut is not None:
                        fut.result()
                up = dl = None
                if msg.kind is MsgKind.COMPUTE_ALL_FINISHED:
                    break
                region.send_to_daemon(MsgKind.EXCHANGE_FINISHED, seq)
            else:
                raise ProtocolError(f"node {self.node_id}: unexpected {msg.kind.value} from daemon")
        return collected

    def _build_work_items(self, op_kind: OpKind) -> list[WorkItem]:
        """Range descriptors instead of triplet blocks (A/agent.py:352-389)."""
        b = self.block_size
        if op_kind is OpKind.GEN:
            lo, hi = 0, self.owned_edges
        elif op_kind in (OpKind.MERGE, OpKind.APPLY):
            lo, hi = self.owned
        else:
            raise ValueError(f"unknown operation kind {op_kind!r}")
        return [WorkItem(op_kind, i, RangeDescriptor(s, min(hi, s + b)), min(hi, s + b) - s)
                for i, s in enumerate(range(lo, hi, b))]

    # ---- iteration phases (A/agent.py:457-622) ------------------------------
    def begin_iteration(self) -> None:
        self.phase = AgentPhase.IN_ITERATION
        self.counters = IterationCounters()
        self._applied_this_iteration = False

    def gen_phase(self) -> None:
        self.update("pull_from_upper")
        if not self.fused:
            self.request(OpKind.GEN)

    def merge_apply_phase(self) -> None:
        if self.fused:
            with self._device_lock:
                self.device_state.iterate()
        else:
            self.request(OpKind.MERGE)
            self.request(OpKind.APPLY)
            with self._device_lock:
                self.device_state.commit()
        self.update("push_to_upper")
        self.stats = self.device_state.stats()
        self._applied_this_iteration = True

    def round_closed(self) -> bool:
        """No next-active vertex has a cross-partition consumer (A/agent.py:533-535)."""
        return self.stats is not None and self.stats["remote_active"] == 0

    def vote(self) -> bool:
        if not self._applied_this_iteration:
            return False
        return bool(self.stats["voted"])

    def end_iteration(self) -> None:
        self.phase = AgentPhase.CONNECTED


Agent = GpuAgent
