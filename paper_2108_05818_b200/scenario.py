"""Rank-local wiring of the chunk step (`/root/reference/pkg/src/chunkstar/scenario.py:105-190`).

``Simulator`` assembles, for one rank, exactly what the reference's
``Simulator`` assembles for rank 0: the timeline, the four chunk lists,
the DP partition, fp16 params initialised on CPU with optimizer state
created lazily at the first ADAM (`scenario.py:122-126`), a GPU pool and a
CPU pool of ``cpu_bytes // nproc``, the manager, the DP runtime and the
engine.  ``run`` is one warm-up plus ``iterations - 1`` measured
iterations.  Here any ``rank`` may be simulated (the reference hard-codes
0), and an executor/collective backend may be attached — the B200 trainer
in :mod:`.trainer` uses precisely this wiring with the payload executor.

Strategy sweeps, verdict tables and time estimates (`scenario.py:193-350`)
are out of scope.
"""

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

from .chunks import ChunkKind, ChunkSet, build_model_chunk_lists
from .config import HardwareSpec, PolicySpec
from .engine import Engine, IterationReport, StepExecutor
from .memory import DevicePool, MemoryManager, PayloadBackend
from .model import CPU, GPU, ModelSchema, Timeline, build_event_timeline
from .parallel import CollectiveBackend, DpPartition, DpRuntime, partition_chunks
from .profiler import PlacementPlan, WarmupStats, compute_placement_plan, \
    embedding_compute_device


@dataclass
class ChunkRunResult:
    schema: ModelSchema
    nproc: int
    reports: List[IterationReport] = field(default_factory=list)
    plan: Optional[PlacementPlan] = None
    warmup_stats: Optional[WarmupStats] = None
    layout_rows: List[Tuple[int, str, int, int, int]] = field(default_factory=list)

    @property
    def feasible(self) -> bool:
        return bool(self.reports) and all(r.feasible for r in self.reports)

    @property
    def failure(self) -> Tuple[Optional[str], Optional[int]]:
        bad = next((r for r in self.reports if not r.feasible), None)
        return (bad.failure_reason, bad.failure_moment) if bad else (None, None)

    @property
    def steady_report(self) -> Optional[IterationReport]:
        ok = [r for r in self.reports if not r.warmup and r.feasible]
        return ok[-1] if ok else None


class Simulator:
    """One rank's chunk-step wiring for a (schema, hardware, policy) point."""

    def __init__(self, schema: ModelSchema, hardware: HardwareSpec,
                 policy: PolicySpec, nproc: int = 1,
                 trace_fn: Optional[Callable] = None, rank: int = 0,
                 payload_backend: Optional[PayloadBackend] = None,
                 collective_backend: Optional[CollectiveBackend] = None,
                 executor: Optional[StepExecutor] = None,
                 non_model_fn: Optional[Callable[[int], int]] = None):
        if nproc < 1:
            raise ValueError("nproc must be >= 1")
        if not 0 <= rank < nproc:
            raise ValueError("rank %d outside [0, %d)" % (rank, nproc))
        self.schema, self.hardware, self.policy = schema, hardware, policy
        self.nproc, self.rank = nproc, rank
        self.timeline: Timeline = build_event_timeline(schema, policy.checkpointing)
        self.chunk_set: ChunkSet = build_model_chunk_lists(schema, policy.capacity_elems)
        self.partition: DpPartition = partition_chunks(self.chunk_set, nproc)
        self.local = self.partition.local_positions(rank)
        self.chunk_set.init_on_cpu(self.local, kinds=(ChunkKind.PARAM_FP16,))
        self.pools: Dict[str, DevicePool] = {
            GPU: DevicePool(GPU, hardware.gpu_bytes),
            CPU: DevicePool(CPU, hardware.cpu_bytes // nproc)}
        self.manager = MemoryManager(self.pools, policy.eviction, backend=payload_backend)
        self.manager.register_chunks(self.chunk_set.chunks.values())
        self.manager.add_extra_model_bytes(CPU, self.chunk_set.embedding.fp16_bytes)
        self.dp = DpRuntime(self.chunk_set, self.partition, self.manager, rank=rank,
                            backend=collective_backend)
        self.engine = Engine(self.chunk_set, self.timeline, self.manager, schema=schema,
                             dp=self.dp, limit_fraction=policy.limit_fraction,
                             non_model_fn=non_model_fn, trace_fn=trace_fn,
                             executor=executor)
        self.engine.embedding_device = embedding_compute_device(schema)

    def _initial_cpu_overflow(self) -> bool:
        pool = self.pools[CPU]
        return pool.used_bytes > pool.capacity_bytes

    def _plan_builder(self):
        gpu_cap = self.pools[GPU].capacity_bytes

        def build(stats: WarmupStats) -> PlacementPlan:
            return compute_placement_plan(stats, self.chunk_set, gpu_cap, self.schema,
                                          local_positions=self.local,
                                          os_placement=self.policy.os_placement)
        return build

    def run(self, iterations: int = 3) -> ChunkRunResult:
        result = ChunkRunResult(schema=self.schema, nproc=self.nproc,
                                layout_rows=self.chunk_set.layout_rows())
        if self._initial_cpu_overflow():
            result.reports.append(IterationReport(iteration=0, warmup=True, feasible=False,
                                                  failure_reason="CPU_OOM",
                                                  failure_moment=0))
            return result
        warm = self.engine.run_iteration(0, warmup=True, plan_builder=self._plan_builder())
        result.reports.append(warm)
        result.warmup_stats, result.plan = self.engine.warmup_stats, self.engine.plan
        for i in range(1, max(iterations, 1)):
            if not result.reports[-1].feasible:
                break
            result.reports.append(self.engine.run_iteration(i, warmup=False))
        return result


def simulate_chunk_strategy(schema: ModelSchema, hardware: HardwareSpec,
                            policy: PolicySpec, nproc: int = 1, iterations: int = 3,
                            trace_fn: Optional[Callable] = None,
                            rank: int = 0) -> ChunkRunResult:
    return Simulator(schema, hardware, policy, nproc, trace_fn=trace_fn,
                     rank=rank).run(iterations)


def _out_of_scope(*args, **kwargs):
    raise NotImplementedError("strategy sweeps / verdict tables are out of scope for "
                              "the B200 chunk-step build (see DESIGN.md)")


run_scenario = _out_of_scope
sweep_max_scale = _out_of_scope
