"""Warm-up statistics and the device-aware optimizer-state placement plan.

Restates `/root/reference/pkg/src/chunkstar/profiler.py` (PatrickStar §5):

* ``MomentSample`` (R, C, R-C per device per moment) with its accounting
  guard (`profiler.py:28-39`); ``WarmupStats`` peaks/curves (`:42-57`);
* margin = max(0, GPU capacity - peak non-model - chunk working set); the
  first ⌊margin / triplet_bytes⌋ local positions (ascending) keep their
  optimizer triplet on the GPU; ``os_placement`` cpu/gpu overrides
  (`profiler.py:93-130`);
* embedding compute device: CPU iff its fp16 weights outweigh an
  activation round trip (`profiler.py:70-74`);
* exact analytic twins of the warm-up (`profiler.py:133-256`) — used by
  the B200 runtime to size the plan before the first step.
"""

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Set, Tuple

from .chunks import ChunkSet
from .fsm import TensorState
from .memory import DevicePool
from .model import (CPU, GPU, ModelSchema, OpKind, Phase, Timeline,
                    activation_bytes_at)
from .parallel import DpPartition


class ProfileError(KeyError):
    """A statistic was requested for a moment that was never sampled."""


@dataclass(frozen=True)
class MomentSample:
    moment: int
    device: str
    used_bytes: int
    chunk_bytes: int
    non_model_bytes: int

    def __post_init__(self) -> None:
        if self.non_model_bytes < 0 or self.used_bytes < self.chunk_bytes:
            raise AssertionError("sample accounting violated at moment %d" % self.moment)


@dataclass
class WarmupStats:
    samples: List[MomentSample] = field(default_factory=list)
    access_moments: Dict[Tuple[str, int], List[int]] = field(default_factory=dict)
    working_set_bytes: int = 0

    def sample_index(self) -> Dict[Tuple[str, int], MomentSample]:
        return {(s.device, s.moment): s for s in self.samples}

    def peak_non_model(self, device: str = GPU) -> int:
        return max((s.non_model_bytes for s in self.samples if s.device == device),
                   default=0)

    def non_model_curve(self, device: str = GPU) -> List[Tuple[int, int]]:
        return [(s.moment, s.non_model_bytes) for s in self.samples
                if s.device == device]


def chunkable_memory(device_pool: DevicePool, moment: int,
                     samples: Sequence[MomentSample]) -> int:
    hit = next((s for s in samples
                if s.device == device_pool.device and s.moment == moment), None)
    if hit is None:
        raise ProfileError("no sample for device %s at moment %d"
                           % (device_pool.device, moment))
    return device_pool.capacity_bytes - hit.non_model_bytes


def embedding_compute_device(schema: ModelSchema) -> str:
    weights = 2 * schema.embedding_param_count
    roundtrip = 2 * schema.act_unit_bytes
    return CPU if weights > roundtrip else GPU


@dataclass(frozen=True)
class PlacementPlan:
    gpu_margin_bytes: int
    peak_non_model_bytes: int
    working_set_bytes: int
    os_positions_on_gpu: Tuple[int, ...]
    embedding_device: str

    @property
    def os_chunks_on_gpu(self) -> int:
        return 3 * len(self.os_positions_on_gpu)

    def device_of_position(self, position: int) -> str:
        return GPU if position in self.os_positions_on_gpu else CPU


def _pack_plan(peak_nm: int, working_set: int, chunk_set: ChunkSet,
               gpu_capacity_bytes: int, schema: Optional[ModelSchema],
               local_positions: Optional[Sequence[int]],
               os_placement: str) -> PlacementPlan:
    margin = max(0, gpu_capacity_bytes - peak_nm - working_set)
    order = sorted(range(chunk_set.positions) if local_positions is None
                   else local_positions)
    triplet = chunk_set.os_triplet_bytes
    if os_placement == "auto":
        on_gpu = tuple(order[:margin // triplet]) if triplet else ()
    elif os_placement == "gpu":
        on_gpu = tuple(order)
    elif os_placement == "cpu":
        on_gpu = ()
    else:
        raise ValueError("os_placement must be auto, cpu, or gpu")
    return PlacementPlan(
        gpu_margin_bytes=margin, peak_non_model_bytes=peak_nm,
        working_set_bytes=working_set, os_positions_on_gpu=on_gpu,
        embedding_device=embedding_compute_device(schema) if schema else CPU)


def compute_placement_plan(stats: WarmupStats, chunk_set: ChunkSet,
                           gpu_capacity_bytes: int, schema: Optional[ModelSchema],
                           local_positions: Optional[Sequence[int]] = None,
                           os_placement: str = "auto") -> PlacementPlan:
    return _pack_plan(stats.peak_non_model(GPU), stats.working_set_bytes, chunk_set,
                      gpu_capacity_bytes, schema, local_positions, os_placement)


def engine_peak_non_model(schema: ModelSchema, timeline: Timeline) -> int:
    """Warm-up-sampled non-model peak: activations + the live transient
    (BWD grad staging, GPU embedding weights) at the during-event moment."""
    emb_extra = (2 * schema.embedding_param_count
                 if embedding_compute_device(schema) == GPU else 0)
    ck = timeline.checkpointed
    peak = activation_bytes_at(schema, timeline, 0, ck)
    for ev in timeline.events:
        if ev.kind is OpKind.EMBEDDING:
            extra = emb_extra
        elif ev.phase is Phase.BWD:
            extra = ev.param_bytes
        else:
            extra = 0
        peak = max(peak,
                   activation_bytes_at(schema, timeline, 2 * ev.index + 1, ck) + extra,
                   activation_bytes_at(schema, timeline, 2 * ev.index + 2, ck))
    return peak


def analytic_working_set(chunk_set: ChunkSet, timeline: Timeline,
                         partition: Optional[DpPartition] = None,
                         rank: int = 0) -> int:
    """Peak pinned fp16 bytes over the FWD/BWD operators, without simulating.

    Operators pin their chunks for their own duration; a gather pins the
    arriving remote chunks until the first operator touching them ends,
    or until the group's FWD/BWD window closes.
    """
    p = partition.nproc if partition is not None else 1
    is_local = (lambda pos: True) if partition is None else (
        lambda pos: partition.owner_of_position(pos) == rank)
    state: Dict[int, TensorState] = {}
    tensors_at: Dict[int, List[int]] = {}
    for pos in range(chunk_set.positions):
        ids = [t.tensor_id for t in chunk_set.param_chunk(pos).tensors]
        tensors_at[pos] = ids
        for tid in ids:
            state[tid] = TensorState.HOLD if is_local(pos) else TensorState.FREE

    def member_states(group):
        return [state[tid] for pos in group.real_positions for tid in tensors_at[pos]]

    held_remote: Dict[int, List[int]] = {}
    pinned: Set[int] = set()
    peak = 0
    for ev in timeline.events:
        if ev.phase is Phase.ADAM or not ev.tensor_refs:
            continue
        positions = [c.position for c in chunk_set.param_chunks_for_tensors(ev.tensor_refs)]
        groups = []
        if partition is not None and p > 1:
            groups = [partition.groups[g] for g in sorted({pos // p for pos in positions})]
            for g in groups:
                if TensorState.FREE in member_states(g):
                    remote = [pos for pos in g.real_positions if not is_local(pos)]
                    for pos in remote:
                        for tid in tensors_at[pos]:
                            state[tid] = TensorState.HOLD
                    held_remote[g.group_id] = remote
                    pinned.update(remote)
        for tid in ev.tensor_refs:
            state[tid] = TensorState.COMPUTE
        pinned.update(positions)
        peak = max(peak, len(pinned) * chunk_set.param_chunk_bytes)
        done = (TensorState.HOLD_AFTER_BWD if ev.phase is Phase.BWD
                else TensorState.HOLD_AFTER_FWD)
        for tid in ev.tensor_refs:
            state[tid] = done
        pinned.difference_update(positions)
        if ev.phase in (Phase.FWD, Phase.BWD):
            for g in groups:
                if all(s is done for s in member_states(g)):
                    for pos in held_remote.pop(g.group_id, []):
                        for tid in tensors_at[pos]:
                            state[tid] = TensorState.FREE
                        pinned.discard(pos)
        if ev.index == timeline.last_fwd_index:
            for tid, s in state.items():
                if s is TensorState.HOLD_AFTER_FWD:
                    state[tid] = TensorState.HOLD
    return peak


def analytic_placement_plan(schema: ModelSchema, timeline: Timeline,
                            chunk_set: ChunkSet, gpu_capacity_bytes: int,
                            partition: Optional[DpPartition] = None,
                            rank: int = 0,
                            os_placement: str = "auto") -> PlacementPlan:
    local = partition.local_positions(rank) if partition is not None else None
    return _pack_plan(engine_peak_non_model(schema, timeline),
                      analytic_working_set(chunk_set, timeline, partition, rank),
                      chunk_set, gpu_capacity_bytes, schema, local, os_placement)
