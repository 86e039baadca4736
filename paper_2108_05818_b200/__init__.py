"""paper_2108_05818_b200 — B200-native PatrickStar chunk-managed training step.

Python keeps the reference's decision API (`/root/reference/pkg/src/chunkstar/__init__.py:98-119`,
hot-path names): chunk layout, tensor FSM, eviction, placement plan, DP
protocol and the engine.  The physical step — chunk payloads in HBM and
pinned host DRAM, the fused chunk Adam, pack/cast kernels and NCCL chunk
collectives — is realised by :mod:`.payload` and :mod:`.trainer` over the
C-ABI library ``libchunkstar_b200.so`` (see ``include/chunkstar_b200.h``).

Importing this package does not load CUDA; :mod:`._native` does, and it
raises if the library is missing (no CPU fallback).
"""

from .chunks import (DEFAULT_CAPACITY_ELEMS, Chunk, ChunkKind, ChunkSet, Movability,
                     PackingError, TensorTooLargeError, build_chunk_lists_from_sizes,
                     build_model_chunk_lists, chunk_movability, map_tensors_to_chunks)
from .config import HardwareSpec, PolicySpec, ScenarioConfig, SweepSpec
from .engine import EMBEDDING_LEDGER_ID, Engine, IterationReport, StepExecutor
from .fsm import PINNING_STATES, TensorState, TransitionError, Trigger, next_state
from .memory import (DevicePool, EvictionStrategy, MemoryManager, OOMError,
                     PayloadBackend, TransferEvent, oracle_min_transfers,
                     simulate_cache_fetches)
from .model import (CPU, GPU, ModelSchema, Phase, Timeline, build_event_timeline,
                    build_gpt_schema, param_tensor_specs)
from .parallel import (CollectiveBackend, CollectiveScheme, DpPartition, DpRuntime,
                       closed_form_volume, partition_chunks)
from .profiler import (MomentSample, PlacementPlan, WarmupStats, analytic_placement_plan,
                       analytic_working_set, compute_placement_plan,
                       embedding_compute_device, engine_peak_non_model)
from .scenario import ChunkRunResult, Simulator, simulate_chunk_strategy

__version__ = "0.1.0"
