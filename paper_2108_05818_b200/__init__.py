"""paper_2108_05818_b200 — B200-native PatrickStar chunk-managed training step.

Python keeps the reference's decision API (`/root/reference/pkg/src/chunkstar/__init__.py:98-119`,
hot-path names): chunk layout, tensor FSM, eviction, placement plan, DP
protocol and the engine.  The physical step — chunk payloads in HBM and
pinned host DRAM, the fused chunk Adam, pack/cast kernels and NCCL chunk
collectives — is realised by :mod:`.payload` and :mod:`.trainer` over the
C-ABI library ``libchunkstar_b200.so`` (see ``include/chunkstar_b200.h``).

Importing this package does not load CUDA; :mod:`._native` does, and it
raises if the library is missing (no CPU fallback).

HBM is shared between chunk slabs (whole 2·cap / 4·cap-byte payloads that
the accounting trades against activation memory every step) and the model's
activations, so unless the user configured the allocator this package asks
PyTorch for expandable segments (read at the allocator's first use): freed
chunk slabs become pages an activation of any size can reuse, instead of
fixed segments whose fragmentation forces the allocator's free-everything-
and-retry path (measured on the 12B mixed-placement step: 0-1 retries and
1.9-3.0 s/step vs 1-3 retries and 2.2-6.8 s/step; profiles/r01).
"""

import os as _os

_os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

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
