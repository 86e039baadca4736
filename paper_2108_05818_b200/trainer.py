"""ChunkTrainer: the chunk-managed GPT training step on B200 (the public API).

Wiring (one process per GPU):

* the accounting is the reference's own ``Simulator`` wiring
  (`/root/reference/pkg/src/chunkstar/scenario.py:105-182`) — layout, DP
  partition, fp16 params initialised on the host, lazily born optimizer
  state, GPU and CPU pools, manager, DP runtime, engine — with the payload
  executor attached as payload / collective / step backend;
* the model is the reference-shaped GPT (:mod:`.gpt`); its slot markers call
  :meth:`Engine.start_event` / :meth:`Engine.finish_event`, so forward and
  backward run the timeline's events in order and every fetch, eviction,
  gather, reduce-scatter and parameter re-binding happens at the reference's
  decision point;
* the ADAM event runs the device-side K2 → step scalars → one K1 launch.

Warm-up (iteration 0) uses list-order eviction, the 0.8 soft limit and
records the access trace; the placement plan is computed at its ADAM event
(`engine.py:282-333`); later iterations use the configured strategy.
"""

import gc
import os
import time
import warnings
from typing import Callable, Dict, List, Optional

import torch

from . import kernels as K
from .chunks import ChunkKind
from .config import HardwareSpec, PolicySpec
from .engine import IterationReport
from .gpt import ReferenceShapedGPT, reference_tensor_shapes
from .memory import OOMError
from .model import CPU, GPU, ModelSchema
from .embedding import HostEmbedding
from .payload import ChunkComm, ChunkPayloadExecutor
from .profiler import embedding_compute_device
from .scenario import Simulator
from . import hostres


def _host_ram_bytes() -> int:
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 256 * 10**9


class PendingLoss:
    """A step's loss on its way to the host (pinned D2H + event)."""

    __slots__ = ("_host", "_done")

    def __init__(self, loss: torch.Tensor):
        self._host = torch.empty((), dtype=loss.dtype, pin_memory=True)
        self._host.copy_(loss, non_blocking=True)
        self._done = torch.cuda.Event()
        self._done.record()

    def ready(self) -> bool:
        return self._done.query()

    def result(self) -> float:
        self._done.synchronize()
        return float(self._host)


class StepInfeasible(OOMError):
    """A training step ran out of memory: the accounting's OOMError, or a
    physical allocation failure (torch.OutOfMemoryError) — the reference
    turns both into an infeasible IterationReport (`engine.py:349-352`),
    which is ``.report`` (also the trainer's last report).  The trainer
    refuses further steps: like the reference's ``Simulator.run``
    (`scenario.py:176-181`), a run stops at its first infeasible iteration."""

    def __init__(self, report: IterationReport, cause: Optional[BaseException] = None):
        dev = "gpu" if report.failure_reason == "GPU_OOM" else "cpu"
        moment = -1 if report.failure_moment is None else report.failure_moment
        super().__init__(dev, moment, 0, 0)
        self.args = ("iteration %d infeasible: %s at moment %d%s"
                     % (report.iteration, report.failure_reason, moment,
                        "" if cause is None else " (%s)" % str(cause).splitlines()[0][:200]),)
        self.report = report
        self.cause = cause


class ChunkTrainer:
    """Chunk-managed (PatrickStar) data-parallel GPT training on one GPU per rank."""

    def __init__(self, schema: ModelSchema, policy: Optional[PolicySpec] = None,
                 hardware: Optional[HardwareSpec] = None, dtype: torch.dtype = torch.float16,
                 seed: int = 0, hyper: Optional[K.AdamHyper] = None,
                 device: Optional[torch.device] = None,
                 process_group=None, max_grad_norm: float = 0.0,
                 init_loss_scale: Optional[float] = None,
                 dynamic_loss_scale: Optional[bool] = None,
                 non_model_fn: Optional[Callable[[int], int]] = None,
                 host_threads: int = 0, time_copies: bool = False,
                 cuda_graph: bool = False, fused_ops: bool = True,
                 prefetch_depth: int = 2, non_model: str = "auto",
                 gather_depth: int = 2, embedding_placement: str = "plan",
                 untied_head: bool = False,
                 async_host_adam: Optional[bool] = None,
                 comm=None, bind_host: Optional[bool] = None,
                 speculative_host_adam: Optional[bool] = None,
                 graph_multi_rank: Optional[bool] = None,
                 embedding_weights: str = "hbm"):
        if not torch.cuda.is_available():
            raise RuntimeError("ChunkTrainer needs a CUDA device (B200); there is no CPU path")
        self.device = torch.device(device or "cuda:%d" % torch.cuda.current_device())
        torch.cuda.set_device(self.device)
        self.schema = schema
        self.dtype = dtype
        self.policy = policy or PolicySpec()
        nproc, rank = 1, 0
        if comm is not None:  # a caller-supplied communicator with ChunkComm's interface
            nproc, rank = comm.world, comm.rank
        elif process_group is not None or (torch.distributed.is_initialized()
                                           and torch.distributed.get_world_size() > 1):
            if os.environ.get("CS_COMM", "torch") == "native":  # the C-ABI communicator
                from .native_comm import NativeChunkComm
                comm = NativeChunkComm(process_group, self.device)
            else:
                comm = ChunkComm(process_group)
            nproc, rank = comm.world, comm.rank
        # host cores: one process per GPU binds to its share of its GPU's NUMA
        # node (pinned slabs are first-touched there too) and every host
        # kernel gets an explicit team size (torchrun sets OMP_NUM_THREADS=1)
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        if bind_host is None:
            bind_host = local_world > 1
        self.host_binding = (hostres.bind_local_rank(
            int(os.environ.get("LOCAL_RANK", "0")), local_world, self.device.index or 0)
            if bind_host else {"bound": False})
        host_threads = hostres.host_threads(host_threads)
        self.host_threads = host_threads
        # where the embedding operator physically runs: the reference's plan
        # (`profiler.py:70-74`, the Simulator sets it on the engine) unless
        # forced.  A CPU-placed embedding needs an untied LM head (the tied
        # head's weights are the embedding's, needed on the GPU from the first
        # forward op to the last backward op), and the untied head is an
        # explicit opt-in: the batch size must not change the model.  So a
        # tied model whose plan says CPU computes the embedding on the GPU.
        planned_emb = embedding_compute_device(schema)
        if embedding_placement == "plan":
            embedding_placement = planned_emb
            if planned_emb == CPU and not untied_head:
                warnings.warn("the placement plan puts the embedding on the CPU, which needs "
                              "an untied LM head (untied_head=True); this tied model computes "
                              "it on the GPU and the ledger's embedding rows are not realized",
                              stacklevel=2)
                embedding_placement = GPU
        if embedding_placement not in (CPU, GPU):
            raise ValueError("embedding_placement must be 'plan', 'cpu' or 'gpu'")
        if embedding_placement == CPU and not untied_head:
            raise ValueError("a CPU-placed embedding needs an untied LM head (untied_head=True)")
        # a GPU-computed embedding's weights and optimizer state: resident in
        # HBM and updated by K1 ("hbm", the default), or in pinned host DRAM
        # with the reference's round trip realised ("host": weights down for
        # the forward, weight gradients up, host Adam; `engine.py:214-219`)
        if embedding_weights not in ("hbm", "host"):
            raise ValueError("embedding_weights must be 'hbm' or 'host'")
        dev_emb_host = embedding_placement == GPU and embedding_weights == "host"
        self.embedding_weights = "host" if embedding_placement == CPU else embedding_weights
        V, H, S = schema.vocab, schema.hidden_dim, schema.seq_len
        # non-chunked parameters that live in HBM for the whole run: fp16/bf16
        # weights (their gradients overwrite them) + fp32 master / m / v
        if embedding_placement == CPU:
            emb_bytes = 0
        elif dev_emb_host:  # wte's HBM copy (fp16 only); wpe with its state
            emb_bytes = V * H * 2 + S * H * 14
        else:
            emb_bytes = (V + S) * H * 14
        self.gpu_resident_bytes = emb_bytes + (V * H * 14 if untied_head else 0)
        if non_model == "auto":
            non_model = "measured" if hardware is None and non_model_fn is None else "analytic"
        if hardware is None:
            total = torch.cuda.get_device_properties(self.device).total_memory
            # the accounting may plan chunks into a fraction of HBM minus the
            # non-chunked state resident beside them (charged here so the
            # planner never commits HBM that is already in use); the rest is
            # the CUDA context, NCCL buffers and allocator slack.  With the
            # measured warm-up tracer R - C already holds the activations and
            # library workspaces, so less slack is kept than with the
            # reference's analytic activation model.
            frac = float(os.environ.get("CS_GPU_FRAC", 0.93 if non_model == "measured" else 0.9))
            hardware = HardwareSpec(gpu_count=nproc,
                                    gpu_bytes=int(total * frac) - self.gpu_resident_bytes,
                                    cpu_bytes=int(_host_ram_bytes() * 0.8))
        fp16 = dtype == torch.float16
        if dynamic_loss_scale is None:
            dynamic_loss_scale = fp16
        if init_loss_scale is None:
            init_loss_scale = 2.0 ** 16 if dynamic_loss_scale else 1.0
        self.hyper = hyper or K.AdamHyper(lr=1e-4, betas=(0.9, 0.999), eps=1e-8)
        self.executor = ChunkPayloadExecutor(
            self.device, dtype, self.hyper, init_loss_scale=init_loss_scale,
            dynamic_loss_scale=dynamic_loss_scale, max_grad_norm=max_grad_norm, comm=comm,
            host_threads=host_threads, time_copies=time_copies)
        ex = self.executor
        if async_host_adam is not None:
            ex.async_host_adam = async_host_adam
        if speculative_host_adam is not None:
            ex.speculative_host_adam = speculative_host_adam
        self.tracer = None
        if non_model == "measured" and non_model_fn is None:
            from .tracer import MemoryTracer
            self.tracer = non_model_fn = MemoryTracer(ex, self.device)
        elif non_model not in ("analytic", "measured"):
            raise ValueError("non_model must be 'analytic' or 'measured'")
        self.sim = Simulator(schema, hardware, self.policy, nproc=nproc, rank=rank,
                             payload_backend=ex, collective_backend=ex, executor=ex,
                             non_model_fn=non_model_fn)
        self.nproc, self.rank = nproc, rank
        assert self.sim.engine.embedding_device == planned_emb
        self.embedding_placement = embedding_placement
        self.untied_head = untied_head
        host_emb = embedding_placement == CPU
        with torch.device(self.device):
            self.model = ReferenceShapedGPT(schema, dtype=dtype, placeholders=True,
                                            fused=fused_ops, untied_head=untied_head)
        self.host_embedding = None
        if host_emb or dev_emb_host:
            self.host_embedding = HostEmbedding(schema.vocab, schema.seq_len,
                                                schema.hidden_dim, dtype, self.device,
                                                threads=host_threads,
                                                device_compute=dev_emb_host)
            if host_emb:
                self.model.host_embedding = self.host_embedding
            else:
                self.host_embedding.device_params = [self.model.embedding_parameters()[0]]
            ex.host_embedding = self.host_embedding
        self.shapes = reference_tensor_shapes(schema)
        if fused_ops and K.layernorm_supported(schema.hidden_dim):
            for blk in self.model.blocks:
                blk.fused_ln = True
        self.model.attach_events(self.sim.timeline)
        self._events = self.sim.timeline.events
        self.model.driver.on_start = self._on_start
        self.model.driver.on_finish = self._on_finish
        # non-chunked GPU parameters updated by K1: the embedding when it is
        # GPU-placed, else the (untied) LM head
        emb = []
        V, H = schema.vocab, schema.hidden_dim
        # (param, shape, seed offset): wte 0, wpe 1, untied head 2 — the same
        # values wherever each one lives
        wte_p, wpe_p = self.model.embedding_parameters()
        gpu_params = ([] if host_emb else
                      [(wpe_p, (schema.seq_len, H), 1)] if dev_emb_host else
                      [(wte_p, (V, H), 0), (wpe_p, (schema.seq_len, H), 1)])
        if untied_head:
            gpu_params.append((self.model.lm_head, (V, H), 2))
        self._emb_seed_offsets = [k for _, _, k in gpu_params]
        for p, shape, _ in gpu_params:
            master = torch.empty(shape, dtype=torch.float32, device=self.device)
            emb.append((p, master, torch.zeros_like(master), torch.zeros_like(master)))
        ex.attach(self.sim.chunk_set, self.sim.partition, rank,
                  self.model.chunk_parameters(), self.shapes,
                  [(p, mst.view(-1), m.view(-1), v.view(-1)) for p, mst, m, v in emb],
                  embedding_keys=self._emb_seed_offsets)
        ex.set_timeline(self.sim.timeline)
        self._init_weights(seed, emb)
        self.iteration = 0
        self.reports: List[IterationReport] = []
        self.failed: Optional[IterationReport] = None
        self.sim.engine.physical_oom = (torch.OutOfMemoryError,)
        self.cuda_graph = cuda_graph
        #: capture the ZeRO step (its NCCL all-gathers / reduce-scatters and
        #: the scalar all-reduces are captured as graph nodes, NCCL >= 2.9.6)
        #: at p > 1 too; opt-in (CS_GRAPH_DP=1) until validated on a multi-GPU
        #: box: this sandbox has one GPU and gloo collectives are not capturable
        if graph_multi_rank is None:
            graph_multi_rank = os.environ.get("CS_GRAPH_DP", "0") == "1"
        self.graph_multi_rank = graph_multi_rank
        self.prefetch_depth = prefetch_depth
        self.gather_depth = gather_depth
        self._graph = None
        self._side = None
        self.graph_kernels_per_step = 0
        self.phase_seconds = {"fwd": 0.0, "bwd": 0.0, "adam": 0.0}
        #: NVTX ranges per timeline event, chunk move and collective (CS_NVTX=1)
        self.nvtx = os.environ.get("CS_NVTX", "0") == "1"
        self.executor.nvtx = self.nvtx

    # -- initialisation ---------------------------------------------------------------

    def _init_weights(self, seed: int, emb) -> None:
        """N(0, 0.02) weights, a pure function of (seed, tensor id): identical
        for every world size.  Each local fp16 chunk is cast+packed (K5) on
        the GPU, then lands in its pinned host slab (`scenario.py:126`
        initialises fp16 params on the CPU); the fp32 values are kept in a
        pinned buffer from which K6 births the master copy at the first ADAM."""
        cs, ex = self.sim.chunk_set, self.executor
        cap = cs.capacity_elems
        staging32 = torch.empty(cap, dtype=torch.float32, device=self.device)
        staging16 = torch.empty(cap, dtype=self.dtype, device=self.device)
        gen = torch.Generator(device=self.device)
        for pos in self.sim.local:
            chunk = cs.param_chunk(pos)
            items = []
            for t in chunk.tensors:
                gen.manual_seed(seed * 1_000_003 + t.tensor_id)
                sl = staging32[t.offset_elems:t.offset_elems + t.numel]
                sl.normal_(0.0, 0.02, generator=gen)
                items.append((staging16, t.offset_elems, sl, t.numel))
            K.cast_pack(items)
            host16 = torch.empty(cap, dtype=self.dtype, pin_memory=True)
            host32 = torch.empty(cap, dtype=torch.float32, pin_memory=True)
            host16.copy_(staging16)
            host32.copy_(staging32)
            ex.seed_host_payload(chunk, host16)
            ex.init32[pos] = host32
        n_chunked = len(self.shapes)
        # wte (seed n), wpe (n+1) and an untied head (n+2): the same values
        # wherever the embedding is placed
        if self.host_embedding is not None:
            w = []
            for k, shape in enumerate([(self.schema.vocab, self.schema.hidden_dim),
                                       (self.schema.seq_len, self.schema.hidden_dim)]):
                gen.manual_seed(seed * 1_000_003 + n_chunked + k)
                w.append(torch.empty(shape, device=self.device).normal_(0.0, 0.02,
                                                                        generator=gen))
            self.host_embedding.load(*w)
            del w
            for p in self.host_embedding.device_params:  # wte: the HBM copy the GPU reads
                p.data = self.host_embedding.wte.to(self.device)
        for k, (p, master, m, v) in zip(self._emb_seed_offsets, emb):
            gen.manual_seed(seed * 1_000_003 + n_chunked + k)
            master.normal_(0.0, 0.02, generator=gen)
            p.data = torch.empty(master.shape, dtype=self.dtype, device=self.device)
            K.cast_pack([(p.data.view(-1), 0, master.view(-1), master.numel())])
        torch.cuda.synchronize(self.device)

    # -- event plumbing ---------------------------------------------------------------------

    def _check(self) -> None:
        if self.sim.engine.iteration_failed:
            raise StepInfeasible(self._end_failed())

    def _end_failed(self, cause: Optional[BaseException] = None) -> IterationReport:
        """Close an infeasible iteration: its report is recorded, the
        host-side work it started is joined, the trainer is marked failed."""
        eng = self.sim.engine
        if cause is not None:
            eng.fail_iteration(GPU)
        try:
            self.executor.join_host_work()
        except Exception:
            pass
        report = eng.end_iteration()
        self.reports.append(report)
        self.failed = report
        return report

    def _on_start(self, idx: int) -> None:
        if self.nvtx:  # one NVTX range per timeline event (SURVEY §5 tracing)
            torch.cuda.nvtx.range_push(self._events[idx].name)
        self.sim.engine.start_event(self._events[idx])
        self._check()

    def _on_finish(self, idx: int) -> None:
        self.sim.engine.finish_event(self._events[idx])
        self._check()
        if self.nvtx:
            torch.cuda.nvtx.range_pop()

    # -- the step -----------------------------------------------------------------------------

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        """One training iteration on device-resident tokens [B, S+1] (int64).

        Returns the (unscaled) loss as a device scalar; no host sync."""
        if self._graph is not None:
            return self._replay(tokens)
        if self._side is not None:           # workspaces exist on the capture stream
            return self._capture(tokens)
        if self.cuda_graph and self._graph_ready():
            # this iteration runs eagerly on the future capture stream so that
            # cuBLAS / cuDNN workspaces exist there; the next one is captured
            self._side = torch.cuda.Stream(self.device)
            self._side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(self._side):
                loss = self._eager_step(tokens)
            torch.cuda.current_stream(self.device).wait_stream(self._side)
            return loss
        return self._eager_step(tokens)

    def _eager_step(self, tokens: torch.Tensor) -> torch.Tensor:
        if self.failed is not None:
            raise RuntimeError("iteration %d was infeasible (%s); this run cannot continue"
                               % (self.failed.iteration, self.failed.failure_reason))
        eng = self.sim.engine
        warm = self.iteration == 0
        eng.begin_iteration(self.iteration, warm,
                            self.sim._plan_builder() if warm else None, self.sim.local)
        self._check()
        he = self.host_embedding
        if he is not None and he.h2d_done is not None:  # last ADAM's weights have landed
            torch.cuda.current_stream(self.device).wait_event(he.h2d_done)
        try:
            t0 = time.perf_counter()
            inp, tgt = tokens[:, :-1], tokens[:, 1:]
            loss = self.model(inp, tgt)
            t1 = time.perf_counter()
            (loss * self.executor.state.loss_scale()).backward()
            t2 = time.perf_counter()
            adam = self._events[-1]
            if self.nvtx:
                torch.cuda.nvtx.range_push(adam.name)
            eng.start_event(adam)
            self._check()
            eng.finish_event(adam)
            self._check()
            if self.nvtx:
                torch.cuda.nvtx.range_pop()
        except torch.OutOfMemoryError as e:
            # a physical allocation failed outside the engine's hooks (the
            # model's activations): the same verdict at the current moment
            raise StepInfeasible(self._end_failed(e), e) from None
        ph = self.phase_seconds  # host time per phase (enqueue + any blocking waits)
        ph["fwd"] += t1 - t0
        ph["bwd"] += t2 - t1
        ph["adam"] += time.perf_counter() - t2
        report = eng.end_iteration()
        self.reports.append(report)
        if warm:
            self.executor.end_of_warmup()
            if self.tracer is not None:
                self.tracer.freeze()
        else:  # the schedule is at its fixed point: prefetch next iteration's moves
            self.executor.prefetch_depth = self.prefetch_depth
            self.executor.gather_depth = self.gather_depth
            self.executor.set_prefetch_schedule(
                report.transfers, report.samples, self.sim.pools[GPU].capacity_bytes,
                self._events[-1].index)
        self.iteration += 1
        return loss.detach()

    # -- CUDA-graph steady state ---------------------------------------------------------
    #
    # Once the schedule has reached its fixed point (the reference's measured
    # iterations are identical, `tests/test_engine.py:121-129`) and it moves
    # no chunk (all-resident, single rank), the whole iteration — forward,
    # backward, K2, step scalars, K1 — is captured once and replayed.  The
    # decision engine still runs every iteration, in accounting-only mode on
    # the host while the GPU replays, so every iteration keeps its ledger.

    @staticmethod
    def _ledger_key(r: IterationReport):
        return ([(t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason) for t in r.transfers],
                [(c.group_id, c.kind, c.bytes) for c in r.collectives])

    def _graph_ready(self) -> bool:
        if (self.nproc != 1 and not self.graph_multi_rank) or len(self.reports) < 3:
            return False
        a, b = self.reports[-2], self.reports[-1]
        if a.warmup or self._ledger_key(a) != self._ledger_key(b):
            return False
        moves = [t for t in b.transfers if t.chunk_id != "embedding"]
        plan = self.sim.engine.plan
        return (not moves and plan is not None and self.host_embedding is None
                and len(plan.os_positions_on_gpu) == len(self.sim.local)
                and self.executor.stats.host_adam_items == 0)

    def _capture(self, tokens: torch.Tensor) -> torch.Tensor:
        """Capture THIS iteration (the graph records, it does not run), then
        replay it once: still exactly one training iteration per call."""
        from . import _native
        ex = self.executor
        record = ex.record_k1
        self.graph_k1 = None
        self._static_tokens = tokens.clone()
        torch.cuda.synchronize(self.device)
        graph = torch.cuda.CUDAGraph()
        n0 = _native.launch_count()
        ex.record_k1, n_ev = True, len(ex.k1_events)
        # no cyclic GC inside the capture: collecting an unrelated dead object
        # that owns CUDA resources (another trainer's events, graphs, pinned
        # buffers) would issue CUDA calls that invalidate a global-mode capture
        gc_was_enabled = gc.isenabled()
        gc.collect()
        gc.disable()
        try:
            with torch.cuda.graph(graph, stream=self._side):
                self._static_loss = self._eager_step(self._static_tokens)
        finally:
            if gc_was_enabled:
                gc.enable()
        self.graph_kernels_per_step = _native.launch_count() - n0
        # event-record nodes of the graph reference these events: they live with it
        self._graph_events = ex.k1_events[n_ev:]
        del ex.k1_events[n_ev:]
        if self._graph_events:  # K1's event-record nodes, re-recorded by every replay
            self.graph_k1 = self._graph_events[-1]
        ex.record_k1 = record
        self._graph = graph
        self._captured_key = self._ledger_key(self.reports[-1])
        # from here on the engine runs detached from the executor
        self.sim.manager.backend = None
        self.sim.dp.backend = None
        self.sim.engine.executor = None
        graph.replay()  # the captured iteration, now physically executed
        return self._static_loss.clone()

    def _replay(self, tokens: torch.Tensor) -> torch.Tensor:
        if tokens.data_ptr() != self._static_tokens.data_ptr():
            self._static_tokens.copy_(tokens, non_blocking=True)
        self._graph.replay()
        eng = self.sim.engine
        report = eng.run_iteration(self.iteration, warmup=False,
                                   local_positions=self.sim.local)
        if not report.feasible or self._ledger_key(report) != self._captured_key:
            raise RuntimeError("schedule left its fixed point under CUDA-graph replay "
                               "(iteration %d)" % self.iteration)
        self.reports.append(report)
        self.iteration += 1
        return self._static_loss.clone()

    def step_host(self, tokens_host: torch.Tensor) -> float:
        """End-to-end step from host memory: H2D tokens, step, D2H loss."""
        return self.step_host_async(tokens_host).result()

    def step_host_async(self, tokens_host: torch.Tensor) -> "PendingLoss":
        """`step_host` without waiting for the loss: H2D tokens (pinned host
        memory; the caller keeps the buffer unchanged until the step has run),
        enqueue the step, and a D2H of its loss into pinned memory whose
        ``result()`` blocks only for that copy.  A training loop that reads
        step k's loss after enqueueing step k+1 keeps the GPU busy across the
        step boundary (the host's accounting and launch overlap the device)."""
        if self._graph is not None:  # land straight in the graph's input buffer
            self._static_tokens.copy_(tokens_host, non_blocking=True)
            loss = self.step(self._static_tokens)
        else:
            tokens = tokens_host.to(self.device, non_blocking=True)
            if self.host_embedding is not None and not self.host_embedding.device_compute:
                # the host lookup reads these, no D2H
                self.host_embedding.host_tokens = tokens_host[:, :-1]
            loss = self.step(tokens)
        return PendingLoss(loss)

    def finish_host_work(self) -> None:
        """Wait for the host-side work a step may leave running (the async
        host Adam of CPU-placed positions and its deferred H2D issues); GPU
        work is stream-ordered behind it.  Call before timing the end of a
        run or inspecting host payloads directly.  The current stream then
        also waits for the copy streams (the deferred H2Ds of those updates)."""
        ex = self.executor
        ex.join_host_work()
        cur = torch.cuda.current_stream(self.device)
        for s in {ex.copy_stream, ex.d2h_stream}:
            cur.wait_stream(s)

    def close(self) -> None:
        """Drop the hook references that tie the model to the trainer, so the
        payloads are freed deterministically rather than by the cycle GC."""
        self.model.driver.on_start = self.model.driver.on_finish = None
        self._graph = None

    # -- inspection -----------------------------------------------------------------------------

    def write_ledgers(self, out_dir: str) -> List[str]:
        """The real run's layout / moments / transfers / collectives CSVs and
        summary in the reference's wire format (:mod:`.ledgers`)."""
        from . import ledgers
        return ledgers.write_ledgers(out_dir, self.reports, self.sim.chunk_set.layout_rows(),
                                     self.sim.engine.plan)

    def ledger_rows_not_realized(self, report: Optional[IterationReport] = None) -> Dict[str, int]:
        """Bytes per step the ledger bills that this run does not physically
        move.  Only the embedding's rows can be: the reference bills a
        GPU-placed embedding as weights down at FWD and weight gradients up
        at BWD (`engine.py:214-219`) because its fp16 weights live in host
        memory (`chunks.py:204-224`, `scenario.py:133`); here a GPU-computed
        embedding keeps weights, gradients and optimizer state resident in
        HBM by default (charged to the GPU pool, ``gpu_resident_bytes``), so
        those rows have no copy behind them; ``embedding_weights="host"``
        realises them (host-resident state, one weight H2D and one gradient
        D2H per step).  A CPU-computed embedding ships exactly the activation
        rows it is billed (realized)."""
        r = report if report is not None else (self.reports[-1] if self.reports else None)
        if r is None:
            return {}
        emb = sum(t.bytes for t in r.transfers if t.chunk_id == "embedding")
        realized = (self.embedding_placement == self.sim.engine.embedding_device
                    and (self.embedding_placement == CPU or self.embedding_weights == "host"))
        return {} if realized or emb == 0 else {"embedding": emb}

    def step_state(self):
        return self.executor.state.read()

    def local_chunk_payload(self, position: int, kind: ChunkKind = ChunkKind.PARAM_FP16,
                            used_only: bool = True):
        """The current payload (device preferred) of a local chunk position:
        its used prefix [0, used_elems) — the tensors packed into it — or,
        with ``used_only=False``, the full capacity (the tail past the last
        tensor is unspecified padding)."""
        chunk = self.sim.chunk_set.chunk_at(kind, position)
        ex = self.executor
        for dev in ("gpu", "cpu"):
            if ex.has(chunk, dev):
                t = ex.tensor(chunk, dev)
                return t[:chunk.used_elems] if used_only else t
        return None
