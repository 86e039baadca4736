"""Payload executor: the physical side of the chunk-managed step on B200.

The accounting core (memory / parallel / engine) decides; this class makes
each decision real at the moment it is taken:

====================================  =====================================================
reference accounting site             realisation here
====================================  =====================================================
``fetch_chunk`` / ``_evict_one``      ``copy``: cudaMemcpyAsync H2D/D2H of the whole chunk
(`memory.py:207-221, 277-301`)        payload on a copy stream per direction between pinned
                                      host slabs and HBM slabs (:mod:`.slabs`); the compute
                                      stream waits on the copy's event only when the chunk
                                      is next *used*; fetches are prefetched from the
                                      previous iteration's ledger
``place_payload`` / lazy OS birth     ``materialize``: an (uninitialised) payload born on
(`memory.py:223-231`,                 the device; lazy optimizer state is initialised by
`engine.py:234-240`)                  K6 ``cs_master_init`` reading the pinned fp32 init
``release_chunk`` / ``note_write``    ``drop``: the payload is freed and every parameter
                                      view into it is unbound
``DpRuntime`` gather / reduce-scatter  NCCL ``all_gather_into_tensor`` into a p×cap group
(`parallel.py:196-264`)               slab (remote members become views of their slot) and
                                      ``reduce_scatter_tensor(AVG)`` of the group's grads
``Engine._compute_event``             parameter ``.data`` re-pointed at the chunk slot
(`engine.py:164-179`)                 before the operator runs
``Engine._adam_event``                K2 grad sum-of-squares → device step scalars
(`engine.py:225-272`)                 (clip / found-inf / loss scale) → ONE K1
                                      ``cs_adam_chunks`` launch over every GPU-placed local
                                      position (+ the non-chunked GPU parameters); host K1
                                      for CPU-placed ones on a worker thread, whose
                                      ``adam_copy`` H2D follows each update
====================================  =====================================================

Chunk payloads are flat tensors of the chunk's full capacity (the reference
charges full capacity, `chunks.py:99-102`).  HBM payloads are slabs of the
stream-ordered :class:`.slabs.SlabPool` (backed by PyTorch's caching
allocator, compute-stream pool), host payloads come from its pinned caching
host allocator.
"""

import os
import threading
import time
from concurrent.futures import Future
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Set, Tuple

import torch
import torch.distributed as dist

from . import kernels as K
from .chunks import Chunk, ChunkKind, ChunkSet
from .engine import StepExecutor
from .memory import PayloadBackend
from .model import CPU, GPU
from .parallel import CollectiveBackend, CommGroup, DpPartition
from .slabs import SlabPool
from .gpt import grad_in_data, mark_grad_in_data


class ChunkComm:
    """Chunk-group collectives for one rank (device-agnostic plumbing over
    ``torch.distributed``: NCCL over NVLink on the B200 box, gloo in the CPU
    tests).  Buffers follow NCCL's layout: slot k of a p×cap group buffer is
    rank k's chunk, which is exactly the group's position g·p+k
    (`parallel.py:107-114`), so no reordering copy is ever needed."""

    def __init__(self, group: Optional["dist.ProcessGroup"] = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.calls: List[Tuple[str, int]] = []

    def all_gather_slab(self, slab: torch.Tensor, async_op: bool = False,
                        src: Optional[torch.Tensor] = None):
        """Gather every rank's chunk into ``slab``.  This rank's contribution
        is ``src`` (out of place: NCCL places it in slot ``rank`` itself, no
        staging copy), or slot ``rank`` of ``slab`` when ``src`` is None (in
        place).  With ``async_op`` returns the Work; ``work.wait()`` orders
        the caller's current stream after it (no host wait on NCCL)."""
        cap = slab.numel() // self.world
        mine = slab[self.rank * cap:(self.rank + 1) * cap] if src is None else src[:cap]
        self.calls.append(("all_gather", slab.numel() * slab.element_size()))
        return dist.all_gather_into_tensor(slab, mine, group=self.group, async_op=async_op)

    def reduce_scatter_avg(self, out: torch.Tensor, slab: torch.Tensor, async_op: bool = False):
        self.calls.append(("reduce_scatter", slab.numel() * slab.element_size()))
        return dist.reduce_scatter_tensor(out, slab, op=dist.ReduceOp.AVG, group=self.group,
                                          async_op=async_op)

    def all_reduce_sum(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def check(self) -> None:
        """Failure detection: torch's NCCL process group surfaces
        asynchronous collective errors from its own watchdog (it aborts the
        communicator and raises at the next call), so there is nothing to
        poll here; :class:`.native_comm.NativeChunkComm` polls
        ncclCommGetAsyncError itself."""

    def all_reduce_avg(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, op=dist.ReduceOp.AVG, group=self.group)


def plan_early_fetches(fetches, used, capacity: int, margin: int, adam_index: int,
                       last_event: int) -> Dict[int, List[int]]:
    """Events at which to issue ADAM's fetches ahead of the ledger.

    ``fetches``: (chunk id, bytes) in the ADAM walk's order; ``used``:
    (moment, GPU pool bytes in use) of the last iteration's samples (the grid
    puts moment 2e before event e and 2e+1 during it, `model.py:209-214`).
    Fetch j, with cumulative bytes B_j, goes before the earliest event e whose
    usage from moment 2e up to the moment before ADAM (2 * adam_index) stayed
    at most capacity - margin - B_j: holding every earlier-issued fetch as
    well, nothing the last iteration used before ADAM would have been short
    of room.  ADAM's own moment is not counted: its usage already includes
    these fetches, and since the early ones are a prefix of the walk's
    fetches, the walk adopts all of them before it fetches anything else.
    Fetches that would land after ``last_event`` (and every one after them:
    the walk's order is kept) are left to the ordinary prefetch."""
    peak: Dict[int, int] = {}
    for m, b in used:
        peak[m] = max(peak.get(m, 0), b)
    if not peak or not fetches:
        return {}
    first = min(peak) // 2
    head: Dict[int, int] = {}  # capacity - margin - max usage over [2e, 2*adam_index]
    run = peak.get(2 * adam_index, 0)
    head[adam_index] = capacity - margin - run
    for e in range(adam_index - 1, first - 1, -1):
        run = max(run, peak.get(2 * e, 0), peak.get(2 * e + 1, 0))
        head[e] = capacity - margin - run
    out: Dict[int, List[int]] = {}
    cum, e = 0, first
    for cid, nbytes in fetches:
        cum += nbytes
        while e <= last_event and head[e] < cum:
            e += 1
        if e > last_event:
            break
        out.setdefault(e, []).append(cid)
    return out


class _PriorityWorker:
    """One host thread running host-Adam jobs, lowest position first among
    the jobs whose inputs are ready.

    Jobs of CPU-placed positions are submitted in two orders: speculative
    updates during the backward, as each position's gradients become final
    (highest position first: the backward walks the layers in reverse), and
    the ADAM walk's in-place updates and settles (ascending).  The host
    enqueues the backward far ahead of the device, so a speculative job is
    submitted long before its gradients have landed in host memory: each job
    may carry a ``ready`` predicate (its D2H event has completed), and the
    worker picks the lowest position among ready jobs — during the backward
    that is whichever position the device has just finished, at ADAM it is
    the position the next forward needs first.  A running job is not
    preempted.  Futures follow concurrent.futures semantics (``cancel()``
    succeeds while the job is still queued)."""

    POLL_S = 1e-3

    def __init__(self):
        self._jobs: List[list] = []  # [priority, seq, future, fn, args, ready]
        self._cv = threading.Condition()
        self._seq = 0
        self._stop = False
        self._thread = threading.Thread(target=self._loop, name="cs-host-adam", daemon=True)
        self._thread.start()

    def submit(self, priority: int, fn, *args, ready=None) -> Future:
        fut: Future = Future()
        with self._cv:
            self._jobs.append([priority, self._seq, fut, fn, args, ready])
            self._seq += 1
            self._cv.notify()
        return fut

    def _pick(self):
        best = None
        for j in self._jobs:
            if j[2].cancelled():
                continue
            if j[5] is not None and not j[5]():
                continue
            if best is None or (j[0], j[1]) < (best[0], best[1]):
                best = j
        return best

    def _loop(self) -> None:
        while True:
            with self._cv:
                while True:
                    if self._stop:
                        return
                    self._jobs = [j for j in self._jobs if not j[2].cancelled()]
                    job = self._pick()
                    if job is not None:
                        self._jobs.remove(job)
                        break
                    # nothing ready: wait for a submission, or poll readiness
                    self._cv.wait(self.POLL_S if self._jobs else None)
            _, _, fut, fn, args, _ = job
            job = None  # no reference to the job's buffers while idle
            if not fut.set_running_or_notify_cancel():
                continue
            try:
                fut.set_result(fn(*args))
            except BaseException as e:  # delivered to whoever joins the job
                fut.set_exception(e)
            fut = fn = args = None

    def shutdown(self) -> None:
        with self._cv:
            self._stop = True
            self._cv.notify()


class _HostAdamJob:
    """One CPU-placed position's host Adam, run by the executor's worker
    thread; the param chunk's ``adam_copy`` H2D (`engine.py:265-267`) is
    issued by whichever thread comes second: the worker right after the
    update, or the main thread if the update already finished."""

    def __init__(self, cids):
        self.cids = tuple(cids)
        self.lock = threading.Lock()
        self.adam_done = False
        self.h2d = None            # deferred (chunk id, dst tensor, prior event)
        self.future: Optional[Future] = None


@dataclass
class ExecStats:
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    copies: int = 0
    gathers: int = 0
    reduce_scatters: int = 0
    adam_launch_items: int = 0
    host_adam_items: int = 0
    prefetch_issued: int = 0
    prefetch_hits: int = 0
    prefetch_discarded: int = 0
    prefetch_discarded_bytes: int = 0
    early_drains: int = 0
    gather_prefetch_issued: int = 0
    gather_prefetch_hits: int = 0
    host_adam_seconds: float = 0.0
    spec_issued: int = 0
    spec_committed: int = 0
    spec_discarded: int = 0
    spec_cancelled: int = 0
    adam_prefetch_early: int = 0
    adam_prefetch_oom: int = 0
    preevict_issued: int = 0
    preevict_hits: int = 0
    preevict_discarded: int = 0
    preevict_discarded_bytes: int = 0
    copy_events: List[Tuple[str, int, "torch.cuda.Event", "torch.cuda.Event"]] = field(
        default_factory=list)


class ChunkPayloadExecutor(PayloadBackend, CollectiveBackend, StepExecutor):
    """Owns every chunk payload of one rank and realises the engine's decisions."""

    def __init__(self, device: torch.device, dtype: torch.dtype, hyper: K.AdamHyper,
                 init_loss_scale: float = 1.0, dynamic_loss_scale: bool = False,
                 max_grad_norm: float = 0.0, comm: Optional[ChunkComm] = None,
                 host_threads: int = 0, time_copies: bool = False):
        if dtype not in (torch.float16, torch.bfloat16):
            raise TypeError("chunk dtype must be float16 or bfloat16")
        self.device = torch.device(device)
        self.dtype = dtype
        self.hyper = hyper
        self.dynamic_loss_scale = dynamic_loss_scale
        self.max_grad_norm = max_grad_norm
        self.comm = comm
        self.host_threads = host_threads
        #: OpenMP team of the host Adam jobs on the worker thread: they run
        #: while the main thread enqueues the step (the backward under
        #: speculation, the next forward otherwise), and a team as wide as the
        #: machine time-slices that Python thread off its core — the device
        #: then starves (measured: a 130 ms backward stretched to 300-500 ms
        #: with 16 threads on the 16-core box).  A quarter of the cores (at
        #: least two) stay with the main thread and the CUDA driver; the memory-bound update loses nothing
        #: (14 vs 16 threads: 5.7 vs 5.2 Gelem/s, profiles/r01/offload_host_threads.jsonl;
        #: all-host 1B step with speculation: 12 threads 281-287 ms, 14 threads
        #: 304-315 ms, profiles/r02/offload_ab.jsonl)
        ht = host_threads if host_threads > 0 else K.host_threads(0)
        reserve = max(2, ht // 4) if ht >= 8 else (1 if ht >= 4 else 0)
        self.worker_threads = int(os.environ.get("CS_WORKER_THREADS", "0")) or max(1, ht - reserve)
        self.time_copies = time_copies
        # test knob: every chunk move first spins this many cycles on its copy
        # stream, and an H2D destination reads NaN until the bytes land, so a
        # consumer not ordered after the move's event sees garbage
        self.copy_delay_cycles = 0
        self._setup_device(init_loss_scale)
        self.payload: Dict[str, Dict[int, torch.Tensor]] = {GPU: {}, CPU: {}}
        self.ready: Dict[Tuple[int, str], torch.cuda.Event] = {}
        self.stats = ExecStats()
        self._retain_req: Set[Tuple[int, str]] = set()
        self._retained: Dict[Tuple[int, str], torch.Tensor] = {}
        self._awaiting_gather: Set[int] = set()
        self._group_slab: Dict[int, torch.Tensor] = {}
        # collectives in flight: chunk id -> Work its payload depends on;
        # Works (with the buffers they use) not yet waited for
        self._coll_work: Dict[int, object] = {}
        self._inflight: List[Tuple[object, Tuple[torch.Tensor, ...]]] = []
        self._gather_log: List[Tuple[int, int]] = []        # (event, group) this iteration
        self._gather_sched: Dict[int, List[int]] = {}       # event -> groups (last iteration)
        self._gather_prefetched: Dict[int, Tuple[torch.Tensor, object]] = {}
        self._cur_event = -1
        self.overlap_collectives = True
        self.gather_depth = 0
        self._pending: List[Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, int]] = []
        self._pending_ids: Set[int] = set()
        self._prefetched: Dict[int, Tuple[torch.Tensor, "torch.cuda.Event"]] = {}
        self._predrained: Dict[int, Tuple[torch.Tensor, "torch.cuda.Event"]] = {}
        self._prefetch_sched: Dict[int, List[int]] = {}
        self.prefetch_depth = 0
        #: ADAM-time fetches issued during the backward, as early as the last
        #: iteration's per-moment GPU usage leaves room for them (event -> ids)
        self._adam_prefetch_at: Dict[int, List[int]] = {}
        #: bytes of HBM left unplanned when placing those early fetches
        self.adam_prefetch_margin = float(os.environ.get("CS_ADAM_PREFETCH_MARGIN", "0.03"))
        self.early_adam_prefetch = os.environ.get("CS_EARLY_ADAM_PREFETCH", "1") != "0"
        #: pre-eviction: an optimizer-state chunk the last iteration evicted
        #: during FWD/BWD is only ever written by K1, so its D2H can start
        #: right after this ADAM's K1 -- when the D2H direction is idle (ADAM
        #: fetches saturate H2D) -- instead of at the eviction moment in the
        #: next forward, where the activations are waiting for its HBM.  The
        #: accounting's eviction then adopts the landed host copy
        self.preevict = os.environ.get("CS_PREEVICT", "1") != "0"
        self._preevict_ids: Set[int] = set()
        self._preevicted: Dict[int, Tuple[torch.Tensor, "torch.cuda.Event"]] = {}
        #: with pre-evictions pending, K1 launches every this many positions
        #: so their D2Hs start during the ADAM walk
        self.preevict_batch = 4
        self._plan = None
        self._host_state = None
        self._state_snap = None
        self._keepalive: List[torch.Tensor] = []  # pinned inits K6 may still be reading
        #: run host Adam of CPU-placed positions on a worker thread, overlapping
        #: the main thread's enqueue of the rest of the step and the next
        #: forward (bit-identical).  12B with 58 host-placed positions: 2.05-2.62
        #: vs 2.28-2.81 s/step; 1B with every triplet on the host: within noise
        #: (the host Adam slows down by what it overlaps).  CS_ASYNC_HOST_ADAM=0
        #: restores the synchronous walk.
        self.async_host_adam = os.environ.get("CS_ASYNC_HOST_ADAM", "1") != "0"
        self._worker: Optional[_PriorityWorker] = None
        #: speculative host Adam: once a CPU-placed position's gradients are
        #: final and drained (see ``early_drain``) its update starts on the
        #: worker during the rest of the backward, out of place into shadow
        #: buffers (cs_adam_chunks_host_oop), with the step scalars
        #: cs_adam_prepare will produce if the step is finite and unclipped
        #: (``kernels.speculate_step_scalars``, bit-exact).  At the position's
        #: ADAM turn a settle job (same priority) adopts the shadows if the real
        #: scalars are those bits (pointer swap), else runs the normal update
        #: from the intact inputs; an update not started yet is cancelled and
        #: replaced by the normal one.  Bit-identical to the non-speculative
        #: walk; off when gradients are clipped (the coefficient needs every
        #: gradient).  Shadow buffers are bounded by ``spec_budget_bytes``.
        self.speculative_host_adam = os.environ.get("CS_SPEC_HOST_ADAM", "1") != "0"
        self.spec_budget_bytes = int(float(os.environ.get("CS_SPEC_HOST_GB", "16")) * 2**30)
        self._spec: Dict[int, tuple] = {}        # position -> (future, d, ins, shadow)
        self._spec_free: List[tuple] = []        # recycled (p16, p32, m, v) host buffers
        self._spec_bytes = 0                     # pinned bytes held by shadow sets
        self._spec_state = None
        self._jobs: Dict[int, _HostAdamJob] = {}   # chunk id -> unfinished job
        #: drain a host-placed position's gradients D2H as soon as they are
        #: final (after its last BWD op; at p > 1 after its reduce-scatter),
        #: during the backward while host DRAM is otherwise idle, instead of at
        #: ADAM beside the host Adam; the accounting still bills the row at the
        #: position's ADAM turn (`engine.py:249-251`), where the copy is adopted
        self.early_drain = os.environ.get("CS_EARLY_DRAIN", "1") != "0"
        self._last_bwd_at: Optional[Dict[int, List[int]]] = None  # event -> positions
        self._drain_candidates: List[int] = []
        self._rs_out: Set[int] = set()  # local chunks whose reduce-scatter was issued
        #: in-step collective timing (bench at N > 1): every chunk-group
        #: collective's (kind, slab bytes, Work, start event) is logged; the
        #: duration is the Work's own (torch's NCCL with TORCH_NCCL_ENABLE_TIMING,
        #: the native communicator's comm-stream events), else issue -> done
        self.time_collectives = False
        self.coll_log: List[tuple] = []
        self._free_host: Dict[tuple, List[tuple]] = {}  # (dtype, numel) -> [(tensor, event)]
        self._free_host_bytes = 0
        #: pinned buffer (data_ptr) -> completion event of the last H2D that read it
        self._host_reads: Dict[int, "torch.cuda.Event"] = {}
        #: HBM slab (data_ptr) -> {side stream: completion event of its last copy there}
        self._side_use: Dict[int, Dict[int, "torch.cuda.Event"]] = {}
        self._host_read_events = os.environ.get("CS_HOST_READ_EVENTS", "1") != "0"
        self.nvtx = False  # NVTX ranges around chunk moves and collectives
        self._stats_lock = threading.Lock()
        #: CPU-placed embedding operator (embedding.HostEmbedding) or None
        self.host_embedding = None
        self._placeholder = torch.empty(0, dtype=dtype, device=self.device)
        self.chunk_set: Optional[ChunkSet] = None
        #: test hook: called as observer("pre"|"post", items) around each K1 launch
        self.adam_observer = None
        #: CUDA events bracketing every K1 launch (bench: in-region kernel timing)
        self.k1_events: List[Tuple["torch.cuda.Event", "torch.cuda.Event", int]] = []
        self.record_k1 = False

    def _setup_device(self, init_loss_scale: float) -> None:
        self.compute = torch.cuda.current_stream(self.device)
        # one copy stream per direction: PCIe is full duplex, so evictions
        # (D2H) and fetches (H2D) proceed concurrently
        self.copy_stream = torch.cuda.Stream(self.device)      # H2D
        self.d2h_stream = (self.copy_stream if os.environ.get("CS_COPY_STREAMS") == "1"
                           else torch.cuda.Stream(self.device))
        streams = [self.compute, self.copy_stream]
        if self.d2h_stream is not self.copy_stream:
            streams.append(self.d2h_stream)
        self.slabs = SlabPool(self.device, streams)
        self.state = K.StepState(self.device, init_loss_scale)
        # K2 (canonical per-item sums of squares): scratch partials, one
        # double per item slot on the device, and the host slots' values
        self._sq_scratch = torch.empty(0, device=self.device)
        self._sq_items = torch.empty(0, dtype=torch.float64, device=self.device)
        self._sq_host: Optional[torch.Tensor] = None
        self._sq_host_ev: Optional[torch.cuda.Event] = None

    # -- wiring -------------------------------------------------------------------

    def attach(self, chunk_set: ChunkSet, partition: DpPartition, rank: int,
               params: Sequence[torch.nn.Parameter], shapes: Sequence[Tuple[int, ...]],
               embedding: Sequence[Tuple[torch.nn.Parameter, torch.Tensor, torch.Tensor,
                                         torch.Tensor]] = (),
               embedding_keys: Optional[Sequence[int]] = None) -> None:
        """Bind the layout, this rank's partition and the model's parameters
        (``params[tid]`` has shape ``shapes[tid]``); ``embedding`` lists the
        non-chunked (param, master, m, v) quadruples updated in the same K1,
        ``embedding_keys`` their place in K2's canonical order (wte 0, wpe 1,
        untied head 2; default: list order)."""
        self.chunk_set, self.partition, self.rank = chunk_set, partition, rank
        self.params, self.shapes = list(params), list(shapes)
        self.offsets = chunk_set.element_offsets()
        self.embedding = list(embedding)
        self.embedding_keys = (list(embedding_keys) if embedding_keys is not None
                               else list(range(len(self.embedding))))
        self._bound: Dict[int, int] = {}  # tid -> chunk id its .data views
        self.init32: Dict[int, torch.Tensor] = {}

    def _is_remote_param(self, chunk: Chunk) -> bool:
        return (chunk.list_kind is ChunkKind.PARAM_FP16
                and self.partition.owner_of_position(chunk.position) != self.rank)

    def _elem_dtype(self, chunk: Chunk) -> torch.dtype:
        return self.dtype if chunk.list_kind is ChunkKind.PARAM_FP16 else torch.float32

    def _alloc(self, chunk: Chunk, device: str) -> torch.Tensor:
        if device == GPU:
            return self.slabs.take(chunk.capacity_elems, self._elem_dtype(chunk), self.compute)
        return torch.empty(chunk.capacity_elems, dtype=self._elem_dtype(chunk), pin_memory=True)

    # -- pinned host buffers as D2H destinations ------------------------------------
    #
    # A dropped host payload (e.g. a host-placed position's parameters, dropped
    # when the backward overwrites them with gradients) is kept as the
    # destination of a later D2H (parameter chunks only: the gradient drains
    # and evictions land there) instead of going back to PyTorch's pinned
    # cache.  That cache only reuses a block once every copy recorded on it
    # has completed — and the host runs a step ahead of the device, so the
    # early gradient drains of the backward always found the previous step's
    # buffers still pending and fell through to cudaHostAlloc (~0.1 s for a
    # 128 MiB block, several per step, measured).  Here reuse is
    # stream-ordered instead: the buffer carries an event recorded on the H2D
    # copy stream when it was dropped (every copy that may still read it),
    # and the D2H stream waits on it before writing.  Only D2H destinations
    # are served this way (the host never writes these buffers before the
    # D2H that fills them has completed).

    #: pinned bytes kept for reuse; beyond it a dropped buffer goes back to
    #: PyTorch's pinned cache (the accounting's CPU pool no longer counts it)
    HOST_FREE_BYTES = int(float(os.environ.get("CS_HOST_FREE_GB", "8")) * 2**30)

    def _give_host(self, t: torch.Tensor, ev: Optional["torch.cuda.Event"] = None) -> None:
        """``ev``: the last device work on ``t`` (default: whatever the H2D
        stream has enqueued so far, i.e. every copy that may still read it)."""
        nbytes = t.numel() * t.element_size()
        if not t.is_pinned() or self._free_host_bytes + nbytes > self.HOST_FREE_BYTES:
            return
        lst = self._free_host.setdefault((t.dtype, t.numel()), [])
        if ev is None and self.copy_stream is not None:
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        lst.append((t, ev))
        self._free_host_bytes += nbytes

    def _alloc_d2h_dst(self, chunk: Chunk) -> torch.Tensor:
        """Pinned host destination of a D2H copy (see ``_give_host``)."""
        lst = self._free_host.get((self._elem_dtype(chunk), chunk.capacity_elems))
        if lst:
            t, ev = lst.pop()
            self._free_host_bytes -= t.numel() * t.element_size()
            if ev is not None:
                self.d2h_stream.wait_event(ev)
            return t
        return self._alloc(chunk, CPU)

    def _alloc_for_copy(self, chunk: Chunk) -> torch.Tensor:
        """HBM destination of an H2D copy, taken from the copy stream's pool so
        the copy need not wait for the compute stream; the compute stream is
        registered as a user (it consumes the payload after `wait_ready`)."""
        return self.slabs.take(chunk.capacity_elems, self._elem_dtype(chunk), self.copy_stream)

    def _side_events(self, t: torch.Tensor):
        return list(self._side_use.pop(t.data_ptr(), {}).values())

    def _release(self, cid: int, t: torch.Tensor) -> None:
        """A GPU payload leaves the executor: back to the slab pool once the
        work already enqueued on it (incl. a collective writing it) is done."""
        if cid in self._coll_work:
            self._wait_collective(cid)
        self.slabs.give(t, self._side_events(t))

    def tensor(self, chunk: Chunk, device: str) -> torch.Tensor:
        self._join(chunk.chunk_id)
        return self.payload[device][chunk.chunk_id]

    def has(self, chunk: Chunk, device: str) -> bool:
        return chunk.chunk_id in self.payload[device]

    def seed_host_payload(self, chunk: Chunk, data: torch.Tensor) -> None:
        """Initial CPU payload of a chunk registered with a CPU copy."""
        assert not data.is_cuda and data.is_pinned()
        self.payload[CPU][chunk.chunk_id] = data

    # -- stream ordering ------------------------------------------------------------

    def _wait_collective(self, cid: int) -> None:
        work = self._coll_work.pop(cid, None)
        if work is not None:
            work.wait()  # the current stream waits for the collective

    def wait_collectives(self) -> None:
        """Order the current stream after every collective still in flight."""
        for work, _ in self._inflight:
            work.wait()
        self._inflight.clear()
        self._coll_work.clear()

    def _join(self, cid: int) -> None:
        """Block until the host Adam job touching chunk ``cid`` (and its
        deferred H2D issue) is done."""
        job = self._jobs.get(cid)
        if job is None:
            return
        job.future.result()
        for c in job.cids:
            if self._jobs.get(c) is job:
                del self._jobs[c]

    def join_host_work(self) -> None:
        for cid in list(self._jobs):
            self._join(cid)

    def wait_ready(self, chunk: Chunk, device: str) -> None:
        self._join(chunk.chunk_id)
        if device == GPU:
            self._wait_collective(chunk.chunk_id)
        ev = self.ready.pop((chunk.chunk_id, device), None)
        if ev is None:
            return
        if device == GPU:
            self.compute.wait_event(ev)
        else:
            ev.synchronize()

    # -- PayloadBackend ------------------------------------------------------------------

    def copy(self, chunk: Chunk, src: str, dst: str, moment: int, reason: str) -> None:
        job = self._jobs.get(chunk.chunk_id)
        if job is not None and src == CPU and dst == GPU:
            if self._defer_h2d(job, chunk):
                return
        self._join(chunk.chunk_id)
        if chunk.chunk_id in self._pending_ids:
            self._flush_adam()  # the move must carry post-update bytes
        if src == GPU and chunk.chunk_id in self._awaiting_gather:
            raise RuntimeError("chunk %d moved before its gather landed" % chunk.chunk_id)
        if dst == CPU and chunk.chunk_id in self._prefetched:
            self._discard_prefetch(chunk)
        if dst == GPU:
            hit = self._prefetched.pop(chunk.chunk_id, None)
        else:
            hit = self._predrained.pop(chunk.chunk_id, None)
            if hit is None:
                hit = self._preevicted.pop(chunk.chunk_id, None)
                if hit is not None:  # moved bytes are counted when adopted
                    self.stats.preevict_hits += 1
                    self.stats.d2h_bytes += hit[0].numel() * hit[0].element_size()
        if hit is not None:  # issued ahead of time from the previous iteration's ledger
            d, done = hit
            self.stats.prefetch_hits += 1
        else:
            if src == GPU:  # a reduce-scatter may still be writing the payload
                self._wait_collective(chunk.chunk_id)
            s = self.payload[src][chunk.chunk_id]
            d = self._retained.pop((chunk.chunk_id, dst), None)
            if d is None:
                d = self._alloc_for_copy(chunk) if dst == GPU else self._alloc_d2h_dst(chunk)
            prior = self.ready.pop((chunk.chunk_id, src), None)
            done = self._transfer(s, d, src, dst, prior)
        if done is not None:
            self.ready[(chunk.chunk_id, dst)] = done
        self.payload[dst][chunk.chunk_id] = d

    def _defer_h2d(self, job: _HostAdamJob, chunk: Chunk) -> bool:
        """The updated params of a position whose host Adam is still running
        go H2D as soon as the update finishes (from the worker); False if it
        already finished (the caller copies now)."""
        cid = chunk.chunk_id
        d = self._alloc_for_copy(chunk)
        prior = self.ready.pop((cid, CPU), None)
        with job.lock:
            if job.adam_done:
                self._jobs.pop(cid, None)
                done = self._transfer(self.payload[CPU][cid], d, CPU, GPU, prior)
                if done is not None:
                    self.ready[(cid, GPU)] = done
                self.payload[GPU][cid] = d
                return True
            # the source is looked up when the job is done: a settled
            # speculative update swaps in its shadow buffer
            job.h2d = (cid, d, prior)
        self.payload[GPU][cid] = d
        return True

    def _job_done(self, job: _HostAdamJob) -> None:
        """The host update of ``job`` is complete: issue its deferred H2D."""
        with job.lock:
            job.adam_done = True
            h2d = job.h2d
            if h2d is not None:
                cid, d, prior = h2d
                done = self._transfer(self.payload[CPU][cid], d, CPU, GPU, prior)
                if done is not None:
                    self.ready[(cid, GPU)] = done

    def _run_host_adam(self, job: _HostAdamJob, item, state) -> None:
        t0 = time.perf_counter()
        K.adam_chunks_host([item], self.hyper, state, self.worker_threads)
        with self._stats_lock:
            self.stats.host_adam_seconds += time.perf_counter() - t0
        self._job_done(job)

    def _transfer(self, s: torch.Tensor, d: torch.Tensor, src: str, dst: str,
                  prior: Optional["torch.cuda.Event"], after=None, count: bool = True):
        """cudaMemcpyAsync of a whole payload on the copy stream of its
        direction; returns the completion event consumers wait on
        (`wait_ready`).  D2H waits for the compute stream (the payload must be
        final); H2D does not (its source is host data already final, its
        destination came from the H2D stream's pool).  A move that depends on
        an earlier one (a fetch of a chunk just evicted) waits on its event;
        ``after``: a collective Work still writing the source (a D2H of
        reduce-scattered gradients waits for it on the copy stream only)."""
        cs = self.d2h_stream if src == GPU else self.copy_stream
        if src == GPU:
            cs.wait_stream(self.compute)
        if prior is not None:
            cs.wait_event(prior)
        if self.nvtx:
            torch.cuda.nvtx.range_push("%s>%s %d B" % (src, dst, d.numel() * d.element_size()))
        with torch.cuda.stream(cs):
            if after is not None:
                after.wait()
            t0 = torch.cuda.Event(enable_timing=True) if self.time_copies else None
            if t0 is not None:
                t0.record(cs)
            if self.copy_delay_cycles:
                if dst == GPU:
                    d.fill_(float("nan"))
                torch.cuda._sleep(self.copy_delay_cycles)
            d.copy_(s, non_blocking=True)
            done = torch.cuda.Event(enable_timing=self.time_copies)
            done.record(cs)
        if self.nvtx:
            torch.cuda.nvtx.range_pop()
        if src == CPU:
            self._host_reads[s.data_ptr()] = done
        for t in ((s,) if src == GPU else ()) + ((d,) if dst == GPU else ()):
            if self.slabs.owns(t):  # handed back to the pool with the slab (``_release``)
                self._side_use.setdefault(t.data_ptr(), {})[id(cs)] = done
            else:
                t.record_stream(cs)
        with self._stats_lock:  # the host-Adam worker issues H2Ds too
            if src == GPU and count:
                self.stats.d2h_bytes += s.numel() * s.element_size()
            if dst == GPU and count:
                self.stats.h2d_bytes += d.numel() * d.element_size()
            if t0 is not None:
                self.stats.copy_events.append(("%s>%s" % (src, dst),
                                               d.numel() * d.element_size(), t0, done))
            self.stats.copies += 1
        return done

    # -- prefetch from the previous iteration's ledger (the warm-up trace) ---------
    #
    # The schedule reaches a fixed point after warm-up (identical ledgers per
    # measured iteration), so the fetches of the next events are known before
    # the accounting takes them.  Before event i, every CPU->GPU fetch the last
    # iteration made during events i+1 .. i+prefetch_depth is issued on the
    # copy stream if the chunk's host payload is final (the chunk is not on the
    # GPU and no host write can intervene before the fetch: prefetches never
    # cross the ADAM event, and any D2H into / drop of the host copy discards
    # them).  The accounting fetch then adopts the in-flight buffer.

    def set_prefetch_schedule(self, transfers, samples=None, gpu_capacity: int = 0,
                              adam_index: int = -1) -> None:
        """Prefetch plan for the next iteration from this one's ledger.
        ``adam_copy`` rows are never prefetched (their host source is what the
        host Adam writes).  With the per-moment samples and the GPU pool's
        capacity, ADAM's fetches are also placed early in the backward (see
        ``_plan_adam_prefetch``); evictions of optimizer-state chunks before
        ADAM become pre-evictions (``preevict``)."""
        sched: Dict[int, List[int]] = {}
        for t in transfers:
            if t.src == CPU and t.dst == GPU and isinstance(t.chunk_id, int) \
                    and t.reason != "adam_copy":
                sched.setdefault((t.moment - 1) // 2, []).append(t.chunk_id)
        self._prefetch_sched = sched
        self._preevict_ids = set()
        self._adam_prefetch_at = {}
        if adam_index < 0 or self.chunk_set is None:
            return
        adam_moment = 2 * adam_index + 1
        if self.preevict:
            for t in transfers:
                if (t.src == GPU and t.dst == CPU and t.reason == "evict" and t.bytes > 0
                        and isinstance(t.chunk_id, int) and t.moment < adam_moment
                        and self.chunk_set.chunks[t.chunk_id].list_kind
                        is not ChunkKind.PARAM_FP16):
                    self._preevict_ids.add(t.chunk_id)
        if self.early_adam_prefetch and samples and gpu_capacity > 0:
            self._plan_adam_prefetch(sched.get(adam_index, ()), samples, gpu_capacity,
                                     adam_index)

    def _plan_adam_prefetch(self, ids, samples, capacity: int, adam_index: int) -> None:
        """Move ADAM's fetches of GPU-placed positions (their host copies
        cannot change before ADAM) into the backward: ``plan_early_fetches``."""
        plan = self._plan
        if not ids or plan is None:
            return
        chunks = [self.chunk_set.chunks[cid] for cid in ids]
        fetches = [(c.chunk_id, c.bytes) for c in chunks
                   if plan.device_of_position(c.position) == GPU]
        used = [(smp.moment, smp.used_bytes) for smp in samples if smp.device == GPU]
        self._adam_prefetch_at = plan_early_fetches(
            fetches, used, capacity, int(self.adam_prefetch_margin * capacity), adam_index,
            adam_index - max(self.prefetch_depth, 1))

    def set_timeline(self, timeline) -> None:
        """Index the positions by their last BWD event (early gradient drain)."""
        last: Dict[int, int] = {}
        for e in timeline.events:
            if e.phase.value == "bwd":
                for tid in e.tensor_refs:
                    pos = self.offsets[tid][0]
                    last[pos] = max(last.get(pos, -1), e.index)
        by_event: Dict[int, List[int]] = {}
        for pos, e in last.items():
            by_event.setdefault(e, []).append(pos)
        self._last_bwd_at = by_event

    def _drain_early(self, ev) -> None:
        """D2H of host-placed positions' final gradients, ahead of ADAM."""
        if self._plan is None or self._last_bwd_at is None or ev.phase.value == "adam":
            return
        local = set(self.partition.local_positions(self.rank))
        for pos in self._last_bwd_at.get(ev.index - 1, ()):
            if pos in local and self._plan.device_of_position(pos) == CPU:
                self._drain_candidates.append(pos)
        if not self._drain_candidates:
            return
        multi = self.comm is not None and self.comm.world > 1
        keep = []
        for pos in self._drain_candidates:
            chunk = self.chunk_set.param_chunk(pos)
            cid = chunk.chunk_id
            if multi and cid not in self._rs_out:
                keep.append(pos)  # its group's reduce-scatter is not issued yet
                continue
            if not self.has(chunk, GPU) or self.has(chunk, CPU) or cid in self._predrained \
                    or cid in self._awaiting_gather:
                continue
            d = self._alloc_d2h_dst(chunk)
            done = self._transfer(self.tensor(chunk, GPU), d, GPU, CPU,
                                  self.ready.get((cid, GPU)), after=self._coll_work.get(cid))
            self._predrained[cid] = (d, done)
            self.stats.early_drains += 1
            self._speculate(pos, chunk, d, done)
        self._drain_candidates = keep

    # -- speculative host Adam (see ``speculative_host_adam``) ----------------------

    def _speculate(self, pos: int, chunk: Chunk, d: torch.Tensor, drained) -> None:
        if (not self.speculative_host_adam or not self.async_host_adam
                or self.max_grad_norm > 0 or self._state_snap is None or pos in self._spec):
            return
        triplet = self.chunk_set.os_triplet(pos)
        if any(not self.has(c, CPU) or c.chunk_id in self._jobs for c in triplet) \
                or chunk.chunk_id in self._jobs:
            return
        shadow = self._take_shadow(chunk, triplet)
        if shadow is None:
            return
        if self._spec_state is None:
            self._spec_state = K.speculate_step_scalars(
                K.StepState.from_snapshot(self._state_snap), self.hyper)
        n = chunk.used_elems
        ins = (d,) + tuple(self.payload[CPU][c.chunk_id] for c in triplet)
        waits = [drained] + [self.ready[(c.chunk_id, CPU)] for c in triplet
                             if (c.chunk_id, CPU) in self.ready]
        if self._worker is None:
            self._worker = _PriorityWorker()
        fut = self._worker.submit(pos, self._run_spec, waits, ins + (n,), shadow + (n,),
                                  self._spec_state,
                                  ready=lambda: all(ev.query() for ev in waits))
        self._spec[pos] = (fut, ins, shadow, self._spec_state)
        self.stats.spec_issued += 1

    def _take_shadow(self, chunk: Chunk, triplet) -> Optional[tuple]:
        if self._spec_free:
            return self._spec_free.pop()
        nbytes = chunk.capacity_elems * (2 + 12)
        if self._spec_bytes + nbytes > self.spec_budget_bytes:
            return None
        self._spec_bytes += nbytes
        return tuple(self._alloc(c, CPU) for c in (chunk,) + tuple(triplet))

    def _run_spec(self, waits, item_in, item_out, state) -> None:
        for ev in waits:
            ev.synchronize()
        t0 = time.perf_counter()
        K.adam_chunks_host_oop([item_in], [item_out], self.hyper, state, self.worker_threads)
        with self._stats_lock:
            self.stats.host_adam_seconds += time.perf_counter() - t0

    def _settle_spec(self, job: _HostAdamJob, spec, param: Chunk, triplet, state) -> None:
        """At the position's ADAM turn, on the worker: adopt the speculative
        update if it used this step's real scalars and the current payloads,
        else run the normal update from the (intact) inputs."""
        fut, ins, shadow, spec_state = spec
        fut.result()
        cpu = self.payload[CPU]
        cids = (param.chunk_id,) + tuple(c.chunk_id for c in triplet)
        ok = (K.same_update_scalars(spec_state, state)
              and all(cpu.get(cid) is t for cid, t in zip(cids, ins)))
        if ok:
            for cid, t in zip(cids, shadow):
                cpu[cid] = t
            self._spec_free.append(ins)
            with self._stats_lock:
                self.stats.spec_committed += 1
            self._job_done(job)
            return
        self._spec_free.append(shadow)
        with self._stats_lock:
            self.stats.spec_discarded += 1
        self._run_host_adam(job, tuple(cpu[cid] for cid in cids) + (param.used_elems,), state)

    def before_event(self, ev, iteration: int) -> None:
        self._cur_event = ev.index
        if self.early_drain:
            self._drain_early(ev)
        if self.comm is not None and self.comm.world > 1:
            self._prefetch_gathers(ev)
        if not self.prefetch_depth or not self._prefetch_sched:
            return
        for cid in self._adam_prefetch_at.get(ev.index, ()):
            try:
                if self._prefetch(cid):
                    self.stats.adam_prefetch_early += 1
            except torch.OutOfMemoryError:
                # the room the ledger promised is not there physically: this
                # chunk and the rest are fetched at ADAM as the ledger says
                self._adam_prefetch_at = {}
                self.stats.adam_prefetch_oom += 1
                break
        for j in range(ev.index + 1, ev.index + 1 + self.prefetch_depth):
            for cid in self._prefetch_sched.get(j, ()):
                self._prefetch(cid)

    def _prefetch(self, cid: int) -> bool:
        if cid in self._prefetched or cid in self.payload[GPU]:
            return False
        src = self.payload[CPU].get(cid)
        if src is None or cid in self._jobs:
            return False
        chunk = self.chunk_set.chunks[cid]
        d = self._alloc_for_copy(chunk)
        prior = self.ready.get((cid, CPU))
        done = self._transfer(src, d, CPU, GPU, prior)
        self._prefetched[cid] = (d, done)
        self.stats.prefetch_issued += 1
        return True

    def _discard_prefetch(self, chunk: Chunk) -> None:
        hit = self._prefetched.pop(chunk.chunk_id, None)
        if hit is not None:
            self.slabs.give(hit[0], self._side_events(hit[0]))
            self.stats.prefetch_discarded += 1
            self.stats.prefetch_discarded_bytes += hit[0].numel() * hit[0].element_size()

    def materialize(self, chunk: Chunk, device: str) -> None:
        key = (chunk.chunk_id, device)  # (no data access: a running host job may go on)
        t = self._retained.pop(key, None)
        if t is None and device == GPU and self._is_remote_param(chunk):
            self._awaiting_gather.add(chunk.chunk_id)  # the group slab will back it
            return
        self.payload[device][chunk.chunk_id] = t if t is not None else self._alloc(chunk, device)

    def drop(self, chunk: Chunk, device: str) -> None:
        cid = chunk.chunk_id
        job = self._jobs.get(cid)
        if job is not None:
            # a host job reads/writes the CPU payloads and, once deferred, the
            # H2D destination; a retained host payload keeps its job running
            if (device == CPU and (cid, CPU) not in self._retain_req) or \
                    (device == GPU and job.h2d is not None):
                self._join(cid)
        key = (cid, device)
        if device == CPU:
            self._discard_prefetch(chunk)
        t = self.payload[device].pop(cid, None)
        self._awaiting_gather.discard(cid)
        ev = self.ready.pop(key, None)
        if key in self._retain_req:
            self._retain_req.discard(key)
            if t is not None:
                if ev is not None:
                    self.ready[key] = ev
                self._retained[key] = t
                t = None
        if t is not None and device == CPU:
            # reusable once the last copy that read it has landed -- not the
            # H2D stream's tail, which at ADAM holds every fetch of the walk
            ev = self._host_reads.pop(t.data_ptr(), None)
            self._give_host(t, ev if self._host_read_events else None)
        if device == GPU:
            self._discard_preevict(cid)
        if t is not None and device == GPU:
            if cid in self._pending_ids:
                self._flush_adam()  # K1 must update this payload before it is recycled
            self._release(cid, t)
        if device == GPU and chunk.list_kind is ChunkKind.PARAM_FP16:
            for tmeta in chunk.tensors:
                if self._bound.get(tmeta.tensor_id) == cid:
                    self.params[tmeta.tensor_id].data = self._placeholder
                    del self._bound[tmeta.tensor_id]
            if self._is_remote_param(chunk):
                self._maybe_free_slab(chunk)

    def _maybe_free_slab(self, chunk: Chunk) -> None:
        gid = chunk.position // self.partition.nproc
        if gid not in self._group_slab:
            return
        group = self.partition.groups[gid]
        alive = any(self.chunk_set.param_chunk(p).chunk_id in self.payload[GPU]
                    for p in group.real_positions
                    if self.partition.owner_of_position(p) != self.rank)
        if not alive:
            del self._group_slab[gid]

    # -- CollectiveBackend -----------------------------------------------------------------

    def _group_slot(self, slab: torch.Tensor, k: int) -> torch.Tensor:
        cap = self.chunk_set.capacity_elems
        return slab[k * cap:(k + 1) * cap]

    def _issue_gather(self, group: CommGroup):
        """Fill this rank's slot of a fresh p×cap slab and all-gather it
        (async when overlapping: the compute stream waits only at use)."""
        cap, p = self.chunk_set.capacity_elems, self.partition.nproc
        slab = torch.empty(p * cap, dtype=self.dtype, device=self.device)
        mine = self._group_slot(slab, self.rank)
        pos = group.member_positions[self.rank]
        src = None
        if pos is None:
            mine.zero_()  # phantom slot of a padded tail group
        else:
            local = self.chunk_set.param_chunk(pos)
            if self.has(local, GPU):  # sent straight from the chunk (out of place)
                self.wait_ready(local, GPU)
                src = self.tensor(local, GPU)
            else:  # local payload lives on the host: stage it into our slot
                self.wait_ready(local, CPU)
                mine.copy_(self.tensor(local, CPU), non_blocking=True)
        t0 = self._coll_start()
        if self.nvtx:
            torch.cuda.nvtx.range_push("all_gather group %d" % group.group_id)
        work = self.comm.all_gather_slab(slab, async_op=self.overlap_collectives, src=src)
        if self.nvtx:
            torch.cuda.nvtx.range_pop()
        if work is not None:
            self._inflight.append((work, (slab,)))
            if src is not None:
                # the collective reads the local chunk itself until it completes:
                # its next writer (the backward's grad overwrite, a K1) and the
                # slab pool wait for it, exactly as for a gathered remote chunk
                local_cid = self.chunk_set.param_chunk(pos).chunk_id
                self._wait_collective(local_cid)
                self._coll_work[local_cid] = work
        self._coll_end("all_gather", slab, work, t0)
        return slab, work

    def _coll_start(self):
        if not self.time_collectives:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def _coll_end(self, kind: str, slab: torch.Tensor, work, t0) -> None:
        if t0 is None:
            return
        end = None
        if work is None or not hasattr(work, "get_duration"):
            end = torch.cuda.Event(enable_timing=True)
            if work is not None:  # completion, seen from a side stream
                if not hasattr(self, "_timing_stream"):
                    self._timing_stream = torch.cuda.Stream(self.device)
                with torch.cuda.stream(self._timing_stream):
                    work.wait()
                    end.record()
            else:
                end.record()
        self.coll_log.append((kind, slab.numel() * slab.element_size(), work, t0, end))

    def collective_durations(self) -> List[Tuple[str, int, float, str]]:
        """(kind, slab bytes, ms, source) of every logged collective; call
        after the device finished them."""
        out = []
        for kind, nbytes, work, t0, end in self.coll_log:
            ms, src = None, "events"
            if end is None:
                try:
                    ms, src = float(work.get_duration()), "work"
                except Exception:
                    ms = None
            if ms is None and end is not None:
                ms = t0.elapsed_time(end)
            if ms is not None:
                out.append((kind, nbytes, ms, src))
        return out

    def all_gather(self, group: CommGroup, kind: str) -> None:
        if self.comm is None:
            raise RuntimeError("data-parallel gather without a communicator")
        hit = self._gather_prefetched.pop(group.group_id, None)
        if hit is not None:  # issued ahead from the previous iteration's gather log
            slab, work = hit
            self.stats.gather_prefetch_hits += 1
        else:
            slab, work = self._issue_gather(group)
        for k, q in enumerate(group.member_positions):
            if q is None or k == self.rank:
                continue
            remote = self.chunk_set.param_chunk(q)
            self.payload[GPU][remote.chunk_id] = self._group_slot(slab, k)
            self.ready.pop((remote.chunk_id, GPU), None)
            self._awaiting_gather.discard(remote.chunk_id)
            if work is not None:
                self._coll_work[remote.chunk_id] = work
        self._group_slab[group.group_id] = slab
        self._gather_log.append((self._cur_event, group.group_id))
        self.stats.gathers += 1

    def reduce_scatter(self, group: CommGroup) -> None:
        if self.comm is None:
            raise RuntimeError("data-parallel reduce-scatter without a communicator")
        cap, p = self.chunk_set.capacity_elems, self.partition.nproc
        slab = self._group_slab.get(group.group_id)
        if slab is None:
            slab = torch.empty(p * cap, dtype=self.dtype, device=self.device)
        out, out_cid = None, None
        for k, q in enumerate(group.member_positions):
            slot = self._group_slot(slab, k)
            if q is None:
                if k == self.rank:
                    slot.zero_()
                continue
            member = self.chunk_set.param_chunk(q)
            self.wait_ready(member, GPU)  # gathered / fetched data has landed
            src = self.tensor(member, GPU)
            if k == self.rank:
                out, out_cid = src, member.chunk_id
            if src.data_ptr() != slot.data_ptr():
                slot.copy_(src)
        if out is None:
            out = torch.empty(cap, dtype=self.dtype, device=self.device)  # phantom owner
        t0 = self._coll_start()
        if self.nvtx:
            torch.cuda.nvtx.range_push("reduce_scatter_avg group %d" % group.group_id)
        work = self.comm.reduce_scatter_avg(out, slab, async_op=self.overlap_collectives)
        if self.nvtx:
            torch.cuda.nvtx.range_pop()
        self._coll_end("reduce_scatter_avg", slab, work, t0)
        if work is not None:  # overlaps the next groups' backward; waited at first use
            self._inflight.append((work, (slab, out)))
            if out_cid is not None:
                self._coll_work[out_cid] = work
        if out_cid is not None:
            self._rs_out.add(out_cid)
        self._group_slab[group.group_id] = slab
        self.stats.reduce_scatters += 1

    def _prefetch_gathers(self, ev) -> None:
        """Issue the gathers the previous iteration made during the next
        ``gather_depth`` events.  The schedule comes from a ledger every rank
        shares, so all ranks issue the same NCCL calls in the same order."""
        if not self.gather_depth or not self._gather_sched:
            return
        for j in range(ev.index + 1, ev.index + 1 + self.gather_depth):
            for gid in self._gather_sched.get(j, ()):
                if gid in self._gather_prefetched:
                    continue
                self._gather_prefetched[gid] = self._issue_gather(self.partition.groups[gid])
                self.stats.gather_prefetch_issued += 1

    # -- StepExecutor ---------------------------------------------------------------------------

    def on_compute_start(self, ev, chunks: Sequence[Chunk]) -> None:
        for chunk in chunks:
            if chunk.chunk_id in self._awaiting_gather:
                raise RuntimeError("chunk %d computes before its gather" % chunk.chunk_id)
            self.wait_ready(chunk, GPU)
        cs, gpu = self.chunk_set, self.payload[GPU]
        for tid in ev.tensor_refs:
            pos, off, n = self.offsets[tid]
            cid = cs.param_chunk(pos).chunk_id
            self.params[tid].data = gpu[cid][off:off + n].view(self.shapes[tid])
            self._bound[tid] = cid

    def on_adam_begin(self, iteration: int, plan=None) -> None:
        """Global grad norm / found-inf and the device step scalars."""
        if self.comm is not None and hasattr(self.comm, "check"):
            self.comm.check()  # a collective of this step failed asynchronously
        self.join_host_work()  # the previous step's host updates are complete
        cs = self.chunk_set
        self._plan = plan
        for cid in list(self._prefetched):
            # a prefetch crosses into ADAM only for a GPU-placed position (a
            # host-placed one's host payload is what the host Adam rewrites)
            if plan is None or plan.device_of_position(cs.chunks[cid].position) != GPU:
                self._discard_prefetch(cs.chunks[cid])
        self._gather_prefetched.clear()     # (their Works are still in _inflight)
        self.wait_collectives()             # reduce-scatters into local chunks landed
        self._host_state = None
        emb_grads = []  # (key, grad): the canonical slot order of non-chunked parameters
        for (param, _, _, _), key in zip(self.embedding, self.embedding_keys):
            # the fused model writes the gradient over the weights (grad
            # overwrite); the plain model leaves it in .grad
            g = param.data if grad_in_data(param) else param.grad
            if g is None:
                raise RuntimeError("non-chunked parameter has no gradient at ADAM")
            if self.comm is not None and self.comm.world > 1:
                self.comm.all_reduce_avg(g)
            emb_grads.append((key, g))
        # K2 item slots: local positions ascending, then the non-chunked
        # parameters by key (wte 0, wpe 1, untied head 2) wherever they live
        dev_items, host_items = [], []  # (grad, n, slot)
        local = self.partition.local_positions(self.rank)
        for slot, pos in enumerate(local):
            chunk = cs.param_chunk(pos)
            n = chunk.used_elems
            if self.has(chunk, GPU):
                self.wait_ready(chunk, GPU)
                dev_items.append((self.tensor(chunk, GPU), n, slot))
            else:
                self.wait_ready(chunk, CPU)
                host_items.append((self.tensor(chunk, CPU), n, slot))
        he = self.host_embedding
        dev_emb = he is not None and he.device_compute
        drained = []
        if dev_emb:  # GPU-computed embedding, weights and optimizer state in host DRAM
            for param in he.device_params:
                g = param.data if grad_in_data(param) else param.grad
                if g is None:
                    raise RuntimeError("embedding has no gradient at ADAM")
                if self.comm is not None and self.comm.world > 1:
                    self.comm.all_reduce_avg(g)
                emb_grads.append((0, g))  # wte
                drained.append(g)
        if he is not None and not dev_emb:
            if not he.grads_ready:
                raise RuntimeError("host embedding has no gradient at ADAM")
            if self.comm is not None and self.comm.world > 1:
                for g16, _ in he.grad_items():  # average over ranks on the GPU
                    d = g16.to(self.device, non_blocking=True)
                    self.comm.all_reduce_avg(d)
                    g16.copy_(d)
        if self.comm is None or self.comm.rank == 0:  # replicated: counted once
            nc = [(key, g, True) for key, g in emb_grads]
            if he is not None and not dev_emb:
                nc += [(key, g16, False) for key, (g16, _) in enumerate(he.grad_items())]
            for k, (key, g, on_gpu) in enumerate(sorted(nc, key=lambda x: x[0])):
                (dev_items if on_gpu else host_items).append((g, g.numel(), len(local) + k))
        self._grad_sumsq(dev_items, host_items)
        if dev_emb:  # the weight gradients go up (`engine.py:214-219`, billed at BWD)
            he.drain_grads(drained, self.d2h_stream, self.compute)
            for param in he.device_params:
                if grad_in_data(param):
                    mark_grad_in_data(param, False)
                else:
                    param.grad = None
        if self.comm is not None and self.comm.world > 1:
            self.comm.all_reduce_sum(self.state.sumsq())
        K.adam_prepare(self.state, self.hyper, max_grad_norm=self.max_grad_norm,
                       dynamic_scale=self.dynamic_loss_scale)
        if not torch.cuda.is_current_stream_capturing():
            # host-side Adam waits for these scalars only, not for K1
            self._state_snap = self.state.snapshot()
        # host-placed positions: drain their gradients D2H now, in walk order,
        # so host Adam on position k overlaps the copy of position k+1 (the
        # accounting bills the same rows at each position's turn)
        plan = self._plan
        if plan is not None and self.prefetch_depth:
            for pos in self.partition.local_positions(self.rank):
                chunk = cs.param_chunk(pos)
                if plan.device_of_position(pos) == CPU and self.has(chunk, GPU) \
                        and not self.has(chunk, CPU) and chunk.chunk_id not in self._predrained:
                    d = self._alloc_d2h_dst(chunk)
                    done = self._transfer(self.tensor(chunk, GPU), d, GPU, CPU,
                                          self.ready.get((chunk.chunk_id, GPU)))
                    self._predrained[chunk.chunk_id] = (d, done)
        # non-chunked GPU parameters: the fused model wrote the gradient over
        # the weights already; a plain model's autograd gradient is packed (K3)
        for param, master, m, v in self.embedding:
            flat = param.data.view(-1)
            if grad_in_data(param):
                mark_grad_in_data(param, False)
            else:
                K.pack([(flat, 0, param.grad.view(-1), flat.numel())])
                param.grad = None
            self._pending.append((flat, master, m, v, flat.numel()))

    def _grad_sumsq(self, dev_items, host_items) -> None:
        """K2 over every local gradient in the canonical slot order: device
        items on the GPU, host items by the host twin (same bits), folded in
        slot order into the step state's sumsq -- the global norm does not
        depend on where each gradient lives."""
        n_slots = len(dev_items) + len(host_items)
        if self._sq_items.numel() != n_slots:
            self._sq_items = torch.zeros(n_slots, dtype=torch.float64, device=self.device)
        if host_items:
            sums = K.grad_sumsq_host([(g, n) for g, n, _ in host_items], self.host_threads)
            if self._sq_host is None or self._sq_host.numel() < n_slots:
                self._sq_host = torch.zeros(max(n_slots, 64), dtype=torch.float64,
                                            pin_memory=True)
            elif self._sq_host_ev is not None:
                self._sq_host_ev.synchronize()  # the last upload has read the buffer
            self._sq_host.zero_()
            for (_, _, slot), v in zip(host_items, sums):
                self._sq_host[slot] = v
            self._sq_items.copy_(self._sq_host[:n_slots], non_blocking=True)
            self._sq_host_ev = torch.cuda.Event()
            self._sq_host_ev.record()
        grads = [(g, n) for g, n, _ in dev_items]
        need = K.sumsq_scratch(grads)
        if self._sq_scratch.numel() < need:
            self._sq_scratch = torch.empty(need, device=self.device)
        K.grad_sumsq(grads, self._sq_scratch, self._sq_items,
                     slots=[slot for _, _, slot in dev_items], dtype=self.dtype)
        K.sumsq_finalize(self._sq_items, self.state)

    def init_optimizer_state(self, position: int, device: str) -> None:
        p32, m, v = (self.tensor(c, device) for c in self.chunk_set.os_triplet(position))
        src = self.init32.pop(position)
        n = self.chunk_set.param_chunk(position).used_elems
        if device == GPU:
            K.master_init(p32, m, v, src, n)   # K6 reads the pinned fp32 init in place
            self._keepalive.append(src)
        else:
            p32[:n].copy_(src[:n])
            m.zero_()
            v.zero_()

    def adam_position(self, position: int, device: str) -> None:
        cs = self.chunk_set
        param = cs.param_chunk(position)
        triplet = cs.os_triplet(position)
        n = param.used_elems
        if device == GPU:
            if self._preevict_ids and len(self._pending) >= self.preevict_batch \
                    and not self._pending_ids.isdisjoint(self._preevict_ids):
                # the pending positions' pre-evictions start behind this K1
                # (their stale host copies were dropped by the walk's note_write)
                self._flush_adam()
            for c in (param,) + triplet:
                self.wait_ready(c, GPU)
                self._discard_preevict(c.chunk_id)  # K1 rewrites it
            p16 = self.tensor(param, GPU)
            p32, m, v = (self.tensor(c, GPU) for c in triplet)
            self._pending.append((p16, p32, m, v, n))
            self._pending_ids.update(c.chunk_id for c in (param,) + triplet)
            return
        if self._host_state is None:
            self._flush_adam()  # device positions update while the host works
            self._host_state = self._step_scalars_on_host()
        for c in (param,) + triplet:
            self.wait_ready(c, CPU)
        self.stats.host_adam_items += 1
        spec = self._spec.pop(position, None)
        if spec is not None and spec[0].cancel():  # not started: the normal update instead
            self._spec_free.append(spec[2])
            self.stats.spec_cancelled += 1
            spec = None
        if spec is not None:
            job = _HostAdamJob(c.chunk_id for c in (param,) + triplet)
            for cid in job.cids:
                self._jobs[cid] = job
            job.future = self._worker.submit(position, self._settle_spec, job, spec, param,
                                             triplet, self._host_state)
            return
        p16 = self.tensor(param, CPU)
        p32, m, v = (self.tensor(c, CPU) for c in triplet)
        item = (p16, p32, m, v, n)
        if not self.async_host_adam:
            t0 = time.perf_counter()
            K.adam_chunks_host([item], self.hyper, self._host_state, self.host_threads)
            self.stats.host_adam_seconds += time.perf_counter() - t0
            return
        if self._worker is None:
            self._worker = _PriorityWorker()
        job = _HostAdamJob(c.chunk_id for c in (param,) + triplet)
        for cid in job.cids:
            self._jobs[cid] = job
        job.future = self._worker.submit(position, self._run_host_adam, job, item,
                                         self._host_state)

    def retain_param_payload(self, chunk: Chunk, device: str) -> None:
        self._retain_req.add((chunk.chunk_id, device))

    def _flush_adam(self) -> None:
        if self._pending:
            if self.adam_observer is not None:
                self.adam_observer("pre", self._pending)
            if self.record_k1:  # inside a graph capture these become event-record nodes
                ext = torch.cuda.is_current_stream_capturing()
                t0 = torch.cuda.Event(enable_timing=True, external=ext)
                t1 = torch.cuda.Event(enable_timing=True, external=ext)
                t0.record()
            K.adam_chunks(self._pending, self.hyper, self.state)
            if self.record_k1:
                t1.record()
                self.k1_events.append((t0, t1, sum(it[4] for it in self._pending)))
            if self.adam_observer is not None:
                self.adam_observer("post", self._pending)
            self.stats.adam_launch_items += len(self._pending)
            if self._preevict_ids and not torch.cuda.is_current_stream_capturing():
                for cid in sorted(self._pending_ids & self._preevict_ids):
                    self._issue_preevict(cid)
        self._pending = []
        self._pending_ids = set()

    def _issue_preevict(self, cid: int) -> None:
        """D2H of an optimizer-state chunk K1 has just updated (enqueued), to
        be adopted by the eviction the last iteration made before ADAM."""
        chunk = self.chunk_set.chunks[cid]
        if cid in self._preevicted or not self.has(chunk, GPU) or self.has(chunk, CPU):
            return
        d = self._alloc_d2h_dst(chunk)
        done = self._transfer(self.payload[GPU][cid], d, GPU, CPU, None, count=False)
        self._preevicted[cid] = (d, done)
        self.stats.preevict_issued += 1

    def _discard_preevict(self, cid: int) -> None:
        hit = self._preevicted.pop(cid, None)
        if hit is not None:
            d, done = hit
            self._give_host(d, done)  # reusable once its D2H has landed
            self.stats.preevict_discarded += 1
            self.stats.preevict_discarded_bytes += d.numel() * d.element_size()

    def _step_scalars_on_host(self):
        """Host copy of this step's scalars (waits for adam_prepare only)."""
        if self._state_snap is None:
            return self.state.read()
        return K.StepState.from_snapshot(self._state_snap)

    def on_adam_end(self) -> None:
        sched: Dict[int, List[int]] = {}
        for ev_index, gid in self._gather_log:
            sched.setdefault(ev_index, []).append(gid)
        self._gather_sched, self._gather_log = sched, []
        self._flush_adam()
        he = self.host_embedding
        if he is not None:  # host-resident embedding state: host Adam overlaps K1
            if self._host_state is None:
                self._host_state = self._step_scalars_on_host()
            if he.device_compute:
                he.d2h_done.synchronize()
            t0 = time.perf_counter()
            K.adam_chunks_host(he.adam_items(), self.hyper, self._host_state,
                               self.host_threads)
            dt = time.perf_counter() - t0
            with self._stats_lock:
                self.stats.host_adam_seconds += dt
            he.host_seconds += dt
            he.grads_ready = False
            if he.device_compute:  # weights down for the next forward (billed at FWD)
                he.upload(self.copy_stream, self.compute)
        for pos in list(self._spec):  # never reached its ADAM turn: recycle
            fut, _, shadow, _ = self._spec.pop(pos)
            if not fut.cancel():
                fut.result()
            self._spec_free.append(shadow)
            self.stats.spec_discarded += 1
        self._spec_state = None
        self._drain_candidates = []
        self._rs_out.clear()
        self._retain_req.clear()
        for (cid, dev), t in self._retained.items():
            if dev == GPU:
                self._release(cid, t)
        self._retained.clear()
        self._predrained.clear()

    def end_of_warmup(self) -> None:
        """The fp32 init copies read zero-copy by K6 can go once it has run."""
        self.join_host_work()
        torch.cuda.synchronize(self.device)
        self._keepalive = []
