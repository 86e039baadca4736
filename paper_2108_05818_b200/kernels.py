"""Tensor-level wrappers over the C ABI (device pointers + the current stream).

Each wrapper takes torch tensors that live on the GPU (or, for
:func:`adam_chunks_host`, in pinned host memory), extracts raw pointers and
calls the corresponding ``cs_*`` entry point on the given/current CUDA
stream.  They validate dtypes and devices and raise on any error: there is
no CPU path for GPU-resident work.
"""

import ctypes
from typing import List, Optional, Sequence, Tuple

import torch

from . import _native as N

DTYPE_CODE = {torch.float16: N.CS_FP16, torch.bfloat16: N.CS_BF16}
SRC_CODE = {torch.float16: N.CS_FP16, torch.bfloat16: N.CS_BF16, torch.float32: N.CS_FP32}


def _code(dtype: torch.dtype) -> int:
    if dtype not in DTYPE_CODE:
        raise TypeError("chunk payload dtype must be float16 or bfloat16, got %s" % dtype)
    return DTYPE_CODE[dtype]


def _stream(stream: Optional[torch.cuda.Stream]) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if not t.is_cuda:
            raise ValueError("expected a CUDA tensor, got one on %s" % t.device)


class AdamHyper:
    def __init__(self, lr: float = 1e-4, betas: Tuple[float, float] = (0.9, 0.999),
                 eps: float = 1e-8, weight_decay: float = 0.0, adamw: bool = False):
        self.lr, self.betas, self.eps = lr, betas, eps
        self.weight_decay, self.adamw = weight_decay, adamw

    def c(self) -> N.CsAdamHyper:
        return N.CsAdamHyper(self.lr, self.betas[0], self.betas[1], self.eps,
                             self.weight_decay, int(self.adamw))


class StepState:
    """Device-resident ``CsStepState`` (one per optimizer)."""

    NBYTES = 64

    def __init__(self, device: torch.device, init_loss_scale: float = 1.0,
                 stream: Optional[torch.cuda.Stream] = None):
        assert ctypes.sizeof(N.CsStepState) <= self.NBYTES
        self.buf = torch.zeros(self.NBYTES, dtype=torch.uint8, device=device)
        N.check(N.load().cs_step_state_init(ctypes.c_void_p(self.buf.data_ptr()),
                                            float(init_loss_scale), _stream(stream)),
                "cs_step_state_init")

    @property
    def ptr(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(self.buf.data_ptr())

    def _f32(self, field: str) -> torch.Tensor:
        off = getattr(N.CsStepState, field).offset
        return self.buf[off:off + 4].view(torch.float32)

    def loss_scale(self) -> torch.Tensor:
        """0-dim device view of the current loss scale (no sync)."""
        return self._f32("loss_scale")[0]

    def grad_norm(self) -> torch.Tensor:
        return self._f32("grad_norm")[0]

    def sumsq(self) -> torch.Tensor:
        return self._f32("sumsq")

    def snapshot(self):
        """Queue an async copy of the state into pinned memory on the current
        stream (after the kernels enqueued so far, not after later ones);
        :meth:`from_snapshot` waits for exactly that copy."""
        host = torch.empty(self.NBYTES, dtype=torch.uint8, pin_memory=True)
        host.copy_(self.buf, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return host, ev

    @staticmethod
    def from_snapshot(snap) -> N.CsStepState:
        host, ev = snap
        ev.synchronize()
        raw = bytes(host.numpy().tobytes())
        return N.CsStepState.from_buffer_copy(raw[:ctypes.sizeof(N.CsStepState)])

    def read(self) -> N.CsStepState:
        """Host copy (synchronises the buffer's stream)."""
        raw = bytes(self.buf.cpu().numpy().tobytes())
        return N.CsStepState.from_buffer_copy(raw[:ctypes.sizeof(N.CsStepState)])


def adam_chunks(items: Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, int]],
                hyper: AdamHyper, state: StepState,
                stream: Optional[torch.cuda.Stream] = None) -> None:
    """K1 over many (p16, p32, m, v, n) items in one launch (per 256 items)."""
    if not items:
        return
    arr = (N.CsAdamItem * len(items))()
    dt = _code(items[0][0].dtype)
    for i, (p16, p32, m, v, n) in enumerate(items):
        _need_cuda(p16, p32, m, v)
        if p16.dtype != items[0][0].dtype or p32.dtype != torch.float32:
            raise TypeError("mixed or wrong dtypes in adam items")
        if min(p16.numel(), p32.numel(), m.numel(), v.numel()) < n:
            raise ValueError("adam item %d: n=%d exceeds a buffer" % (i, n))
        arr[i] = N.CsAdamItem(p16.data_ptr(), p32.data_ptr(), m.data_ptr(), v.data_ptr(), n)
    h = hyper.c()
    N.check(N.load().cs_adam_chunks(arr, len(items), dt, ctypes.byref(h), state.ptr,
                                    _stream(stream)), "cs_adam_chunks")


def host_threads(requested: int = 0) -> int:
    """OpenMP team size the host kernels use (``cs_host_threads``)."""
    return int(N.load().cs_host_threads(int(requested)))


def adam_chunks_host(items, hyper: AdamHyper, state: N.CsStepState, n_threads: int = 0) -> None:
    """Host Adam for CPU-placed positions (tensors in host memory)."""
    if not items:
        return
    arr = (N.CsAdamItem * len(items))()
    dt = _code(items[0][0].dtype)
    for i, (p16, p32, m, v, n) in enumerate(items):
        if p16.is_cuda or p32.is_cuda:
            raise ValueError("host adam needs host tensors")
        arr[i] = N.CsAdamItem(p16.data_ptr(), p32.data_ptr(), m.data_ptr(), v.data_ptr(), n)
    h = hyper.c()
    N.check(N.load().cs_adam_chunks_host(arr, len(items), dt, ctypes.byref(h),
                                         ctypes.byref(state), int(n_threads)),
            "cs_adam_chunks_host")


def speculate_step_scalars(prev: N.CsStepState, hyper: AdamHyper) -> N.CsStepState:
    """The step scalars ``cs_adam_prepare`` will produce for the NEXT step if
    its gradients are finite and not clipped, from the state it left after
    this one (same IEEE operations, so the same bits): grad_scale = 1 / loss
    scale, step + 1, beta powers, step_size, sqrt_bc2, skip = 0.  Only the
    fields the Adam reads are meaningful."""
    import numpy as np
    s = N.CsStepState.from_buffer_copy(bytes(prev))
    b1p = float(np.float64(prev.beta1_pow) * np.float64(hyper.betas[0]))
    b2p = float(np.float64(prev.beta2_pow) * np.float64(hyper.betas[1]))
    s.grad_scale = float(np.float32(1.0) / np.float32(prev.loss_scale))
    s.step = prev.step + 1
    s.beta1_pow, s.beta2_pow = b1p, b2p
    s.step_size = float(np.float32(np.float64(hyper.lr) / (np.float64(1.0) - np.float64(b1p))))
    s.sqrt_bc2 = float(np.float32(np.sqrt(np.float64(1.0) - np.float64(b2p))))
    s.skip = 0
    return s


def same_update_scalars(a: N.CsStepState, b: N.CsStepState) -> bool:
    """True when two states drive the Adam identically (the fields it reads)."""
    import numpy as np
    f32 = lambda x: np.float32(x).tobytes()  # noqa: E731
    return (a.skip == b.skip == 0 and f32(a.grad_scale) == f32(b.grad_scale)
            and f32(a.step_size) == f32(b.step_size) and f32(a.sqrt_bc2) == f32(b.sqrt_bc2))


def adam_chunks_host_oop(items_in, items_out, hyper: AdamHyper, state: N.CsStepState,
                         n_threads: int = 0) -> None:
    """Out-of-place host Adam (cs_adam_chunks_host_oop): reads (g16, p32, m, v)
    of items_in, writes (p16, p32, m, v) of items_out; same bits as
    :func:`adam_chunks_host`."""
    if not items_in:
        return
    if len(items_in) != len(items_out):
        raise ValueError("adam_chunks_host_oop: in / out item counts differ")
    a = (N.CsAdamItem * len(items_in))()
    b = (N.CsAdamItem * len(items_in))()
    dt = _code(items_in[0][0].dtype)
    for i, (x, y) in enumerate(zip(items_in, items_out)):
        if any(t.is_cuda for t in x[:4] + y[:4]):
            raise ValueError("host adam needs host tensors")
        a[i] = N.CsAdamItem(*(t.data_ptr() for t in x[:4]), x[4])
        b[i] = N.CsAdamItem(*(t.data_ptr() for t in y[:4]), y[4])
    h = hyper.c()
    N.check(N.load().cs_adam_chunks_host_oop(a, b, len(items_in), dt, ctypes.byref(h),
                                             ctypes.byref(state), int(n_threads)),
            "cs_adam_chunks_host_oop")


def grad_sumsq_host(grads: Sequence[Tuple[torch.Tensor, int]], n_threads: int = 0) -> List[float]:
    """K2's host twin: the canonical sum of squares S_i (double) of each
    host-resident fp16/bf16 gradient prefix -- the same bits K2 writes for
    the same bytes in HBM."""
    if not grads:
        return []
    arr = (N.CsGradItem * len(grads))()
    for i, (g, n) in enumerate(grads):
        if g.is_cuda:
            raise ValueError("grad_sumsq_host needs host tensors")
        arr[i] = N.CsGradItem(g.data_ptr(), n)
    out = (ctypes.c_double * len(grads))()
    N.check(N.load().cs_grad_sumsq_host(arr, len(grads), _code(grads[0][0].dtype), out,
                                        int(n_threads)), "cs_grad_sumsq_host")
    return list(out)


def _host_contig(*ts: torch.Tensor) -> None:
    for t in ts:
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("host embedding kernels need contiguous host tensors")


def embed_fwd_host(tokens: torch.Tensor, wte: torch.Tensor, wpe: torch.Tensor,
                   out: torch.Tensor, n_threads: int = 0) -> torch.Tensor:
    """CPU-placed embedding lookup (cs_embed_fwd_host): tokens [B, S] int64,
    wte [V, H], wpe [>=S, H], out [B, S, H] (all host, fp16/bf16)."""
    _host_contig(tokens, wte, wpe, out)
    if tokens.dtype != torch.int64:
        raise TypeError("tokens must be int64")
    B, S = tokens.shape
    V, H = wte.shape
    N.check(N.load().cs_embed_fwd_host(tokens.data_ptr(), B * S, S, wte.data_ptr(),
                                       wpe.data_ptr(), V, H, out.data_ptr(), _code(wte.dtype),
                                       int(n_threads)), "cs_embed_fwd_host")
    return out


def embed_bwd_host(tokens: torch.Tensor, dout: torch.Tensor, gwte: torch.Tensor,
                   gwpe: torch.Tensor, n_threads: int = 0) -> float:
    """Gradient of the lookup written over gwte [V, H] / gwpe [S, H]
    (cs_embed_bwd_host; deterministic fp32 sums, ascending token order).
    Returns the sum of squares of the written gradients (double, row order)."""
    _host_contig(tokens, dout, gwte, gwpe)
    B, S = tokens.shape
    V, H = gwte.shape
    if gwpe.shape[0] != S:
        raise ValueError("gwpe must have seq_len rows")
    out = ctypes.c_double(0.0)
    N.check(N.load().cs_embed_bwd_host(tokens.data_ptr(), B * S, S, dout.data_ptr(), V, H,
                                       gwte.data_ptr(), gwpe.data_ptr(), _code(gwte.dtype),
                                       int(n_threads), ctypes.byref(out)), "cs_embed_bwd_host")
    return out.value


def embed_fwd(tokens: torch.Tensor, wte: torch.Tensor, wpe: torch.Tensor,
              stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """GPU-placed embedding lookup (cs_embed_fwd): tokens [B, S] int64 ->
    [B, S, H]; same bits as :func:`embed_fwd_host`."""
    _need_cuda(tokens, wte, wpe)
    tok = tokens.contiguous()
    if tok.dtype != torch.int64:
        raise TypeError("tokens must be int64")
    B, S = tok.shape
    V, H = wte.shape
    out = torch.empty(B, S, H, dtype=wte.dtype, device=wte.device)
    N.check(N.load().cs_embed_fwd(tok.data_ptr(), B * S, S, wte.data_ptr(), wpe.data_ptr(), V,
                                  H, out.data_ptr(), _code(wte.dtype), _stream(stream)),
            "cs_embed_fwd")
    return out


def embed_bwd(tokens: torch.Tensor, dout: torch.Tensor, vocab: int, seq_rows: int,
              stream: Optional[torch.cuda.Stream] = None):
    """(gwte [V, H], gwpe [seq_rows, H]) for the lookup's output gradient
    (cs_embed_bwd; the stable sort of the token ids is torch plumbing).
    Rows of gwpe beyond the sequence length are zero."""
    H = dout.shape[-1]
    gwte = torch.empty(vocab, H, dtype=dout.dtype, device=dout.device)
    gwpe = torch.empty(seq_rows, H, dtype=dout.dtype, device=dout.device)
    embed_bwd_into(tokens, dout, gwte, gwpe, accumulate=False, stream=stream)
    return gwte, gwpe


def embed_bwd_into(tokens: torch.Tensor, dout: torch.Tensor, gwte: torch.Tensor,
                   gwpe: torch.Tensor, accumulate: bool = False,
                   stream: Optional[torch.cuda.Stream] = None) -> None:
    """The lookup's gradient written over (or, ``accumulate``, added to)
    gwte [V, H], and written over gwpe [>=S, H] (rows >= S zeroed) — e.g. the
    weight buffers themselves (grad overwrite)."""
    _need_cuda(tokens, dout, gwte, gwpe)
    tok = tokens.contiguous().view(-1)
    B, S = tokens.shape
    V, H = gwte.shape
    d = dout.contiguous()
    srt, order = torch.sort(tok, stable=True)
    bounds = torch.arange(V + 1, device=tok.device, dtype=torch.int64)
    row_start = torch.searchsorted(srt, bounds)
    if gwpe.shape[0] > S:
        gwpe[S:].zero_()
    N.check(N.load().cs_embed_bwd(order.data_ptr(), row_start.data_ptr(), B * S, S, d.data_ptr(),
                                  V, H, gwte.data_ptr(), gwpe.data_ptr(), int(accumulate),
                                  _code(dout.dtype), _stream(stream)), "cs_embed_bwd")


def _grad_items(grads):
    arr = (N.CsGradItem * max(len(grads), 1))()
    for i, (g, n) in enumerate(grads):
        arr[i] = N.CsGradItem(g.data_ptr(), n)
    return arr


def sumsq_scratch(grads: Sequence[Tuple[torch.Tensor, int]]) -> int:
    """Floats of K2 scratch the given gradient prefixes need."""
    n = N.load().cs_sumsq_scratch(_grad_items(grads), len(grads))
    if n < 0:
        raise N.NativeError("cs_sumsq_scratch: invalid items")
    return int(n)


def grad_sumsq(grads: Sequence[Tuple[torch.Tensor, int]], scratch: torch.Tensor,
               item_sums: torch.Tensor, slots: Optional[Sequence[int]] = None,
               stream: Optional[torch.cuda.Stream] = None,
               dtype: Optional[torch.dtype] = None) -> None:
    """K2: the canonical sum of squares S_i of each gradient prefix, written
    into ``item_sums[slots[i]]`` (float64, on the device)."""
    for g, _ in grads:
        _need_cuda(g)
    if item_sums.dtype != torch.float64 or not item_sums.is_cuda:
        raise ValueError("item_sums must be a float64 CUDA tensor")
    arr = _grad_items(grads)
    sl = None
    if slots is not None:
        sl = (ctypes.c_int * max(len(slots), 1))(*slots)
    dt = _code(dtype if dtype is not None else (grads[0][0].dtype if grads else torch.float16))
    N.check(N.load().cs_grad_sumsq(arr, len(grads), dt, sl, ctypes.c_void_p(scratch.data_ptr()),
                                   scratch.numel(), ctypes.c_void_p(item_sums.data_ptr()),
                                   _stream(stream)), "cs_grad_sumsq")


def sumsq_finalize(item_sums: torch.Tensor, state: StepState,
                   stream: Optional[torch.cuda.Stream] = None) -> None:
    """state.sumsq = (float) of the slots of ``item_sums`` folded in order (double)."""
    N.check(N.load().cs_sumsq_finalize(ctypes.c_void_p(item_sums.data_ptr()), item_sums.numel(),
                                       state.ptr, _stream(stream)), "cs_sumsq_finalize")


def adam_prepare(state: StepState, hyper: AdamHyper, max_grad_norm: float = 0.0,
                 growth_factor: float = 2.0, backoff_factor: float = 0.5,
                 growth_interval: int = 2000, dynamic_scale: bool = False,
                 stream: Optional[torch.cuda.Stream] = None) -> None:
    h = hyper.c()
    N.check(N.load().cs_adam_prepare(state.ptr, ctypes.byref(h), float(max_grad_norm),
                                     float(growth_factor), float(backoff_factor),
                                     int(growth_interval), int(dynamic_scale),
                                     _stream(stream)), "cs_adam_prepare")


def _pack_items(items) -> "ctypes.Array":
    arr = (N.CsPackItem * len(items))()
    for i, (chunk, offset, src, n) in enumerate(items):
        _need_cuda(chunk, src)
        if offset < 0 or offset + n > chunk.numel() or n > src.numel():
            raise ValueError("pack item %d out of bounds" % i)
        arr[i] = N.CsPackItem(chunk.data_ptr(), offset, src.data_ptr(), n)
    return arr


def pack(items: Sequence[Tuple[torch.Tensor, int, torch.Tensor, int]], accumulate: bool = False,
         stream: Optional[torch.cuda.Stream] = None) -> None:
    """K3 (slot = src) / K4 (slot += src) over (chunk, offset, src, n) items."""
    if not items:
        return
    dt = _code(items[0][0].dtype)
    for chunk, _, src, _ in items:
        if chunk.dtype != src.dtype:
            raise TypeError("pack: chunk and source dtypes differ")
    N.check(N.load().cs_pack(_pack_items(items), len(items), dt, int(accumulate),
                             _stream(stream)), "cs_pack")


def cast_pack(items: Sequence[Tuple[torch.Tensor, int, torch.Tensor, int]],
              stream: Optional[torch.cuda.Stream] = None) -> None:
    """K5: fp32 sources -> fp16/bf16 chunk slots."""
    if not items:
        return
    dt = _code(items[0][0].dtype)
    for _, _, src, _ in items:
        if src.dtype != torch.float32:
            raise TypeError("cast_pack sources must be float32")
    N.check(N.load().cs_cast_pack(_pack_items(items), len(items), dt, _stream(stream)),
            "cs_cast_pack")


def master_init(p32: torch.Tensor, m: torch.Tensor, v: torch.Tensor, src: torch.Tensor,
                n: int, stream: Optional[torch.cuda.Stream] = None) -> None:
    """K6: p32 = float(src[:n]), m = v = 0.  ``src`` may be pinned host memory."""
    _need_cuda(p32, m, v)
    if src.dtype not in SRC_CODE:
        raise TypeError("master_init source dtype %s" % src.dtype)
    if not src.is_cuda and not src.is_pinned():
        raise ValueError("master_init host source must be pinned (device-mapped)")
    N.check(N.load().cs_master_init(ctypes.c_void_p(p32.data_ptr()), ctypes.c_void_p(m.data_ptr()),
                                    ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                    SRC_CODE[src.dtype], int(n), _stream(stream)),
            "cs_master_init")


def xent_fwd(logits: torch.Tensor, targets: torch.Tensor,
             stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per-row cross-entropy loss and logsumexp of fp16/bf16 logits [rows, vocab]."""
    _need_cuda(logits, targets)
    if logits.dim() != 2 or not logits.is_contiguous() or targets.dtype != torch.int64:
        raise ValueError("xent_fwd wants contiguous 2-D logits and int64 targets")
    rows, vocab = logits.shape
    tg = targets.reshape(-1).contiguous()
    loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
    N.check(N.load().cs_xent_fwd(ctypes.c_void_p(logits.data_ptr()), ctypes.c_void_p(tg.data_ptr()),
                                 rows, vocab, _code(logits.dtype), ctypes.c_void_p(loss.data_ptr()),
                                 ctypes.c_void_p(lse.data_ptr()), _stream(stream)), "cs_xent_fwd")
    return loss, lse


def xent_bwd_(logits: torch.Tensor, targets: torch.Tensor, lse: torch.Tensor,
              dloss: torch.Tensor, scale: float,
              stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """In place: logits <- (softmax - onehot) * dloss * scale."""
    rows, vocab = logits.shape
    tg = targets.reshape(-1).contiguous()
    d = dloss.reshape(1).float().contiguous()
    N.check(N.load().cs_xent_bwd(ctypes.c_void_p(logits.data_ptr()), ctypes.c_void_p(tg.data_ptr()),
                                 ctypes.c_void_p(lse.data_ptr()), ctypes.c_void_p(d.data_ptr()),
                                 float(scale), rows, vocab, _code(logits.dtype),
                                 _stream(stream)), "cs_xent_bwd")
    return logits


_WORKSPACE = {}


def _lt_workspace(device: torch.device) -> torch.Tensor:
    ws = _WORKSPACE.get(device)
    if ws is None:
        ws = _WORKSPACE[device] = torch.empty(32 << 20, dtype=torch.uint8, device=device)
    return ws


def gemm_gelu_fwd(x2d: torch.Tensor, w: torch.Tensor,
                  stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """(u, g) = (x·Wᵀ, gelu_tanh(x·Wᵀ)) in one cuBLASLt GEMM (GELU_AUX epilogue)."""
    _need_cuda(x2d, w)
    T, K = x2d.shape
    O = w.shape[0]
    if w.shape[1] != K or not x2d.is_contiguous() or not w.is_contiguous():
        raise ValueError("gemm_gelu_fwd: shapes/contiguity")
    g = torch.empty(T, O, dtype=x2d.dtype, device=x2d.device)
    u = torch.empty(T, O, dtype=x2d.dtype, device=x2d.device)
    ws = _lt_workspace(x2d.device)
    N.check(N.load().cs_gemm_gelu(0, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(x2d.data_ptr()),
                                  ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(u.data_ptr()),
                                  T, O, K, _code(x2d.dtype), ctypes.c_void_p(ws.data_ptr()),
                                  ws.numel(), _stream(stream)), "cs_gemm_gelu(fwd)")
    return u, g


def gemm_dgelu(dy2d: torch.Tensor, w: torch.Tensor, u: torch.Tensor,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """du = (dy·W) ⊙ gelu_tanh'(u) in one cuBLASLt GEMM (DGELU epilogue); W [K,O]."""
    _need_cuda(dy2d, w, u)
    T, K = dy2d.shape
    O = w.shape[1]
    if w.shape[0] != K or tuple(u.shape) != (T, O) or not dy2d.is_contiguous() \
            or not w.is_contiguous() or not u.is_contiguous():
        raise ValueError("gemm_dgelu: shapes/contiguity")
    du = torch.empty(T, O, dtype=dy2d.dtype, device=dy2d.device)
    ws = _lt_workspace(dy2d.device)
    N.check(N.load().cs_gemm_gelu(1, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(dy2d.data_ptr()),
                                  ctypes.c_void_p(du.data_ptr()), ctypes.c_void_p(u.data_ptr()),
                                  T, O, K, _code(dy2d.dtype), ctypes.c_void_p(ws.data_ptr()),
                                  ws.numel(), _stream(stream)), "cs_gemm_gelu(bwd)")
    return du


def gemm_res(x2d: torch.Tensor, w: torch.Tensor, res2d: torch.Tensor,
             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """out = x·Wᵀ + res in one cuBLASLt GEMM that reads res itself (C ≠ D,
    beta = 1) — torch.addmm would first copy res into its output."""
    _need_cuda(x2d, w, res2d)
    T, K_ = x2d.shape
    O = w.shape[0]
    if w.shape[1] != K_ or tuple(res2d.shape) != (T, O) or not x2d.is_contiguous() \
            or not w.is_contiguous() or not res2d.is_contiguous():
        raise ValueError("gemm_res: shapes/contiguity")
    out = torch.empty(T, O, dtype=x2d.dtype, device=x2d.device)
    ws = _lt_workspace(x2d.device)
    N.check(N.load().cs_gemm_res(ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(x2d.data_ptr()),
                                 ctypes.c_void_p(res2d.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                 T, O, K_, _code(x2d.dtype), ctypes.c_void_p(ws.data_ptr()),
                                 ws.numel(), _stream(stream)), "cs_gemm_res")
    return out


def layernorm_supported(H: int) -> bool:
    return bool(N.load().cs_layernorm_supported(int(H)))


def layernorm_fwd(x2d: torch.Tensor, eps: float = 1e-5,
                  stream: Optional[torch.cuda.Stream] = None):
    """Non-affine LN over the last dim of a contiguous [rows, H] tensor."""
    _need_cuda(x2d)
    rows, H = x2d.shape
    y = torch.empty_like(x2d)
    mean = torch.empty(rows, dtype=torch.float32, device=x2d.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=x2d.device)
    N.check(N.load().cs_layernorm_fwd(ctypes.c_void_p(x2d.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                      ctypes.c_void_p(mean.data_ptr()),
                                      ctypes.c_void_p(rstd.data_ptr()), rows, H, float(eps),
                                      _code(x2d.dtype), _stream(stream)), "cs_layernorm_fwd")
    return y, mean, rstd


def layernorm_bwd(dy2d: torch.Tensor, x2d: torch.Tensor, mean: torch.Tensor, rstd: torch.Tensor,
                  dres2d: Optional[torch.Tensor] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    rows, H = x2d.shape
    dx = torch.empty_like(x2d)
    N.check(N.load().cs_layernorm_bwd(ctypes.c_void_p(dy2d.data_ptr()), ctypes.c_void_p(x2d.data_ptr()),
                                      ctypes.c_void_p(mean.data_ptr()),
                                      ctypes.c_void_p(rstd.data_ptr()),
                                      ctypes.c_void_p(dres2d.data_ptr() if dres2d is not None else 0),
                                      ctypes.c_void_p(dx.data_ptr()), rows, H, _code(x2d.dtype),
                                      _stream(stream)), "cs_layernorm_bwd")
    return dx
