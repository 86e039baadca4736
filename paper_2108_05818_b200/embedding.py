"""CPU-placed embedding operator (PatrickStar's device-aware operator placement).

The reference decides where the embedding computes
(`profiler.py:70-74` ``embedding_compute_device``: CPU whenever the fp16
weights outweigh a round trip of their activations) and bills the CPU branch
as "weights stay put; one activation block crosses per pass"
(`engine.py:202-213`: B·S·H fp16 H2D at ``embedding.fwd``, its gradient D2H at
``embedding.bwd``).  This module makes that physical:

* ``wte`` [V, H] and ``wpe`` [S, H] fp16/bf16 weights, their fp32 masters and
  Adam moments live in pinned host DRAM — never in HBM;
* forward: host lookup (``cs_embed_fwd_host``) into a pinned activation block,
  one H2D of exactly B·S·H elements;
* backward: one D2H of the activation gradient, host scatter-add
  (``cs_embed_bwd_host``) written over the fp16 weight buffers (the chunk
  path's grad overwrite, `engine.py:177-190`);
* ADAM: the host fused Adam (``cs_adam_chunks_host``, bit-identical to K1)
  updates the weights in place; with p > 1 ranks the gradient is averaged
  over the data-parallel group first.

A CPU-placed embedding cannot share its weights with the GPU LM head without
shipping them each step (the traffic the placement exists to avoid), so the
model gets an untied, GPU-resident head in this mode (``ReferenceShapedGPT``
``untied_head``).
"""

from typing import List, Optional, Tuple

import torch

from . import kernels as K


class HostEmbedding:
    """Host-resident embedding weights + the host operator; one per trainer."""

    def __init__(self, vocab: int, seq_len: int, hidden: int, dtype: torch.dtype,
                 device: torch.device, threads: int = 0, device_compute: bool = False):
        self.vocab, self.seq_len, self.hidden = vocab, seq_len, hidden
        self.dtype, self.device, self.threads = dtype, torch.device(device), threads
        pin = dict(pin_memory=True)
        self.wte = torch.empty(vocab, hidden, dtype=dtype, **pin)
        self.wpe = torch.empty(seq_len, hidden, dtype=dtype, **pin)
        self.state: List[Tuple[torch.Tensor, torch.Tensor, torch.Tensor]] = [
            tuple(torch.zeros(t.shape, dtype=torch.float32, **pin) for _ in range(3))
            for t in (self.wte, self.wpe)]
        self._act: Optional[torch.Tensor] = None      # pinned activation block
        self._dout: Optional[torch.Tensor] = None     # pinned activation gradient
        self._tok: Optional[torch.Tensor] = None      # pinned tokens of the pass
        self._act_free: Optional[torch.cuda.Event] = None
        self.host_tokens: Optional[torch.Tensor] = None  # set by step_host (no D2H)
        self.grads_ready = False
        self.grad_sumsq = 0.0      # of the last backward's gradients (cs_embed_bwd_host)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.host_seconds = 0.0
        # a leaf that requires grad, so autograd calls the host backward
        self.anchor = torch.zeros(0, device=self.device, requires_grad=True)
        #: GPU-computed embedding with host-resident weights and optimizer
        #: state (the reference's GPU branch realised, `engine.py:214-219`):
        #: the model computes on ``device_params`` = [wte] (the HBM copy of
        #: the V x H weights the reference bills, `chunks.py:204-224`, shared
        #: with a tied LM head; the small wpe is not billed and stays an HBM
        #: parameter updated by K1); the gradient goes D2H at ADAM, the host
        #: Adam updates the host state, the new weights go H2D for the next
        #: forward (``h2d_done``)
        self.device_compute = device_compute
        self.device_params: List[torch.nn.Parameter] = []
        self.d2h_done: Optional[torch.cuda.Event] = None
        self.h2d_done: Optional[torch.cuda.Event] = None

    def load(self, wte32: torch.Tensor, wpe32: torch.Tensor) -> None:
        """Initial weights (fp32, any device): masters, and the fp16 copies
        rounded on the GPU by K5 exactly as the GPU-placed path rounds them."""
        for (p16, (p32, m, v)), w32 in zip(zip((self.wte, self.wpe), self.state),
                                           (wte32, wpe32)):
            w = w32.to(self.device, torch.float32).contiguous()
            h = torch.empty(w.shape, dtype=self.dtype, device=self.device)
            K.cast_pack([(h.view(-1), 0, w.view(-1), w.numel())])
            p16.copy_(h)
            p32.copy_(w)
            m.zero_()
            v.zero_()

    # -- the operator ------------------------------------------------------------------

    def _buffers(self, B: int, S: int):
        if self._act is None or self._act.shape != (B, S, self.hidden):
            pin = dict(pin_memory=True)
            self._act = torch.empty(B, S, self.hidden, dtype=self.dtype, **pin)
            self._dout = torch.empty(B, S, self.hidden, dtype=self.dtype, **pin)
            self._tok = torch.empty(B, S, dtype=torch.int64, **pin)
            self._act_free = None
        return self._act, self._dout, self._tok

    def forward(self, tokens: torch.Tensor) -> torch.Tensor:
        return _HostEmbeddingFn.apply(tokens, self, self.anchor)

    def drain_grads(self, grads, d2h: torch.cuda.Stream, compute: torch.cuda.Stream) -> None:
        """D2H of the device weight gradients over the host fp16 weights (the
        host copy of the grad overwrite), ordered after ``compute``."""
        d2h.wait_stream(compute)
        with torch.cuda.stream(d2h):
            for host, g in zip(self._host_weights(), grads):
                host.view(-1).copy_(g.reshape(-1), non_blocking=True)
                g.record_stream(d2h)
                self.d2h_bytes += host.numel() * host.element_size()
            self.d2h_done = torch.cuda.Event()
            self.d2h_done.record(d2h)

    def upload(self, h2d: torch.cuda.Stream, compute: torch.cuda.Stream) -> None:
        """H2D of the updated host weights into the device copies, after every
        device read of the gradients they held (K2 on ``compute``, the D2H)."""
        h2d.wait_stream(compute)
        h2d.wait_event(self.d2h_done)
        with torch.cuda.stream(h2d):
            for host, p in zip(self._host_weights(), self.device_params):
                p.data.view(-1).copy_(host.view(-1), non_blocking=True)
                self.h2d_bytes += host.numel() * host.element_size()
            self.h2d_done = torch.cuda.Event()
            self.h2d_done.record(h2d)

    def _host_weights(self):
        return (self.wte,) if self.device_compute else (self.wte, self.wpe)

    def adam_items(self):
        """(g16/p16, p32, m, v, n) host items for ``cs_adam_chunks_host``."""
        return [(p16.view(-1), p32.view(-1), m.view(-1), v.view(-1), p16.numel())
                for p16, (p32, m, v) in zip(self._host_weights(), self.state)]

    def grad_items(self):
        return [(p16.view(-1), p16.numel()) for p16 in self._host_weights()]


class _HostEmbeddingFn(torch.autograd.Function):

    @staticmethod
    def forward(ctx, tokens, emb: HostEmbedding, anchor):
        import time
        B, S = tokens.shape
        act, _, tok = emb._buffers(B, S)
        if emb._act_free is not None:     # the previous pass's H2D has read the block
            emb._act_free.synchronize()
        src = emb.host_tokens
        emb.host_tokens = None
        if src is not None and tuple(src.shape) == (B, S):
            tok.copy_(src)
        else:
            tok.copy_(tokens)              # device tokens: one small D2H (synchronous)
        t0 = time.perf_counter()
        K.embed_fwd_host(tok, emb.wte, emb.wpe, act, emb.threads)
        emb.host_seconds += time.perf_counter() - t0
        out = torch.empty(B, S, emb.hidden, dtype=emb.dtype, device=emb.device)
        out.copy_(act, non_blocking=True)
        emb._act_free = torch.cuda.Event()
        emb._act_free.record()
        emb.h2d_bytes += act.numel() * act.element_size()
        emb.grads_ready = False
        ctx.emb = emb
        return out

    @staticmethod
    def backward(ctx, grad):
        import time
        emb = ctx.emb
        _, dout, tok = emb._buffers(*grad.shape[:2])
        dout.copy_(grad.contiguous(), non_blocking=True)
        torch.cuda.current_stream(emb.device).synchronize()
        emb.d2h_bytes += dout.numel() * dout.element_size()
        t0 = time.perf_counter()
        # grad overwrite; the squares of the written rows come back with it
        emb.grad_sumsq = K.embed_bwd_host(tok, dout, emb.wte, emb.wpe, emb.threads)
        emb.host_seconds += time.perf_counter() - t0
        emb.grads_ready = True
        return None, None, None
