"""Reference-shaped GPT whose chunk-managed parameters are exactly
``param_tensor_specs(schema)`` (`/root/reference/pkg/src/chunkstar/model.py:163-191`).

Per layer, four operator slots:

    qkv      three [H, H] projections           (tensor ids 8l+0..2)
    attn_out one [H, H] projection              (8l+3)
    mlp_in   two [2H, H] halves, outputs concat (8l+4, 8l+5)
    mlp_out  two [H, 2H] halves, outputs summed (8l+6, 8l+7)

No biases and non-affine LayerNorms, so nothing else needs chunk
management; token/position embeddings (tied LM head) are the reference's
non-chunked embedding allocation (`chunks.py:204-224`).  Splitting a GEMM
along N (concat) or K (sum) changes nothing but rounding order.

Each slot is bracketed by two autograd markers so the *real* forward and
backward drive the engine's events in timeline order (`model.py:263-329`):

* ``_SlotEnter`` on the slot inputs: forward = event start (gather, fetch,
  bind parameter views); backward = BWD event *finish* (it runs only once
  every dX of the slot is computed, i.e. after all of its dW were written);
* ``_SlotExit`` on the slot outputs: forward = FWD event finish; backward =
  BWD event *start* (before any of the slot's backward GEMMs).

:class:`ChunkLinear` keeps a reference to the ``nn.Parameter`` itself rather
than a saved view, so a chunk that was evicted and re-fetched (new storage)
between FWD and BWD is read from its current location; in backward it
computes dX first and then writes dW *directly into the parameter's chunk
slot* (``torch.mm(..., out=slot)``) — the gradient-overwrites-parameter
reuse of PatrickStar §4 with zero extra traffic (the K3 pack kernel is used
where a gradient arrives from autograd instead, e.g. the embedding).
"""

from typing import Callable, List, Optional, Tuple

import torch
import torch.nn as nn
import torch.nn.functional as F

from .model import ModelSchema, OP_SLOTS, param_tensor_specs


class _ChunkLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x: torch.Tensor, weight: nn.Parameter, grad_sink: Callable):
        ctx.weight = weight          # the Parameter object, not a saved view
        ctx.grad_sink = grad_sink
        ctx.save_for_backward(x)
        return F.linear(x, weight)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        (x,) = ctx.saved_tensors
        w = ctx.weight
        dx = dy.matmul(w)            # needs W: computed before the slot is overwritten
        ctx.grad_sink(w, dy.reshape(-1, dy.shape[-1]), x.reshape(-1, x.shape[-1]))
        return dx, None, None


def _residual_gemm(x2: torch.Tensor, w: torch.Tensor, r2: torch.Tensor) -> torch.Tensor:
    """x Wᵀ + r with the residual read by the GEMM (cs_gemm_res) when the
    operands are contiguous fp16/bf16 CUDA tensors, else torch.addmm."""
    from . import kernels as K
    if (x2.is_cuda and x2.dtype in K.DTYPE_CODE and x2.is_contiguous() and r2.is_contiguous()
            and w.is_contiguous()):
        return K.gemm_res(x2, w, r2)
    return torch.addmm(r2, x2, w.t())


class _ChunkLinearResFn(torch.autograd.Function):
    """y = residual + x W^T with the add inside the GEMM (C ≠ D, beta = 1)."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, weight: nn.Parameter, residual: torch.Tensor,
                grad_sink: Callable):
        ctx.weight = weight
        ctx.grad_sink = grad_sink
        ctx.save_for_backward(x)
        shp = residual.shape
        out = _residual_gemm(x.reshape(-1, x.shape[-1]), weight, residual.reshape(-1, shp[-1]))
        return out.view(shp)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        (x,) = ctx.saved_tensors
        w = ctx.weight
        dx = dy.matmul(w)
        ctx.grad_sink(w, dy.reshape(-1, dy.shape[-1]), x.reshape(-1, x.shape[-1]))
        return dx, None, dy, None


class _GeluLinearResFn(torch.autograd.Function):
    """mlp_out half: y = residual + gelu(u) Wᵀ, given g = gelu(u) from the
    forward epilogue; backward's dX GEMM applies gelu'(u) in its DGELU
    epilogue (cs_gemm_gelu mode 1) and hands du straight to mlp_in."""

    @staticmethod
    def forward(ctx, g: torch.Tensor, u: torch.Tensor, weight: nn.Parameter,
                residual: torch.Tensor, grad_sink: Callable):
        ctx.weight, ctx.grad_sink = weight, grad_sink
        ctx.save_for_backward(g, u)
        shp = residual.shape
        out = _residual_gemm(g.reshape(-1, g.shape[-1]), weight, residual.reshape(-1, shp[-1]))
        return out.view(shp)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        from . import kernels as K
        g, u = ctx.saved_tensors
        w = ctx.weight
        dy2 = dy.reshape(-1, dy.shape[-1]).contiguous()
        du = K.gemm_dgelu(dy2, w, u.reshape(-1, u.shape[-1]))
        ctx.grad_sink(w, dy2, g.reshape(-1, g.shape[-1]))
        return None, du.view(u.shape), None, dy, None


class _LNResFn(torch.autograd.Function):
    """(LN(h), h): the residual stream passes through the LayerNorm function so
    that its backward gets both gradients and returns LN_bwd(dy) + d_residual
    from one kernel (cs_layernorm_bwd) — no autograd accumulation pass."""

    @staticmethod
    def forward(ctx, h: torch.Tensor):
        from . import kernels as K
        h2 = h.reshape(-1, h.shape[-1])
        y, mean, rstd = K.layernorm_fwd(h2)
        ctx.save_for_backward(h2, mean, rstd)
        return y.view_as(h), h.view_as(h)

    @staticmethod
    def backward(ctx, dy: torch.Tensor, dres: torch.Tensor):
        from . import kernels as K
        h2, mean, rstd = ctx.saved_tensors
        H = h2.shape[-1]
        dx = K.layernorm_bwd(dy.reshape(-1, H).contiguous(), h2, mean, rstd,
                             None if dres is None else dres.reshape(-1, H).contiguous())
        return dx.view_as(dy)


class _LNFn(torch.autograd.Function):
    """Plain non-affine LayerNorm on cs_layernorm_fwd/bwd (the final LN)."""

    @staticmethod
    def forward(ctx, h: torch.Tensor):
        from . import kernels as K
        h2 = h.reshape(-1, h.shape[-1])
        y, mean, rstd = K.layernorm_fwd(h2)
        ctx.save_for_backward(h2, mean, rstd)
        return y.view_as(h)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        from . import kernels as K
        h2, mean, rstd = ctx.saved_tensors
        H = h2.shape[-1]
        return K.layernorm_bwd(dy.reshape(-1, H).contiguous(), h2, mean, rstd).view_as(dy)


class _QKVFn(torch.autograd.Function):
    """q, k, v = x Wqᵀ, x Wkᵀ, x Wvᵀ; backward accumulates dX = dq Wq + dk Wk
    + dv Wv in the GEMM epilogue (beta = 1) instead of two add passes, then
    writes each dW over its chunk slot."""

    @staticmethod
    def forward(ctx, x, wq, wk, wv, grad_sink):
        ctx.ws, ctx.grad_sink = (wq, wk, wv), grad_sink
        ctx.save_for_backward(x)
        return F.linear(x, wq), F.linear(x, wk), F.linear(x, wv)

    @staticmethod
    def backward(ctx, dq, dk, dv):
        (x,) = ctx.saved_tensors
        x2 = x.reshape(-1, x.shape[-1])
        ds = [d.reshape(-1, d.shape[-1]) for d in (dq, dk, dv)]
        dx = torch.mm(ds[0], ctx.ws[0])
        dx.addmm_(ds[1], ctx.ws[1])
        dx.addmm_(ds[2], ctx.ws[2])
        for w, d in zip(ctx.ws, ds):
            ctx.grad_sink(w, d, x2)
        return dx.view_as(x), None, None, None, None


class _MLPInFn(torch.autograd.Function):
    """Both mlp_in halves with the GELU_AUX epilogue; backward accumulates
    dX = du1 W1a + du2 W1b in the GEMM epilogue."""

    @staticmethod
    def forward(ctx, x, wa, wb, grad_sink):
        from . import kernels as K
        ctx.set_materialize_grads(False)
        ctx.ws, ctx.grad_sink = (wa, wb), grad_sink
        ctx.save_for_backward(x)
        x2 = x.reshape(-1, x.shape[-1])
        u1, g1 = K.gemm_gelu_fwd(x2, wa)
        u2, g2 = K.gemm_gelu_fwd(x2, wb)
        ctx.mark_non_differentiable(g1, g2)
        shp = x.shape[:-1] + (wa.shape[0],)
        return u1.view(shp), g1.view(shp), u2.view(shp), g2.view(shp)

    @staticmethod
    def backward(ctx, du1, _dg1, du2, _dg2):
        (x,) = ctx.saved_tensors
        x2 = x.reshape(-1, x.shape[-1])
        d1, d2 = du1.reshape(-1, du1.shape[-1]), du2.reshape(-1, du2.shape[-1])
        dx = torch.mm(d1, ctx.ws[0])
        dx.addmm_(d2, ctx.ws[1])
        ctx.grad_sink(ctx.ws[0], d1, x2)
        ctx.grad_sink(ctx.ws[1], d2, x2)
        return dx.view_as(x), None, None, None


class _FusedXentFn(torch.autograd.Function):
    """Mean token cross entropy of fp16/bf16 logits via cs_xent_fwd/bwd; the
    gradient overwrites the (dead) logits buffer."""

    @staticmethod
    def forward(ctx, logits: torch.Tensor, targets: torch.Tensor):
        from . import kernels as K
        loss_rows, lse = K.xent_fwd(logits, targets)
        ctx.save_for_backward(logits, targets, lse)
        return loss_rows.mean()

    @staticmethod
    def backward(ctx, dloss: torch.Tensor):
        from . import kernels as K
        logits, targets, lse = ctx.saved_tensors
        K.xent_bwd_(logits, targets, lse, dloss, 1.0 / logits.shape[0])
        return logits, None


def fused_cross_entropy(logits: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
    return _FusedXentFn.apply(logits, targets)


def write_grad_into_slot(w: nn.Parameter, dy2: torch.Tensor, x2: torch.Tensor) -> None:
    """dW = dy^T x written over the parameter's own chunk slot."""
    torch.mm(dy2.t(), x2, out=w.data)


class _SlotEnter(torch.autograd.Function):
    @staticmethod
    def forward(ctx, driver, ev_fwd, ev_bwd, *xs):
        ctx.set_materialize_grads(False)
        ctx.driver, ctx.ev_bwd = driver, ev_bwd
        driver.start(ev_fwd)
        return tuple(x.view_as(x) for x in xs) if len(xs) > 1 else xs[0].view_as(xs[0])

    @staticmethod
    def backward(ctx, *grads):
        ctx.driver.finish(ctx.ev_bwd)
        return (None, None, None) + grads


class _SlotExit(torch.autograd.Function):
    @staticmethod
    def forward(ctx, driver, ev_fwd, ev_bwd, *ys):
        ctx.set_materialize_grads(False)
        ctx.driver, ctx.ev_bwd = driver, ev_bwd
        driver.finish(ev_fwd)
        return tuple(y.view_as(y) for y in ys) if len(ys) > 1 else ys[0].view_as(ys[0])

    @staticmethod
    def backward(ctx, *grads):
        ctx.driver.start(ctx.ev_bwd)
        return (None, None, None) + grads


def grad_in_data(p: nn.Parameter) -> bool:
    """True once this step's gradient was written over ``p.data`` itself (the
    reference's grad overwrite, `engine.py:177-190`) instead of ``p.grad``;
    the executor consumes it at ADAM and clears the mark."""
    return getattr(p, "_cs_grad_in_data", False)


def mark_grad_in_data(p: nn.Parameter, value: bool = True) -> None:
    p._cs_grad_in_data = value


class _DeviceEmbedding(torch.autograd.Function):
    """GPU-placed embedding lookup on the sm_100a kernels (cs_embed_fwd/bwd):
    the host operator's exact semantics (embedding.py), one backward kernel
    instead of torch's sort + segmented-reduce + scatter pipeline.  The
    gradients are written over the weights' own storage (grad overwrite); a
    tied LM head has already written its dW over wte, so the lookup's
    gradient is added to it (K4 accumulate, fused into the kernel)."""

    @staticmethod
    def forward(ctx, tokens, wte, wpe):
        from . import kernels as K
        ctx.save_for_backward(tokens)
        ctx.wte, ctx.wpe = wte, wpe
        return K.embed_fwd(tokens, wte, wpe)

    @staticmethod
    def backward(ctx, grad):
        from . import kernels as K
        (tokens,) = ctx.saved_tensors
        wte, wpe = ctx.wte, ctx.wpe
        K.embed_bwd_into(tokens, grad, wte.data, wpe.data, accumulate=grad_in_data(wte))
        mark_grad_in_data(wte)
        mark_grad_in_data(wpe)
        return None, None, None


class _LMHead(torch.autograd.Function):
    """logits = h Wᵀ; the backward computes dh = dlogits W first and then
    writes dW = dlogitsᵀ h over W's own storage (grad overwrite): W is not
    read again this step (the embedding lookup's backward needs only the
    token ids)."""

    @staticmethod
    def forward(ctx, h, w):
        ctx.save_for_backward(h)
        ctx.w = w
        return F.linear(h, w)

    @staticmethod
    def backward(ctx, dlogits):
        (h,) = ctx.saved_tensors
        w = ctx.w
        d2 = dlogits.reshape(-1, dlogits.shape[-1])
        dh = torch.mm(d2, w)
        torch.mm(d2.t(), h.reshape(-1, h.shape[-1]), out=w.data)
        mark_grad_in_data(w)
        return dh.view_as(h), None


class _EmbeddingMark(torch.autograd.Function):
    """embedding.fwd finishes at the lookup; embedding.bwd is the gradient
    arriving at the embedding output (after l0.qkv.bwd), start and finish."""

    @staticmethod
    def forward(ctx, driver, ev_fwd, ev_bwd, h):
        ctx.driver, ctx.ev_bwd = driver, ev_bwd
        driver.finish(ev_fwd)
        return h.view_as(h)

    @staticmethod
    def backward(ctx, grad):
        ctx.driver.start(ctx.ev_bwd)
        ctx.driver.finish(ctx.ev_bwd)
        return None, None, None, grad


class EventDriver:
    """Forwards marker callbacks to the engine; inert when no engine is attached.

    While a checkpointed layer is recomputed (``recomputing``), the FWD event
    indices its markers carry are remapped to the layer's RE_FWD events."""

    def __init__(self):
        self.on_start: Optional[Callable[[int], None]] = None
        self.on_finish: Optional[Callable[[int], None]] = None
        self.refwd_of: dict = {}
        self.recomputing = False

    def _map(self, ev: int) -> int:
        return self.refwd_of.get(ev, -1) if self.recomputing else ev

    def start(self, ev: int) -> None:
        ev = self._map(ev)
        if self.on_start is not None and ev >= 0:
            self.on_start(ev)

    def finish(self, ev: int) -> None:
        ev = self._map(ev)
        if self.on_finish is not None and ev >= 0:
            self.on_finish(ev)


class _LayerCheckpoint(torch.autograd.Function):
    """Activation checkpointing of one GPT block (`model.py:294-306`).

    Forward runs the block without a graph and keeps only the layer input
    (the reference's checkpointed activation is this one ``u`` per layer).
    Backward re-runs the block with the driver in RE_FWD mode — its four
    RE_FWD events fire, with any ``regather_refwd`` all-gathers — and then
    back-propagates through the recomputed graph, whose markers fire the
    layer's BWD events: exactly the checkpointed timeline order."""

    @staticmethod
    def forward(ctx, block, h_in):
        ctx.block = block
        ctx.save_for_backward(h_in)
        with torch.no_grad():
            return block(h_in)

    @staticmethod
    def backward(ctx, dout):
        (h_in,) = ctx.saved_tensors
        block = ctx.block
        h = h_in.detach().requires_grad_(True)
        block.driver.recomputing = True
        try:
            with torch.enable_grad():
                out = block(h)
        finally:
            block.driver.recomputing = False
        torch.autograd.backward(out, dout)
        return None, h.grad


def _bracket(marker, driver, ev_fwd, ev_bwd, xs):
    out = marker.apply(driver, ev_fwd, ev_bwd, *xs)
    return out if isinstance(out, tuple) else (out,)


class GPTBlock(nn.Module):
    def __init__(self, schema: ModelSchema, layer: int, driver: EventDriver,
                 dtype: torch.dtype, grad_sink: Callable, placeholders: bool = False,
                 fused: bool = False):
        super().__init__()
        self.fused = fused
        self.fused_ln = False  # set when the LN kernels support the width (attach time)
        H = schema.hidden_dim
        self.heads, self.layer, self.driver, self.grad_sink = schema.heads, layer, driver, grad_sink
        shapes = {"qkv": [(H, H)] * 3, "attn_out": [(H, H)], "mlp_in": [(2 * H, H)] * 2,
                  "mlp_out": [(H, 2 * H)] * 2}
        self.slots = nn.ModuleDict()
        for name, _ in OP_SLOTS:
            self.slots[name] = nn.ParameterList(
                [nn.Parameter(torch.empty(0 if placeholders else s, dtype=dtype),
                              requires_grad=True)
                 for s in shapes[name]])
        # (fwd event index, bwd event index) per slot, filled by attach_events
        self.events = {name: (-1, -1) for name, _ in OP_SLOTS}

    def _lin(self, x, w):
        return _ChunkLinearFn.apply(x, w, self.grad_sink)

    def _lin_res(self, x, w, residual):
        if not self.fused:
            return residual + self._lin(x, w)
        return _ChunkLinearResFn.apply(x, w, residual, self.grad_sink)

    def _slot(self, name, xs, fn):
        fwd, bwd = self.events[name]
        xs = _bracket(_SlotEnter, self.driver, fwd, bwd, xs)
        ys = fn(*xs)
        return _bracket(_SlotExit, self.driver, fwd, bwd, ys)

    def _ln(self, h):
        """(LN(h), residual h) — fused kernels when the width is supported."""
        if self.fused and self.fused_ln:
            return _LNResFn.apply(h)
        return F.layer_norm(h, (h.shape[-1],)), h

    def forward(self, h: torch.Tensor) -> torch.Tensor:
        B, S, H = h.shape
        nh = self.heads
        a, h = self._ln(h)
        wq, wk, wv = self.slots["qkv"]
        if self.fused:
            q, k, v = self._slot("qkv", (a,), lambda x: _QKVFn.apply(x, wq, wk, wv,
                                                                      self.grad_sink))
        else:
            q, k, v = self._slot("qkv", (a,), lambda x: (self._lin(x, wq), self._lin(x, wk),
                                                         self._lin(x, wv)))

        def heads(t):
            return t.view(B, S, nh, H // nh).transpose(1, 2)

        o = F.scaled_dot_product_attention(heads(q), heads(k), heads(v), is_causal=True)
        o = o.transpose(1, 2).reshape(B, S, H)
        (wo,) = self.slots["attn_out"]
        (h,) = self._slot("attn_out", (o, h), lambda x, r: (self._lin_res(x, wo, r),))
        b, h = self._ln(h)
        w1a, w1b = self.slots["mlp_in"]
        w2a, w2b = self.slots["mlp_out"]
        if self.fused:  # GELU in the GEMM epilogues (forward GELU_AUX, backward DGELU)
            sink = self.grad_sink
            u1, g1, u2, g2 = self._slot(
                "mlp_in", (b,), lambda x: _MLPInFn.apply(x, w1a, w1b, sink))
            (h,) = self._slot(
                "mlp_out", (g1, u1, g2, u2, h),
                lambda a1, v1, a2, v2, r: (_GeluLinearResFn.apply(
                    a2, v2, w2b, _GeluLinearResFn.apply(a1, v1, w2a, r, sink), sink),))
            return h
        u1, u2 = self._slot("mlp_in", (b,), lambda x: (self._lin(x, w1a), self._lin(x, w1b)))
        g1, g2 = F.gelu(u1, approximate="tanh"), F.gelu(u2, approximate="tanh")
        (h,) = self._slot("mlp_out", (g1, g2, h),
                          lambda x1, x2, r: (self._lin_res(x2, w2b, self._lin_res(x1, w2a, r)),))
        return h


class ReferenceShapedGPT(nn.Module):
    """GPT with tied embedding/LM head; see module docstring."""

    def __init__(self, schema: ModelSchema, dtype: torch.dtype = torch.float16,
                 grad_sink: Callable = write_grad_into_slot, placeholders: bool = False,
                 fused: bool = False, untied_head: bool = False):
        """``placeholders``: parameters start as empty tensors; their ``.data``
        is bound to chunk slots (or embedding buffers) by the executor.
        ``untied_head``: the LM head has its own [V, H] weight (used when the
        embedding is CPU-placed, :mod:`.embedding`)."""
        super().__init__()
        self.schema = schema
        self.driver = EventDriver()
        V, S, H = schema.vocab, schema.seq_len, schema.hidden_dim
        self.wte = nn.Parameter(torch.empty(0 if placeholders else (V, H), dtype=dtype))
        self.wpe = nn.Parameter(torch.empty(0 if placeholders else (S, H), dtype=dtype))
        self.lm_head = (nn.Parameter(torch.empty(0 if placeholders else (V, H), dtype=dtype))
                        if untied_head else None)
        #: a CPU-placed embedding operator (HostEmbedding); None = GPU lookup
        self.host_embedding = None
        self.fused = fused
        self.checkpointing = False
        self.blocks = nn.ModuleList([GPTBlock(schema, l, self.driver, dtype, grad_sink,
                                              placeholders, fused)
                                     for l in range(schema.layers)])
        self.embedding_events = (-1, -1)

    def chunk_parameters(self) -> List[nn.Parameter]:
        """Chunk-managed parameters in tensor-id order (== param_tensor_specs)."""
        out: List[nn.Parameter] = []
        for blk in self.blocks:
            for name, _ in OP_SLOTS:
                out.extend(blk.slots[name])
        return out

    def embedding_parameters(self) -> List[nn.Parameter]:
        return [self.wte, self.wpe]

    def attach_events(self, timeline) -> None:
        """Map every slot / the embedding to its (FWD, BWD) timeline indices."""
        idx = {ev.name: ev.index for ev in timeline.events}
        self.driver.refwd_of = {}
        for blk in self.blocks:
            for name, _ in OP_SLOTS:
                fwd = idx["l%d.%s.fwd" % (blk.layer, name)]
                blk.events[name] = (fwd, idx["l%d.%s.bwd" % (blk.layer, name)])
                refwd = idx.get("l%d.%s.refwd" % (blk.layer, name))
                if refwd is not None:
                    self.driver.refwd_of[fwd] = refwd
        self.embedding_events = (idx["embedding.fwd"], idx["embedding.bwd"])
        self.checkpointing = timeline.checkpointed

    def forward(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        B, S = tokens.shape
        efwd, ebwd = self.embedding_events
        self.driver.start(efwd)
        if self.host_embedding is not None:
            h = self.host_embedding.forward(tokens)
        elif self.fused:
            h = _DeviceEmbedding.apply(tokens, self.wte, self.wpe)
        else:
            h = F.embedding(tokens, self.wte) + self.wpe[:S]
        h = _EmbeddingMark.apply(self.driver, efwd, ebwd, h)
        for blk in self.blocks:
            h = _LayerCheckpoint.apply(blk, h) if self.checkpointing else blk(h)
        if self.fused and self.blocks and self.blocks[0].fused_ln:
            h = _LNFn.apply(h)
        else:
            h = F.layer_norm(h, (self.schema.hidden_dim,))
        head = self.wte if self.lm_head is None else self.lm_head
        logits = _LMHead.apply(h, head) if self.fused else F.linear(h, head)
        if self.fused:  # sm_100a fused loss kernels (cs_xent_fwd/bwd)
            return fused_cross_entropy(logits.view(B * S, -1), targets.reshape(B * S))
        return F.cross_entropy(logits.float().view(B * S, -1), targets.reshape(B * S))


def init_std() -> float:
    return 0.02


def reference_tensor_shapes(schema: ModelSchema) -> List[Tuple[int, int]]:
    """Shapes in tensor-id order, matching param_tensor_specs numels."""
    H = schema.hidden_dim
    per_layer = [(H, H)] * 4 + [(2 * H, H)] * 2 + [(H, 2 * H)] * 2
    shapes = per_layer * schema.layers
    specs = param_tensor_specs(schema)
    assert [a * b for a, b in shapes] == [s.numel for s in specs]
    return shapes
