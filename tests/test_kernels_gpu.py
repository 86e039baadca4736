"""GPU parity of the sm_100a chunk kernels vs the C oracle (bit-exact).

K1 fused chunk Adam, K2 grad sum-of-squares (+ deterministic finalize and
the device-side step scalars), K3 pack, K4 accumulate, K5 cast+pack, K6
optimizer-state birth.  Inputs are seeded; sizes cover tails (n % 4, n % 8),
multi-item launches (> 256 items → several launches), unaligned slot
offsets, fp16 and bf16, L2 and decoupled weight decay, and the skip path.
"""

import random

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

from paper_2108_05818_b200 import kernels as K  # noqa: E402

DEV = "cuda"


def _bits16(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16).copy()


def _code(O, dtype):
    return O.FP16 if dtype == torch.float16 else O.BF16


def _oracle_state(O, st: "K.N.CsStepState"):
    s = O.OrStepState()
    for f, _ in s._fields_:
        setattr(s, f, getattr(st, f))
    return s


@pytest.fixture(params=[0, 1],
                ids=lambda v: "variant%d" % v)
def adam_variant(request, native_lib):
    old = native_lib.cs_adam_variant(-1)
    native_lib.cs_adam_variant(request.param)
    assert native_lib.cs_adam_variant(-1) == request.param
    yield request.param
    native_lib.cs_adam_variant(old)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("wd,adamw", [(0.0, False), (0.1, False), (0.01, True)])
def test_adam_chunks_bit_exact(native_lib, oracle_lib, adam_variant, dtype, wd, adamw):
    O = oracle_lib
    g = torch.Generator(device="cpu").manual_seed(11)
    sizes = [1, 3, 4, 5, 4095, 4096, 4097, 70001, (1 << 20) + 7]
    hyper = K.AdamHyper(lr=3e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd, adamw=adamw)
    state = K.StepState(DEV, init_loss_scale=4.0)
    state.sumsq().fill_(5.0)
    K.adam_prepare(state, hyper)
    host_state = state.read()
    items, ref = [], []
    for n in sizes:
        gr = (torch.randn(n, generator=g) * 1e-2).to(dtype)
        p = torch.randn(n, generator=g) * 0.02
        m = torch.randn(n, generator=g) * 1e-3
        v = torch.rand(n, generator=g) * 1e-5
        ref.append([_bits16(gr), p.numpy().copy(), m.numpy().copy(), v.numpy().copy()])
        items.append((gr.to(DEV), p.to(DEV), m.to(DEV), v.to(DEV), n))
    K.adam_chunks(items, hyper, state)
    torch.cuda.synchronize()
    s = _oracle_state(O, host_state)
    for (gr, p, m, v, n), (rg, rp, rm, rv) in zip(items, ref):
        O.adam(rg, rp, rm, rv, n, _code(O, dtype), 3e-4, 0.9, 0.999, 1e-8, wd, adamw, s)
        np.testing.assert_array_equal(p.cpu().numpy().view(np.uint32), rp.view(np.uint32))
        np.testing.assert_array_equal(m.cpu().numpy().view(np.uint32), rm.view(np.uint32))
        np.testing.assert_array_equal(v.cpu().numpy().view(np.uint32), rv.view(np.uint32))
        np.testing.assert_array_equal(_bits16(gr), rg)


def test_adam_chunks_many_items_and_prefix_only(native_lib, oracle_lib, adam_variant):
    """300 items plus 43 zero-length ones interleaved (two launches, the
    batch boundary falls among empty items); only the used prefix of each
    chunk changes and every item is updated exactly once (a double update
    would not match the oracle's single step)."""
    O = oracle_lib
    cap, used = 8192, 5000
    hyper = K.AdamHyper(lr=1e-3)
    state = K.StepState(DEV)
    state.sumsq().fill_(1.0)
    K.adam_prepare(state, hyper)
    s = _oracle_state(O, state.read())
    chunks = []
    for i in range(300):
        gen = torch.Generator().manual_seed(i)
        p16 = (torch.randn(cap, generator=gen) * 1e-3).half()
        p32 = torch.randn(cap, generator=gen) * 0.02
        m = torch.zeros(cap)
        v = torch.zeros(cap)
        chunks.append([x.to(DEV) for x in (p16, p32, m, v)] + [x.numpy().copy() for x in (p32, m, v)]
                      + [_bits16(p16)])
    items = []
    for i, c in enumerate(chunks):
        items.append((c[0], c[1], c[2], c[3], used))
        if i % 7 == 3:  # an empty item takes no batch slot
            items.append((c[0], c[1], c[2], c[3], 0))
    assert len(items) > 256 + 30
    K.adam_chunks(items, hyper, state)
    torch.cuda.synchronize()
    for c in chunks:
        rp, rm, rv, rg = c[4], c[5], c[6], c[7]
        tail = rg[used:].copy(), rp[used:].copy()
        O.adam(rg, rp, rm, rv, used, O.FP16, 1e-3, 0.9, 0.999, 1e-8, 0.0, False, s)
        np.testing.assert_array_equal(c[1].cpu().numpy().view(np.uint32), rp.view(np.uint32))
        np.testing.assert_array_equal(_bits16(c[0]), rg)
        np.testing.assert_array_equal(_bits16(c[0])[used:], tail[0])


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_adam_skip_restores_params_and_leaves_state(native_lib, oracle_lib, adam_variant, dtype):
    """Skipped step (non-finite gradients): p32 / m / v untouched, and the
    16-bit chunk — which holds the step's (overflowed) gradients under the
    grad overwrite — gets the unchanged parameters back, p16 = round(p32);
    same bits as the oracle.  Ragged sizes, several items."""
    O = oracle_lib
    hyper = K.AdamHyper()
    state = K.StepState(DEV, init_loss_scale=65536.0)
    state.sumsq().fill_(float("inf"))
    K.adam_prepare(state, hyper, dynamic_scale=True)
    st = state.read()
    assert st.skip == 1 and st.step == 0 and st.loss_scale == 32768.0
    g = torch.Generator().manual_seed(8)
    items, refs = [], []
    for n in (1, 1000, 4099, 70001):
        p32 = torch.randn(n, generator=g)
        p16 = torch.full((n,), float("inf"), dtype=dtype)
        m, v = torch.randn(n, generator=g), torch.rand(n, generator=g)
        refs.append((_bits16(p16), p32.numpy().copy(), m.numpy().copy(), v.numpy().copy()))
        items.append((p16.to(DEV), p32.to(DEV), m.to(DEV), v.to(DEV), n))
    K.adam_chunks(items, hyper, state)
    torch.cuda.synchronize()
    s = _oracle_state(O, st)
    for (d16, d32, dm, dv, n), (r16, r32, rm, rv) in zip(items, refs):
        O.adam(r16, r32, rm, rv, n, _code(O, dtype), 1e-4, 0.9, 0.999, 1e-8, 0.0, False, s)
        assert np.array_equal(d32.cpu().numpy(), r32) and np.array_equal(dm.cpu().numpy(), rm)
        assert np.array_equal(dv.cpu().numpy(), rv)
        assert np.array_equal(_bits16(d16), r16)
        assert torch.equal(d16.cpu(), d32.cpu().to(dtype))  # the parameters are back


def _sumsq(items, state, dtype=None, slots=None, n_slots=None):
    scratch = torch.empty(max(K.sumsq_scratch(items), 1), device=DEV)
    sums = torch.zeros(n_slots if n_slots is not None else len(items), dtype=torch.float64,
                       device=DEV)
    K.grad_sumsq(items, scratch, sums, slots=slots, dtype=dtype)
    K.sumsq_finalize(sums, state)
    return sums


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_grad_sumsq_canonical_bit_exact(native_lib, oracle_lib, dtype):
    """K2 = the C oracle's restatement of the canonical order, bit for bit,
    per item (whole and ragged tiles, empty items, an item misaligned for
    128-bit loads) and for the slot fold; = the host twin on the same bytes."""
    O = oracle_lib
    code = O.FP16 if dtype == torch.float16 else O.BF16
    gen = torch.Generator().manual_seed(9)
    base = (torch.randn(3 * 8192 + 9000, generator=gen) * 0.05).to(dtype)
    host_items = [(base[:n], n) for n in (1, 8191, 8192, 8193, 3 * 8192 + 4100)]
    host_items += [(base[:0], 0), (base[3:3 + 20000], 20000)]  # empty; 6-byte offset
    dev = base.to(DEV)
    items = [(dev[:n], n) for n in (1, 8191, 8192, 8193, 3 * 8192 + 4100)]
    items += [(dev[:0], 0), (dev[3:3 + 20000], 20000)]
    state = K.StepState(DEV)
    sums = _sumsq(items, state, dtype=dtype).cpu().numpy()
    want = [O.grad_sumsq_item(_bits16(t.contiguous()), code) if n else 0.0
            for t, n in host_items]
    assert sums.tobytes() == np.array(want, dtype=np.float64).tobytes()
    assert K.grad_sumsq_host([(t.contiguous(), n) for t, n in host_items]) == list(sums)
    assert np.float32(state.read().sumsq) == np.float32(O.sumsq_total(want))


def test_grad_sumsq_slots_and_batches(native_lib, oracle_lib):
    """Slot order is the fold order whatever the item order or the launch
    batching (more items than one launch takes)."""
    gen = torch.Generator().manual_seed(4)
    grads = [(torch.randn(500 + 37 * i, generator=gen) * 0.1).half().to(DEV) for i in range(300)]
    perm = list(range(300))
    random.Random(1).shuffle(perm)
    s1, s2 = K.StepState(DEV), K.StepState(DEV)
    a = _sumsq([(g, g.numel()) for g in grads], s1)
    b = _sumsq([(grads[i], grads[i].numel()) for i in perm], s2, slots=perm, n_slots=300)
    assert torch.equal(a, b) and s1.read().sumsq == s2.read().sumsq


def test_grad_sumsq_and_step_scalars_match_oracle(native_lib, oracle_lib):
    O = oracle_lib
    gen = torch.Generator().manual_seed(5)
    grads = [(torch.randn(n, generator=gen) * 3).half() for n in (1, 4097, 300000, 1 << 21)]
    state = K.StepState(DEV, init_loss_scale=2.0)
    _sumsq([(x.to(DEV), x.numel()) for x in grads], state)
    hyper = K.AdamHyper(lr=1e-3, betas=(0.9, 0.99))
    K.adam_prepare(state, hyper, max_grad_norm=1.0, dynamic_scale=True, growth_interval=1)
    st = state.read()
    ref = sum(O.grad_sumsq(_bits16(x), O.FP16) for x in grads)
    assert abs(st.sumsq - ref) <= 1e-5 * ref
    s = O.step_state(2.0)
    s.sumsq = st.sumsq  # same input -> identical scalars
    O.adam_prepare(s, 1e-3, 0.9, 0.99, max_norm=1.0, dynamic=True, interval=1)
    for f in ("grad_scale", "step_size", "sqrt_bc2", "grad_norm", "loss_scale", "step", "skip",
              "beta1_pow", "beta2_pow"):
        assert getattr(st, f) == getattr(s, f), f
    # determinism: same inputs, bit-identical sumsq
    _sumsq([(x.to(DEV), x.numel()) for x in grads], state)
    assert state.read().sumsq == st.sumsq


def test_grad_sumsq_detects_inf(native_lib):
    g = torch.randn(10000, device=DEV).half()
    g[1234] = float("inf")
    state = K.StepState(DEV)
    _sumsq([(g, g.numel())], state)
    assert not np.isfinite(state.read().sumsq)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("accumulate", [False, True])
def test_pack_and_accumulate_bit_exact(native_lib, oracle_lib, dtype, accumulate):
    O = oracle_lib
    gen = torch.Generator().manual_seed(2)
    cap = 200003
    chunk = (torch.randn(cap, generator=gen)).to(dtype)
    # aligned, unaligned and tail-heavy slots (gap-free packing offsets)
    slots = [(0, 65536), (65536, 131072 - 65536 + 5), (131077, 3), (131080, 68923)]
    srcs = [(torch.randn(n, generator=gen)).to(dtype) for _, n in slots]
    ref = _bits16(chunk)
    for (off, n), s in zip(slots, srcs):
        O.pack(ref, off, _bits16(s), _code(O, dtype), accumulate)
    dchunk = chunk.to(DEV)
    K.pack([(dchunk, off, s.to(DEV), n) for (off, n), s in zip(slots, srcs)], accumulate=accumulate)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits16(dchunk), ref)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_cast_pack_bit_exact(native_lib, oracle_lib, dtype):
    O = oracle_lib
    gen = torch.Generator().manual_seed(4)
    cap = 100000
    chunk = torch.zeros(cap, dtype=dtype)
    slots = [(0, 4096), (4096, 12345), (16441, 7), (16448, 83552)]
    srcs = [torch.randn(n, generator=gen) * 0.02 for _, n in slots]
    ref = _bits16(chunk)
    for (off, n), s in zip(slots, srcs):
        O.cast_pack(ref, off, s.numpy().copy(), _code(O, dtype))
    dchunk = chunk.to(DEV)
    K.cast_pack([(dchunk, off, s.to(DEV), n) for (off, n), s in zip(slots, srcs)])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits16(dchunk), ref)
    # and the GPU cast equals torch's own RN cast
    np.testing.assert_array_equal(_bits16(dchunk[:4096].cpu()), _bits16(srcs[0].to(dtype)))


@pytest.mark.parametrize("src_dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("pinned_host", [False, True])
def test_master_init(native_lib, src_dtype, pinned_host):
    n = 70001
    src = (torch.randn(n) * 0.02).to(src_dtype)
    src = src.pin_memory() if pinned_host else src.to(DEV)
    p32 = torch.full((n,), 7.0, device=DEV)
    m = torch.full((n,), 7.0, device=DEV)
    v = torch.full((n,), 7.0, device=DEV)
    K.master_init(p32, m, v, src, n)
    torch.cuda.synchronize()
    assert torch.equal(p32.cpu(), src.cpu().float())
    assert (m == 0).all() and (v == 0).all()


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("vocab", [50304, 1001])
def test_fused_cross_entropy_vs_torch_fp32(native_lib, dtype, vocab):
    """cs_xent_fwd/bwd vs a plain PyTorch fp32 reference (F.cross_entropy on
    upcast logits).  Tolerances: loss rel 1e-5; dlogits within 2 ulps of the
    16-bit result of the fp32 reference gradient."""
    gen = torch.Generator(device=DEV).manual_seed(9)
    rows = 333
    logits = (torch.randn(rows, vocab, device=DEV, generator=gen) * 3).to(dtype)
    targets = torch.randint(0, vocab, (rows,), device=DEV, generator=gen)
    ref_in = logits.float().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(ref_in, targets)
    dloss = torch.tensor(1024.0, device=DEV)
    ref.backward(dloss)
    loss_rows, lse = K.xent_fwd(logits, targets)
    loss = loss_rows.mean()
    assert abs(loss.item() - ref.item()) <= 1e-5 * abs(ref.item())
    g = logits.clone()
    K.xent_bwd_(g, targets, lse, dloss, 1.0 / rows)
    ref_g = ref_in.grad.to(dtype).float()
    err = (g.float() - ref_g).abs()
    ulp = ref_g.abs().clamp_min(1e-30) * (2 ** -10 if dtype == torch.float16 else 2 ** -7)
    assert (err <= 2 * ulp + 1e-6).all(), float((err / (ulp + 1e-12)).max())


def test_fused_gpt_matches_unfused_gpt(native_lib):
    """Residual adds and GELU in the GEMM epilogues + the fused loss give the
    same gradients as the unfused model (one step; loss within 1e-3, every
    dW within 4e-3 of its max-norm — a few fp16 ulps at that scale)."""
    from paper_2108_05818_b200.gpt import ReferenceShapedGPT
    from paper_2108_05818_b200.model import build_gpt_schema
    schema = build_gpt_schema(layers=2, hidden_dim=256, heads=4, seq_len=64, vocab=1000,
                              batch=2)
    models = {}
    for fused in (False, True):
        torch.manual_seed(0)
        m = ReferenceShapedGPT(schema, dtype=torch.float16, fused=fused).to(DEV)
        for blk in m.blocks:
            blk.fused_ln = fused  # cs_layernorm kernels (H=256 supported)
        for p in m.parameters():
            torch.nn.init.normal_(p, std=0.02)
        models[fused] = m
    tok = torch.randint(0, 1000, (2, 65), device=DEV, generator=torch.Generator(device=DEV).manual_seed(1))
    out = {}
    for fused, m in models.items():
        loss = m(tok[:, :-1], tok[:, 1:])
        (loss * 256).backward()
        # chunk slots hold the dW; the fused model also writes the tied
        # embedding/head and position gradients over wte / wpe (grad overwrite
        # + the lookup's accumulate), the plain model leaves them in .grad
        emb = [p.data.clone() if fused else p.grad.clone() for p in (m.wte, m.wpe)]
        out[fused] = (loss.item(), [p.data.clone() for p in m.chunk_parameters()] + emb)
    assert abs(out[True][0] - out[False][0]) < 1e-3
    for a, b in zip(out[True][1], out[False][1]):
        # max-norm relative error within a few fp16 ulps of the tensor's scale
        err = (a.float() - b.float()).abs().max()
        assert err <= 4e-3 * b.float().abs().max(), float(err)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_gemm_gelu_epilogues_vs_torch_fp32(native_lib, dtype):
    """cuBLASLt GELU_AUX / DGELU epilogues vs a plain PyTorch fp32 reference
    (tanh-approximate GELU).  Tolerance: 16-bit output rounding + fp32
    accumulation order (rtol 2e-2 fp16 / 5e-2 bf16 relative to the row scale)."""
    gen = torch.Generator(device=DEV).manual_seed(3)
    T, K_, O = 1000, 256, 512
    x = (torch.randn(T, K_, device=DEV, generator=gen)).to(dtype)
    w = (torch.randn(O, K_, device=DEV, generator=gen) * 0.05).to(dtype)
    u, g = K.gemm_gelu_fwd(x, w)
    u_ref = x.float() @ w.float().t()
    g_ref = torch.nn.functional.gelu(u_ref, approximate="tanh")
    tol = 2e-2 if dtype == torch.float16 else 5e-2
    scale = u_ref.abs().amax(dim=1, keepdim=True)
    assert ((u.float() - u_ref).abs() <= tol * scale).all()
    assert ((g.float() - g_ref).abs() <= tol * scale).all()
    # backward: du = (dy @ W2) * gelu'(u), W2 [K,O] row-major
    dy = (torch.randn(T, K_, device=DEV, generator=gen)).to(dtype)
    w2 = (torch.randn(K_, O, device=DEV, generator=gen) * 0.05).to(dtype)
    du = K.gemm_dgelu(dy, w2, u)
    uu = u.float().requires_grad_(True)
    gg = torch.nn.functional.gelu(uu, approximate="tanh")
    gg.backward(dy.float() @ w2.float())
    ref = uu.grad
    s2 = ref.abs().amax(dim=1, keepdim=True)
    assert ((du.float() - ref).abs() <= tol * s2 + 1e-3).all()


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("H", [256, 2048, 2304])
def test_layernorm_kernels_vs_torch_fp32(native_lib, dtype, H):
    """cs_layernorm_fwd/bwd (non-affine, residual grad folded in) vs a plain
    PyTorch fp32 reference: outputs and dx within 2 ulps of the 16-bit result."""
    gen = torch.Generator(device=DEV).manual_seed(H)
    rows = 777
    x = (torch.randn(rows, H, device=DEV, generator=gen) * 3 + 1).to(dtype)
    dy = torch.randn(rows, H, device=DEV, generator=gen).to(dtype)
    dres = torch.randn(rows, H, device=DEV, generator=gen).to(dtype)
    y, mean, rstd = K.layernorm_fwd(x)
    xr = x.float().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (H,), eps=1e-5)
    yr.backward(dy.float())
    ref_dx = xr.grad + dres.float()
    dx = K.layernorm_bwd(dy, x, mean, rstd, dres)
    ulp = 2 ** -10 if dtype == torch.float16 else 2 ** -7
    for got, ref in ((y, yr.detach()), (dx, ref_dx)):
        err = (got.float() - ref).abs()
        assert (err <= 2 * ulp * ref.abs() + 4 * ulp * ref.abs().amax(dim=1, keepdim=True) * 1e-2
                + 1e-3).all(), float(err.max())
    assert not K.layernorm_supported(128)


def test_chunk_kernels_past_2pow31_elements(native_lib, oracle_lib):
    """Maximum sizes: one K1 item of 2^31 + 13 elements (30 GB of state,
    int64 tile/element indexing, ragged tail) and a K3/K5 pack at an offset
    past 2^31 — checked against the oracle on windows at the start, across
    the 2^31 boundary and at the end (the update is elementwise)."""
    O = oracle_lib
    n = (1 << 31) + 13
    free, _ = torch.cuda.mem_get_info()
    if free < 40 << 30:
        pytest.skip("needs ~40 GB of free HBM")
    g = torch.Generator(device=DEV).manual_seed(5)
    p16 = (torch.randn(n, device=DEV, generator=g) * 1e-2).half()
    p32 = torch.randn(n, device=DEV, generator=g) * 0.02
    m = torch.randn(n, device=DEV, generator=g) * 1e-3
    v = torch.rand(n, device=DEV, generator=g) * 1e-5
    wins = [(0, 8192), ((1 << 31) - 5000, (1 << 31) + 9), (n - 3, n)]
    before = [(_bits16(p16[a:b]), p32[a:b].cpu().numpy().copy(), m[a:b].cpu().numpy().copy(),
               v[a:b].cpu().numpy().copy()) for a, b in wins]
    hyper = K.AdamHyper(lr=1e-3)
    state = K.StepState(DEV)
    state.sumsq().fill_(1.0)
    K.adam_prepare(state, hyper)
    s = _oracle_state(O, state.read())
    K.adam_chunks([(p16, p32, m, v, n)], hyper, state)
    torch.cuda.synchronize()
    for (a, b), (rg, rp, rm, rv) in zip(wins, before):
        O.adam(rg, rp, rm, rv, b - a, O.FP16, 1e-3, 0.9, 0.999, 1e-8, 0.0, False, s)
        np.testing.assert_array_equal(p32[a:b].cpu().numpy().view(np.uint32), rp.view(np.uint32))
        np.testing.assert_array_equal(v[a:b].cpu().numpy().view(np.uint32), rv.view(np.uint32))
        np.testing.assert_array_equal(_bits16(p16[a:b]), rg)
    del m, v
    # K3 / K5 at an element offset past 2^31 (chunk = the 4 GB fp16 buffer)
    big = torch.zeros(n + 20000, dtype=torch.float16, device=DEV)
    off = (1 << 31) + 5
    src16 = (torch.randn(9001, device=DEV, generator=g)).half()
    src32 = torch.randn(9001, device=DEV, generator=g)
    K.pack([(big, off, src16, 9001)])
    torch.cuda.synchronize()
    assert torch.equal(big[off:off + 9001], src16)
    K.cast_pack([(big, off + 3, src32, 9001)])
    torch.cuda.synchronize()
    assert torch.equal(big[off + 3:off + 3 + 9001], src32.half())
    del big
    # K2 over all 2^31 + 13 elements vs a float64 torch reduction
    st = K.StepState(DEV)
    _sumsq([(p16, n)], st)
    ref = float((p16.double() ** 2).sum())
    assert abs(float(st.sumsq().item()) - ref) <= 1e-5 * ref


def test_adam_chunks_8_byte_aligned_items_take_the_simt_path(native_lib, oracle_lib):
    """The TMA variants need 16-byte aligned streams; an fp16 view offset by
    8 bytes is routed to the SIMT kernel (same bits), not rejected."""
    O = oracle_lib
    n = 70001
    g = torch.Generator().manual_seed(4)
    base16 = (torch.randn(n + 4, generator=g) * 1e-2).half()
    p = torch.randn(n, generator=g) * 0.02
    m = torch.randn(n, generator=g) * 1e-3
    v = torch.rand(n, generator=g) * 1e-5
    hyper = K.AdamHyper(lr=1e-3)
    state = K.StepState(DEV)
    state.sumsq().fill_(1.0)
    K.adam_prepare(state, hyper)
    s = _oracle_state(O, state.read())
    d16 = base16.to(DEV)[4:]            # data_ptr % 16 == 8
    assert d16.data_ptr() % 16 == 8
    dp, dm, dv = p.to(DEV), m.to(DEV), v.to(DEV)
    rg, rp, rm, rv = _bits16(base16[4:]), p.numpy().copy(), m.numpy().copy(), v.numpy().copy()
    K.adam_chunks([(d16, dp, dm, dv, n)], hyper, state)
    torch.cuda.synchronize()
    O.adam(rg, rp, rm, rv, n, O.FP16, 1e-3, 0.9, 0.999, 1e-8, 0.0, False, s)
    np.testing.assert_array_equal(dp.cpu().numpy().view(np.uint32), rp.view(np.uint32))
    np.testing.assert_array_equal(_bits16(d16), rg)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_gemm_res_vs_torch_fp32(native_lib, dtype):
    """cs_gemm_res: out = x·Wᵀ + res (residual read by the GEMM, res intact)
    vs a plain PyTorch fp32 reference; tolerance a few 16-bit ulps of the
    output scale."""
    g = torch.Generator(device=DEV).manual_seed(3)
    T, K_, O = 777, 512, 384
    x = torch.randn(T, K_, device=DEV, generator=g).to(dtype)
    w = (torch.randn(O, K_, device=DEV, generator=g) * 0.05).to(dtype)
    r = torch.randn(T, O, device=DEV, generator=g).to(dtype)
    r0 = r.clone()
    out = K.gemm_res(x, w, r)
    ref = x.float() @ w.float().t() + r.float()
    tol = (2 ** -9 if dtype == torch.float16 else 2 ** -6) * ref.abs().max()
    assert (out.float() - ref).abs().max() <= tol
    assert torch.equal(r, r0)


def test_k1_at_the_bench_layout_every_element_bit_exact(native_lib, oracle_lib):
    """K1 at BASELINE's full size: the 1B bench model's 15 chunk positions
    (cap 64Mi, 1,006,632,960 used elements, the chunk layout of
    `chunks.py:168-201`) in ONE default-variant launch, every element of p16,
    p32, m and v compared with the C oracle (slice by slice on the host)."""
    from paper_2108_05818_b200.chunks import build_model_chunk_lists
    from paper_2108_05818_b200.model import build_gpt_schema
    O = oracle_lib
    cap = 64 << 20
    schema = build_gpt_schema(layers=20, hidden_dim=2048, heads=16, seq_len=1024,
                              vocab=50304, batch=32)
    cs = build_model_chunk_lists(schema, cap)
    used = [cs.param_chunk(p).used_elems for p in range(cs.positions)]
    assert len(used) == 15 and sum(used) == 1_006_632_960
    g = torch.Generator(device=DEV).manual_seed(11)
    items, host = [], []
    for n in used:
        p16 = (torch.randn(cap, device=DEV, generator=g) * 1e-2).half()
        p32 = torch.randn(cap, device=DEV, generator=g) * 0.02
        m = torch.randn(cap, device=DEV, generator=g) * 1e-3
        v = torch.rand(cap, device=DEV, generator=g) * 1e-5
        items.append((p16, p32, m, v, n))
    hyper = K.AdamHyper(lr=1e-4)
    state = K.StepState(DEV)
    state.sumsq().fill_(4.0)
    K.adam_prepare(state, hyper)
    s = _oracle_state(O, state.read())
    # inputs to the host in 8Mi slices (bounded host memory per slice pair)
    sl = 8 << 20
    for p16, p32, m, v, n in items:
        host.append([(_bits16(p16[a:min(a + sl, n)]), p32[a:a + sl][:n - a].cpu().numpy(),
                      m[a:a + sl][:n - a].cpu().numpy(), v[a:a + sl][:n - a].cpu().numpy())
                     for a in range(0, n, sl)])
    tail = [(it[0][it[4]:].clone(), it[1][it[4]:].clone()) for it in items]
    K.adam_chunks(items, hyper, state)
    torch.cuda.synchronize()
    for (p16, p32, m, v, n), slices, (t16, t32) in zip(items, host, tail):
        for k, (rg, rp, rm, rv) in enumerate(slices):
            a = k * sl
            b = a + rg.size
            O.adam(rg, rp, rm, rv, b - a, O.FP16, 1e-4, 0.9, 0.999, 1e-8, 0.0, False, s)
            assert np.array_equal(_bits16(p16[a:b]), rg)
            assert np.array_equal(p32[a:b].cpu().numpy().view(np.uint32), rp.view(np.uint32))
            assert np.array_equal(m[a:b].cpu().numpy().view(np.uint32), rm.view(np.uint32))
            assert np.array_equal(v[a:b].cpu().numpy().view(np.uint32), rv.view(np.uint32))
        # the unused tail of each chunk is never touched
        assert torch.equal(p16[n:], t16) and torch.equal(p32[n:], t32)


def test_sumsq_and_pack_with_zero_length_items_across_batches(native_lib):
    """K2 and K3/K4 work lists longer than one launch's batch with empty
    items mixed in: every non-empty item is counted / packed exactly once."""
    gen = torch.Generator().manual_seed(11)
    grads, items = [], []
    for i in range(300):
        g = (torch.randn(1000 + i, generator=gen) * 0.1).half().to(DEV)
        grads.append(g)
        items.append((g, g.numel()))
        if i % 5 == 0:
            items.append((g, 0))
    assert len(items) > 256 + 30
    st = K.StepState(DEV)
    sums = _sumsq(items, st, dtype=torch.float16)
    want = sum(float((g.double() ** 2).sum()) for g in grads)
    assert abs(float(sums.sum()) - want) <= 1e-6 * want
    assert all(float(s) == 0.0 for (g, n), s in zip(items, sums.cpu()) if n == 0)
    for acc in (0, 1):
        dst = torch.zeros(sum(g.numel() for g in grads), dtype=torch.float16, device=DEV)
        pk, off = [], 0
        for g in grads:
            pk.append((dst, off, g, g.numel()))
            pk.append((dst, off, g, 0))
            off += g.numel()
        K.pack(pk, accumulate=bool(acc))
        torch.cuda.synchronize()
        assert torch.equal(dst, torch.cat(grads)), acc


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_nan_masters_narrow_like_the_host(native_lib, adam_variant, dtype):
    """A NaN master narrows to the same 16-bit pattern on the device (K1)
    and on the host (cs_adam_chunks_host): the canonical NaN 0x7fff."""
    n = 4096 + 24
    bits = np.array([0x7fc00000, 0xffc00000, 0x7fffffff, 0xffffffff, 0x7f800001, 0x7fbfffff,
                     0xff800001, 0x7ff0f0f0], dtype=np.uint32)
    p = np.resize(bits, n).view(np.float32)
    hyper = K.AdamHyper()
    state = K.StepState(DEV)
    state.sumsq().fill_(1.0)
    K.adam_prepare(state, hyper)
    dev = [torch.zeros(n, dtype=dtype, device=DEV), torch.from_numpy(p.copy()).to(DEV),
           torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)]
    K.adam_chunks([(*dev, n)], hyper, state)
    host = [torch.zeros(n, dtype=dtype), torch.from_numpy(p.copy()), torch.zeros(n),
            torch.zeros(n)]
    K.adam_chunks_host([(*host, n)], hyper, state.read(), n_threads=2)
    torch.cuda.synchronize()
    assert np.array_equal(_bits16(dev[0]), _bits16(host[0]))
    assert (_bits16(dev[0]) == 0x7fff).all(), hex(int(_bits16(dev[0])[0]))
