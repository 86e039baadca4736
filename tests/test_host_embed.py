"""Host embedding operator (CPU-placed embedding, PAPER §5 device-aware
placement; `profiler.py:70-74`, `engine.py:202-213`) vs the numpy oracle:
bit-exact.  Host product code, so it runs without a GPU.  The oracle's
forward is pinned to torch's own `F.embedding(tok, wte) + wpe[:S]`."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2108_05818_b200 import kernels as K

CODE = {torch.float16: 0, torch.bfloat16: 1}


def _bits(t):
    return t.view(torch.int16).numpy().view(np.uint16)


def _case(dtype, B, S, V, H, seed, repeat_tokens=False):
    g = torch.Generator().manual_seed(seed)
    hi = 7 if repeat_tokens else V
    tok = torch.randint(0, hi, (B, S), generator=g)
    wte = (torch.randn(V, H, generator=g) * 0.02).to(dtype)
    wpe = (torch.randn(S, H, generator=g) * 0.02).to(dtype)
    dout = (torch.randn(B, S, H, generator=g) * 4.0).to(dtype)
    return tok, wte, wpe, dout


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("B,S,V,H,rep", [(2, 16, 97, 64, False), (4, 128, 512, 256, True),
                                         (3, 5, 11, 8, False), (1, 1, 1, 16, False)])
def test_embed_fwd_bwd_bit_exact(native_lib, oracle_lib, dtype, B, S, V, H, rep):
    O = oracle_lib
    tok, wte, wpe, dout = _case(dtype, B, S, V, H, seed=B * 1000 + H, repeat_tokens=rep)
    out = torch.empty(B, S, H, dtype=dtype)
    K.embed_fwd_host(tok, wte, wpe, out, n_threads=4)
    ref = O.embed_fwd(tok.numpy(), _bits(wte), _bits(wpe), CODE[dtype])
    assert np.array_equal(_bits(out), ref)
    gwte = torch.full((V, H), 7.0, dtype=dtype)   # overwritten, including unhit rows
    gwpe = torch.full((S, H), 7.0, dtype=dtype)
    sq = K.embed_bwd_host(tok, dout, gwte, gwpe, n_threads=3)
    rw, rp = O.embed_bwd(tok.numpy(), _bits(dout), V, CODE[dtype])
    assert np.array_equal(_bits(gwte), rw)
    assert np.array_equal(_bits(gwpe), rp)
    # the fused sum of squares = the squares of the written (rounded) gradients
    ref_sq = sum(float((t.double() ** 2).sum()) for t in (gwte, gwpe))
    assert sq == pytest.approx(ref_sq, rel=1e-12, abs=0.0)
    # K2's host twin (fp32 lane sums in the canonical order) agrees to fp32 rounding
    assert sq == pytest.approx(sum(K.grad_sumsq_host([(gwte.view(-1), V * H),
                                                      (gwpe.view(-1), S * H)])), rel=1e-6)
    # deterministic for any thread count (row-order reduction)
    for threads in (1, 7):
        assert K.embed_bwd_host(tok, dout, gwte.clone(), gwpe.clone(), n_threads=threads) == sq


def test_oracle_forward_pinned_to_torch(oracle_lib):
    tok, wte, wpe, _ = _case(torch.float16, 4, 32, 300, 64, seed=5)
    ref = F.embedding(tok, wte) + wpe[:32]
    got = oracle_lib.embed_fwd(tok.numpy(), _bits(wte), _bits(wpe), 0)
    assert np.array_equal(_bits(ref.contiguous()), got)


def test_oracle_backward_close_to_float64():
    import oracle.numerics as O
    tok, _, _, dout = _case(torch.float16, 4, 32, 50, 64, seed=6, repeat_tokens=True)
    gw, gp = O.embed_bwd(tok.numpy(), _bits(dout), 50, 0)
    d = dout.double().view(-1, 64)
    ref = torch.zeros(50, 64, dtype=torch.float64).index_add_(0, tok.view(-1), d)
    np.testing.assert_allclose(gw.view(np.float16).astype(np.float64), ref.numpy(),
                               rtol=2e-3, atol=2e-3)
    np.testing.assert_allclose(gp.view(np.float16).astype(np.float64),
                               dout.double().sum(0).numpy(), rtol=2e-3, atol=2e-3)


def test_weights_may_be_overwritten_in_place(native_lib):
    """The trainer writes the gradient over the weight buffers themselves."""
    tok, wte, wpe, dout = _case(torch.float16, 2, 8, 13, 16, seed=9)
    a, b = torch.empty(13, 16, dtype=torch.float16), torch.empty(8, 16, dtype=torch.float16)
    K.embed_bwd_host(tok, dout, a, b)
    K.embed_bwd_host(tok, dout, wte, wpe)
    assert torch.equal(a, wte) and torch.equal(b, wpe)


def test_out_of_range_token_rejected(native_lib):
    from paper_2108_05818_b200._native import NativeError
    tok, wte, wpe, dout = _case(torch.float16, 1, 4, 10, 8, seed=1)
    tok[0, 2] = 10
    with pytest.raises(NativeError, match="out of"):
        K.embed_fwd_host(tok, wte, wpe, torch.empty(1, 4, 8, dtype=torch.float16))
    with pytest.raises(NativeError):
        K.embed_bwd_host(tok, dout, wte, wpe)


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("B,S,V,H,rep", [(2, 16, 97, 64, False), (4, 128, 512, 256, True),
                                         (3, 5, 11, 8, False), (8, 64, 50304, 2048, False)])
def test_device_embedding_bit_identical_to_host_and_oracle(native_lib, oracle_lib, dtype, B, S,
                                                           V, H, rep):
    """cs_embed_fwd/bwd (GPU-placed operator) == cs_embed_*_host == oracle."""
    O = oracle_lib
    tok, wte, wpe, dout = _case(dtype, B, S, V, H, seed=B * 7 + H, repeat_tokens=rep)
    wpe_big = torch.cat([wpe, (torch.randn(3, H) * 0.02).to(dtype)])  # wpe has spare rows
    out = K.embed_fwd(tok.cuda(), wte.cuda(), wpe_big.cuda()).cpu()
    assert np.array_equal(_bits(out), O.embed_fwd(tok.numpy(), _bits(wte), _bits(wpe),
                                                  CODE[dtype]))
    gw, gp = K.embed_bwd(tok.cuda(), dout.cuda(), V, S + 3)
    rw, rp = O.embed_bwd(tok.numpy(), _bits(dout), V, CODE[dtype])
    assert np.array_equal(_bits(gw.cpu()), rw)
    assert np.array_equal(_bits(gp[:S].cpu()), rp) and not bool(gp[S:].any())
    hw, hp = torch.empty(V, H, dtype=dtype), torch.empty(S, H, dtype=dtype)
    K.embed_bwd_host(tok, dout, hw, hp)
    assert torch.equal(hw.view(torch.int16), gw.cpu().view(torch.int16))


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_device_embedding_backward_accumulates_into_weights(native_lib, oracle_lib, dtype):
    """Tied head: wte already holds the head's dW; the lookup gradient is
    added in place (K4 semantics), wpe is overwritten, spare wpe rows zeroed."""
    O = oracle_lib
    B, S, V, H = 4, 32, 300, 64
    tok, _, _, dout = _case(dtype, B, S, V, H, seed=3, repeat_tokens=True)
    head = (torch.randn(V, H) * 0.5).to(dtype)
    wte, wpe = head.clone().cuda(), torch.full((S + 2, H), 3.0, dtype=dtype).cuda()
    K.embed_bwd_into(tok.cuda(), dout.cuda(), wte, wpe, accumulate=True)
    ref = O.embed_bwd_accumulate(tok.numpy(), _bits(dout), _bits(head), CODE[dtype])
    assert np.array_equal(_bits(wte.cpu()), ref)
    _, rp = O.embed_bwd(tok.numpy(), _bits(dout), V, CODE[dtype])
    assert np.array_equal(_bits(wpe[:S].cpu()), rp) and not bool(wpe[S:].any())


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")
def test_device_out_of_range_ids_read_nothing_and_poison_their_rows(native_lib):
    """Device-resident token ids and targets are not validated on the host:
    an id outside [0, V) must not be dereferenced; the embedding row and the
    cross-entropy row (loss and gradient) become NaN, so the overflow check
    skips the step; valid rows are unchanged and the backward ignores the id."""
    tok, wte, wpe, dout = _case(torch.float16, 2, 4, 10, 8, seed=2)
    good = K.embed_fwd(tok.cuda(), wte.cuda(), wpe.cuda()).cpu()
    bad = tok.clone()
    bad[0, 1], bad[1, 3] = 10, -5
    out = K.embed_fwd(bad.cuda(), wte.cuda(), wpe.cuda()).cpu()
    assert torch.isnan(out[0, 1]).all() and torch.isnan(out[1, 3]).all()
    mask = torch.ones(2, 4, dtype=torch.bool)
    mask[0, 1] = mask[1, 3] = False
    assert torch.equal(out[mask].view(torch.int16), good[mask].view(torch.int16))
    gw = torch.empty_like(wte).cuda()
    gp = torch.empty_like(wpe).cuda()
    K.embed_bwd_into(bad.cuda(), dout.cuda(), gw, gp)  # the bad ids contribute nothing
    torch.cuda.synchronize()
    logits = torch.randn(3, 40, device="cuda").half()
    tgt = torch.tensor([5, 40, -1], device="cuda")
    loss, lse = K.xent_fwd(logits, tgt)
    assert torch.isfinite(loss[0]) and torch.isnan(loss[1:]).all()
    g = K.xent_bwd_(logits.clone(), tgt, lse, torch.ones((), device="cuda"), 1.0)
    assert torch.isfinite(g[0]).all() and torch.isnan(g[1:]).all()
