"""Host fused Adam (CPU-placed optimizer triplets) vs the C oracle: bit-exact.

This is product code that runs on the host by design (PAPER §5 device-aware
placement), so it is testable without a GPU.
"""

import numpy as np
import pytest
import torch

from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200 import _native as N


def _state(O, lr, b1, b2, loss_scale, sumsq, steps=1):
    s = O.step_state(loss_scale)
    for _ in range(steps):
        s.sumsq = sumsq
        O.adam_prepare(s, lr, b1, b2)
    c = N.CsStepState()
    for f, _ in N.CsStepState._fields_:
        setattr(c, f, getattr(s, f))
    return s, c


@pytest.mark.parametrize("dtype,wd,adamw", [(torch.float16, 0.0, False),
                                            (torch.float16, 0.1, False),
                                            (torch.bfloat16, 0.01, True)])
def test_host_adam_bit_exact_vs_oracle(native_lib, oracle_lib, dtype, wd, adamw):
    O = oracle_lib
    rng = np.random.default_rng(3)
    sizes = [1, 7, 8, 4099, 65536 + 13]
    hyper = K.AdamHyper(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=wd, adamw=adamw)
    s_or, s_c = _state(O, 1e-3, 0.9, 0.95, 8.0, 3.0, steps=3)
    items, refs = [], []
    for n in sizes:
        g = torch.from_numpy(rng.standard_normal(n).astype(np.float32) * 8e-3).to(dtype)
        p = torch.from_numpy(rng.standard_normal(n).astype(np.float32) * 0.02)
        m = torch.from_numpy(rng.standard_normal(n).astype(np.float32) * 1e-3)
        v = torch.from_numpy(np.abs(rng.standard_normal(n)).astype(np.float32) * 1e-6)
        refs.append((g.view(torch.int16).numpy().view(np.uint16).copy(), p.numpy().copy(),
                     m.numpy().copy(), v.numpy().copy()))
        items.append((g, p, m, v, n))
    K.adam_chunks_host(items, hyper, s_c, n_threads=4)
    code = O.FP16 if dtype == torch.float16 else O.BF16
    for (g, p, m, v, n), (rg, rp, rm, rv) in zip(items, refs):
        O.adam(rg, rp, rm, rv, n, code, 1e-3, 0.9, 0.95, 1e-8, wd, adamw, s_or)
        np.testing.assert_array_equal(p.numpy().view(np.uint32), rp.view(np.uint32))
        np.testing.assert_array_equal(m.numpy().view(np.uint32), rm.view(np.uint32))
        np.testing.assert_array_equal(v.numpy().view(np.uint32), rv.view(np.uint32))
        np.testing.assert_array_equal(g.view(torch.int16).numpy().view(np.uint16), rg)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_host_adam_skip_restores_params(native_lib, oracle_lib, dtype):
    """Skipped step: p32 / m / v untouched, p16 (holding the overflowed
    gradients) gets round(p32) back — same bits as the oracle, ragged tail."""
    O = oracle_lib
    n = 8 * 1000 + 5
    gen = torch.Generator().manual_seed(6)
    g = torch.full((n,), float("inf")).to(dtype)
    p = torch.randn(n, generator=gen)
    m, v = torch.randn(n, generator=gen), torch.rand(n, generator=gen)
    ref = (g.view(torch.int16).numpy().view(np.uint16).copy(), p.numpy().copy(),
           m.numpy().copy(), v.numpy().copy())
    s = N.CsStepState()
    s.skip = 1
    K.adam_chunks_host([(g, p, m, v, n)], K.AdamHyper(), s, n_threads=3)
    so = O.step_state(1.0)
    so.skip = 1
    O.adam(*ref, n, O.FP16 if dtype == torch.float16 else O.BF16, 1e-4, 0.9, 0.999, 1e-8, 0.0,
           False, so)
    assert np.array_equal(p.numpy(), ref[1]) and np.array_equal(m.numpy(), ref[2])
    assert np.array_equal(g.view(torch.int16).numpy().view(np.uint16), ref[0])
    assert torch.equal(g, p.to(dtype))


def test_host_adam_nan_params_narrow_to_canonical_nan(native_lib):
    """A NaN master narrows to the canonical NaN 0x7fff in both 16-bit
    formats (what the device's cvt.rn.{f16,bf16}.f32 produce); bf16 NaNs
    with high mantissa bits must not wrap to -0 or turn into infinity."""
    n = 24
    st = N.CsStepState()
    st.grad_scale, st.step_size, st.sqrt_bc2, st.skip = 1.0, 1e-3, 0.5, 0
    bits = np.array([0x7fc00000, 0xffc00000, 0x7fffffff, 0xffffffff, 0x7f800001, 0x7fbfffff,
                     0xff800001, 0x7ff0f0f0] * 3, dtype=np.uint32)
    for dtype in (torch.float16, torch.bfloat16):
        g = torch.zeros(n, dtype=dtype)
        p = torch.from_numpy(bits.view(np.float32).copy())
        m, v = torch.zeros(n), torch.zeros(n)
        K.adam_chunks_host([(g, p, m, v, n)], K.AdamHyper(), st, n_threads=2)
        out = g.view(torch.int16).numpy().view(np.uint16)
        assert (out == 0x7fff).all(), (dtype, [hex(x) for x in out])


def test_host_threads_share_of_the_affinity_mask(native_lib):
    """cs_host_threads(0) = cores in the affinity mask / LOCAL_WORLD_SIZE
    (never omp_get_max_threads(): torchrun sets OMP_NUM_THREADS=1), unless
    CS_HOST_BOUND=1 says the mask is already this rank's own share."""
    import os
    import subprocess
    import sys
    cores = len(os.sched_getaffinity(0))
    code = ("import sys; sys.path.insert(0, %r); from paper_2108_05818_b200 import _native as N; "
            "print(N.load().cs_host_threads(0), N.load().cs_host_threads(5))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    for env, want in (({"LOCAL_WORLD_SIZE": "1"}, cores), ({"LOCAL_WORLD_SIZE": "2"}, cores // 2),
                      ({"LOCAL_WORLD_SIZE": str(4 * cores)}, 1),
                      ({"LOCAL_WORLD_SIZE": "2", "CS_HOST_BOUND": "1"}, cores),
                      ({"LOCAL_WORLD_SIZE": "2", "OMP_NUM_THREADS": "1"}, cores // 2)):
        e = dict(os.environ)
        e.pop("CS_HOST_BOUND", None)
        e.update(env)
        out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True,
                             text=True, check=True).stdout.split()
        assert [int(x) for x in out] == [max(want, 1), 5], (env, out)


def test_out_of_place_host_adam_equals_in_place(native_lib):
    """cs_adam_chunks_host_oop: same bits as the in-place update, inputs intact."""
    rng = np.random.default_rng(9)
    hyper = K.AdamHyper(lr=1e-3, betas=(0.9, 0.95), weight_decay=0.01, adamw=True)
    st = N.CsStepState()
    st.grad_scale, st.step_size, st.sqrt_bc2, st.skip = 0.125, 1e-3, 0.3, 0
    for dtype in (torch.float16, torch.bfloat16):
        for n in (1, 9, 65536 + 5):
            g = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(dtype)
            p, m = (torch.from_numpy(rng.standard_normal(n).astype(np.float32) * 0.02)
                    for _ in range(2))
            v = torch.from_numpy(np.abs(rng.standard_normal(n)).astype(np.float32) * 1e-6)
            ins = [t.clone() for t in (g, p, m, v)]
            outs = [torch.empty_like(t) for t in ins]
            K.adam_chunks_host_oop([(*ins, n)], [(*outs, n)], hyper, st, n_threads=3)
            for a, b in zip(ins, (g, p, m, v)):      # inputs untouched
                assert torch.equal(a, b)
            K.adam_chunks_host([(g, p, m, v, n)], hyper, st, n_threads=2)
            for a, b in zip(outs, (g, p, m, v)):     # outputs == in-place result
                assert torch.equal(a.view(torch.int16 if a.dtype != torch.float32
                                          else torch.int32),
                                   b.view(torch.int16 if b.dtype != torch.float32
                                          else torch.int32))
    st.skip = 1
    with pytest.raises(N.NativeError):
        K.adam_chunks_host_oop([(*ins, n)], [(*outs, n)], hyper, st)


def test_speculated_step_scalars_match_prepare(oracle_lib):
    """kernels.speculate_step_scalars reproduces cs_adam_prepare (the oracle's
    restatement, pinned to the device kernel by tests/test_kernels_gpu.py)
    bit for bit for finite, unclipped steps — through loss-scale growth."""
    O = oracle_lib
    for lr, b1, b2 in ((1e-4, 0.9, 0.999), (3e-3, 0.8, 0.95)):
        hyper = K.AdamHyper(lr=lr, betas=(b1, b2))
        s = O.step_state(65536.0)
        for step in range(40):
            prev = N.CsStepState()
            for f, _ in N.CsStepState._fields_:
                setattr(prev, f, getattr(s, f))
            s.sumsq = 1.0 + step
            O.adam_prepare(s, lr, b1, b2, growth=2.0, backoff=0.5, interval=7, dynamic=True)
            real = N.CsStepState()
            for f, _ in N.CsStepState._fields_:
                setattr(real, f, getattr(s, f))
            spec = K.speculate_step_scalars(prev, hyper)
            assert K.same_update_scalars(spec, real), (lr, step)
            assert spec.step == real.step
        # an overflowing step is never matched (its update is a skip)
        prev = real
        s.sumsq = float("inf")
        O.adam_prepare(s, lr, b1, b2, dynamic=True)
        real = N.CsStepState()
        for f, _ in N.CsStepState._fields_:
            setattr(real, f, getattr(s, f))
        assert not K.same_update_scalars(K.speculate_step_scalars(prev, hyper), real)
