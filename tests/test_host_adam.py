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


def test_host_adam_respects_skip(native_lib):
    g = torch.ones(16, dtype=torch.float16)
    p = torch.zeros(16)
    m, v = torch.zeros(16), torch.zeros(16)
    s = N.CsStepState()
    s.skip = 1
    K.adam_chunks_host([(g, p, m, v, 16)], K.AdamHyper(), s)
    assert (g == 1).all() and (p == 0).all()
