"""Pin the C oracle before trusting it (CPU only).

* Adam: against torch.optim.Adam / AdamW (PyTorch 2.11 CPU fp32) golden
  trajectories, tests/golden/adam_torch.npz (gen_adam_golden.py).
  Tolerance: m and v bit-exact; p within rtol 1e-6 / atol 1e-9 (the only
  residual is torch's CPU sqrt, which is not correctly rounded);
  fp16 params within 1 ulp.
* fp16 / bf16 conversions: bit-exact vs numpy / torch over every fp16 and
  1.6M fp32 values.
"""

import os

import numpy as np
import pytest
import torch

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "adam_torch.npz")


@pytest.mark.parametrize("case", ["adam", "adam_l2", "adamw"])
def test_oracle_adam_matches_torch(oracle_lib, case):
    O = oracle_lib
    d = np.load(GOLDEN)
    lr, b1, b2, eps, wd, adamw = d[case + "/hyper"]
    p32 = d[case + "/p0"].copy()
    m = np.zeros_like(p32)
    v = np.zeros_like(p32)
    s = O.step_state(1.0)
    for t in range(d[case + "/g16"].shape[0]):
        p16 = d[case + "/g16"][t].copy()
        s.sumsq = 1.0
        O.adam_prepare(s, lr, b1, b2)
        assert s.step == t + 1 and not s.skip
        O.adam(p16, p32, m, v, p32.size, O.FP16, lr, b1, b2, eps, wd, bool(adamw), s)
        np.testing.assert_array_equal(m, d[case + "/m"][t])
        np.testing.assert_array_equal(v, d[case + "/v"][t])
        np.testing.assert_allclose(p32, d[case + "/p"][t], rtol=1e-6, atol=1e-9)
        ref16 = d[case + "/p"][t].astype(np.float16).view(np.uint16).astype(np.int32)
        assert np.abs(p16.astype(np.int32) - ref16).max() <= 1


def test_oracle_half_conversions_exhaustive(oracle_lib):
    L = oracle_lib.lib()
    ref = np.arange(65536, dtype=np.uint16).view(np.float16).astype(np.float32)
    mine = np.array([L.or_half_to_float(h) for h in range(65536)], dtype=np.float32)
    finite = ~np.isnan(ref)
    np.testing.assert_array_equal(mine[finite].view(np.uint32), ref[finite].view(np.uint32))
    assert np.isnan(mine[~finite]).all()


def test_oracle_narrowing_rounds_to_nearest_even(oracle_lib):
    L = oracle_lib.lib()
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.standard_normal(20000).astype(np.float32) * s
                         for s in (1e-8, 1e-6, 1e-4, 1e-2, 1, 100, 1e4, 6e4)] +
                        [np.array([65504, 65519.996, 65520, 65536, 6.1035156e-05, 5.96e-08,
                                   2.98e-08, 2.99e-08, 0.0, -0.0], np.float32)])
    with np.errstate(over="ignore"):
        ref16 = xs.astype(np.float16).view(np.uint16)
    mine16 = np.array([L.or_float_to_half(float(x)) for x in xs], dtype=np.uint16)
    np.testing.assert_array_equal(mine16, ref16)
    refb = torch.from_numpy(xs).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    mineb = np.array([L.or_float_to_bf16(float(x)) for x in xs], dtype=np.uint16)
    np.testing.assert_array_equal(mineb, refb)


def test_oracle_step_scalars_skip_and_scaler(oracle_lib):
    O = oracle_lib
    s = O.step_state(1024.0)
    s.sumsq = float("inf")
    O.adam_prepare(s, 1e-3, 0.9, 0.999, dynamic=True, backoff=0.5)
    assert s.skip == 1 and s.step == 0 and s.loss_scale == 512.0
    s.sumsq = 512.0 ** 2 * 4.0   # unscaled norm 2
    O.adam_prepare(s, 1e-3, 0.9, 0.999, max_norm=1.0, dynamic=True, interval=1, growth=2.0)
    assert s.skip == 0 and s.step == 1
    assert abs(s.grad_norm - 2.0) < 1e-6
    assert abs(s.grad_scale - (1.0 / 512.0) * (1.0 / (2.0 + 1e-6))) < 1e-9
    assert s.loss_scale == 1024.0  # grew after `interval` good steps
    assert abs(s.step_size - 1e-3 / (1 - 0.9)) < 1e-9
