"""K2's canonical order, host side (no GPU): the host twin
``cs_grad_sumsq_host`` equals the C oracle's restatement of the order
(``or_grad_sumsq_item``) bit for bit -- fp16 and bf16, whole and ragged
tiles, empty items, inf / NaN -- and stays within double rounding of the
plain sum of squares."""

import numpy as np
import pytest
import torch

from oracle import numerics as O
from paper_2108_05818_b200 import kernels as K


def _grads(n, dtype, seed, scale=1e-2):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(n, generator=g) * scale).to(dtype)


@pytest.mark.parametrize("dtype,code", [(torch.float16, O.FP16), (torch.bfloat16, O.BF16)])
@pytest.mark.parametrize("n", [0, 1, 7, 8, 8191, 8192, 8193, 3 * 8192 + 4100, 1 << 20])
def test_host_twin_matches_oracle(dtype, code, n):
    g = _grads(n, dtype, seed=n)
    host = K.grad_sumsq_host([(g, n)], 4)
    bits = g.view(torch.int16).numpy().view(np.uint16).copy()
    want = O.grad_sumsq_item(bits, code)
    assert np.float64(host[0]).tobytes() == np.float64(want).tobytes(), (host[0], want)
    if n:
        plain = O.grad_sumsq(bits, code)
        assert abs(host[0] - plain) <= 1e-5 * plain


def test_host_twin_items_and_threads_independent():
    items = [(_grads(n, torch.float16, s), n) for s, n in enumerate([5000, 0, 70000, 8192])]
    a = K.grad_sumsq_host(items, 1)
    b = K.grad_sumsq_host(items, 7)
    c = [K.grad_sumsq_host([it], 3)[0] for it in items]
    assert a == b == c


def test_non_finite_propagates():
    g = _grads(20000, torch.float16, 3)
    g[12345] = float("inf")
    assert K.grad_sumsq_host([(g, g.numel())])[0] == float("inf")
    g[7] = float("nan")
    assert np.isnan(K.grad_sumsq_host([(g, g.numel())])[0])


def test_total_folds_slots_in_order():
    vals = [1e10, 1.0, -1e10, 3.5]
    assert O.sumsq_total(vals) == np.float32(((1e10 + 1.0) - 1e10) + 3.5)
