"""ctypes view of oracle/cs_oracle.c (TEST INFRASTRUCTURE ONLY).

Restates the chunk-step numerics on the CPU; see the header of
cs_oracle.c for what is pinned to what.  numpy arrays in, numpy arrays
modified in place.
"""

import ctypes
import os
from typing import Optional

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_DIR, "_build", "libcs_oracle.so")
_lib: Optional[ctypes.CDLL] = None

FP16, BF16, FP32 = 0, 1, 2


class OrStepState(ctypes.Structure):
    _fields_ = [("beta1_pow", ctypes.c_double), ("beta2_pow", ctypes.c_double),
                ("step", ctypes.c_int64), ("loss_scale", ctypes.c_float),
                ("good_steps", ctypes.c_int32), ("grad_scale", ctypes.c_float),
                ("step_size", ctypes.c_float), ("sqrt_bc2", ctypes.c_float),
                ("skip", ctypes.c_int32), ("grad_norm", ctypes.c_float),
                ("sumsq", ctypes.c_float)]


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import sys
            sys.path.insert(0, os.path.dirname(_DIR))
            from paper_2108_05818_b200._build import build_oracle
            build_oracle()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.or_float_to_half.restype = ctypes.c_uint16
        L.or_float_to_half.argtypes = [ctypes.c_float]
        L.or_half_to_float.restype = ctypes.c_float
        L.or_half_to_float.argtypes = [ctypes.c_uint16]
        L.or_float_to_bf16.restype = ctypes.c_uint16
        L.or_float_to_bf16.argtypes = [ctypes.c_float]
        L.or_step_state_init.argtypes = [ctypes.POINTER(OrStepState), ctypes.c_float]
        L.or_adam_prepare.argtypes = [ctypes.POINTER(OrStepState)] + [ctypes.c_double] * 3 + [ctypes.c_float] * 3 + \
            [ctypes.c_int32, ctypes.c_int32]
        L.or_adam.argtypes = [P, P, P, P, ctypes.c_int64, ctypes.c_int] + [ctypes.c_double] * 5 + \
            [ctypes.c_int, ctypes.POINTER(OrStepState), ctypes.c_int]
        L.or_grad_sumsq.restype = ctypes.c_double
        L.or_grad_sumsq.argtypes = [P, ctypes.c_int64, ctypes.c_int]
        L.or_grad_sumsq_item.restype = ctypes.c_double
        L.or_grad_sumsq_item.argtypes = [P, ctypes.c_int64, ctypes.c_int]
        L.or_sumsq_total.restype = ctypes.c_float
        L.or_sumsq_total.argtypes = [P, ctypes.c_int]
        L.or_pack.argtypes = [P, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.or_cast_pack.argtypes = [P, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_int]
        L.or_master_init.argtypes = [P, P, P, P, ctypes.c_int, ctypes.c_int64]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> ctypes.c_void_p:
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def step_state(loss_scale: float = 1.0) -> OrStepState:
    s = OrStepState()
    lib().or_step_state_init(ctypes.byref(s), loss_scale)
    return s


def adam_prepare(s: OrStepState, lr, beta1, beta2, max_norm=0.0, growth=2.0, backoff=0.5,
                 interval=2000, dynamic=False) -> None:
    lib().or_adam_prepare(ctypes.byref(s), lr, beta1, beta2, max_norm, growth, backoff,
                          interval, int(dynamic))


def adam(p16: np.ndarray, p32: np.ndarray, m: np.ndarray, v: np.ndarray, n: int, dtype: int,
         lr, beta1, beta2, eps, wd, adamw, s: OrStepState, threads: int = 1) -> None:
    assert p16.dtype == np.uint16 and p32.dtype == m.dtype == v.dtype == np.float32
    lib().or_adam(_p(p16), _p(p32), _p(m), _p(v), n, dtype, lr, beta1, beta2, eps, wd,
                  int(adamw), ctypes.byref(s), threads)


def grad_sumsq(g16: np.ndarray, dtype: int) -> float:
    """Plain double sum of squares (reference value for tolerance checks)."""
    return lib().or_grad_sumsq(_p(g16), g16.size, dtype)


def grad_sumsq_item(g16: np.ndarray, dtype: int) -> float:
    """K2's canonical per-item value S (bit-exact target of K2 and its host twin)."""
    return lib().or_grad_sumsq_item(_p(g16), g16.size, dtype)


def sumsq_total(item_sums) -> float:
    a = np.ascontiguousarray(np.asarray(item_sums, dtype=np.float64))
    return lib().or_sumsq_total(_p(a), a.size)


def pack(chunk: np.ndarray, offset: int, src: np.ndarray, dtype: int, accumulate: bool) -> None:
    lib().or_pack(_p(chunk), offset, _p(src), src.size, dtype, int(accumulate))


def cast_pack(chunk: np.ndarray, offset: int, src32: np.ndarray, dtype: int) -> None:
    lib().or_cast_pack(_p(chunk), offset, _p(src32), src32.size, dtype)


def master_init(p32, m, v, src: np.ndarray, src_dtype: int) -> None:
    lib().or_master_init(_p(p32), _p(m), _p(v), _p(src), src_dtype, src.size)


def to_half_bits(x: np.ndarray) -> np.ndarray:
    return x.astype(np.float16).view(np.uint16)


def from_half_bits(h: np.ndarray) -> np.ndarray:
    return h.view(np.float16).astype(np.float32)


# -- host embedding operator (CPU-placed embedding; cs_embed_*_host) --------------
# Restates the semantics `include/chunkstar_b200.h` declares for the lookup the
# reference places on the CPU (`profiler.py:70-74`, `engine.py:202-213`) in
# plain numpy: fp32 arithmetic, one rounding per output, sums in ascending
# token order.  Forward is pinned to torch's `F.embedding(tok, wte) + wpe[:S]`
# (tests/test_host_embed.py); bits in / bits out (uint16).

def _widen(bits: np.ndarray, dtype: int) -> np.ndarray:
    if dtype == FP16:
        return bits.view(np.float16).astype(np.float32)
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _narrow(x: np.ndarray, dtype: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == FP16:
        return x.astype(np.float16).view(np.uint16)
    u = x.view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def embed_fwd(tokens: np.ndarray, wte: np.ndarray, wpe: np.ndarray, dtype: int) -> np.ndarray:
    """tokens [B, S] int64; wte [V, H], wpe [>=S, H] uint16 bits -> [B, S, H] bits."""
    B, S = tokens.shape
    return _narrow(_widen(wte[tokens], dtype) + _widen(wpe[:S], dtype)[None], dtype)


def embed_bwd(tokens: np.ndarray, dout: np.ndarray, V: int, dtype: int):
    """dout [B, S, H] bits -> (gwte [V, H], gwpe [S, H]) bits; sequential fp32
    sums in ascending flat token order (np.add.at is unbuffered, in order)."""
    B, S = tokens.shape
    H = dout.shape[-1]
    d = _widen(dout.reshape(B * S, H), dtype)
    gw = np.zeros((V, H), dtype=np.float32)
    np.add.at(gw, tokens.reshape(-1), d)
    gp = np.zeros((S, H), dtype=np.float32)
    np.add.at(gp, np.tile(np.arange(S), B), d)
    return _narrow(gw, dtype), _narrow(gp, dtype)


def embed_bwd_accumulate(tokens: np.ndarray, dout: np.ndarray, gwte_old: np.ndarray, dtype: int):
    """cs_embed_bwd(accumulate=1) for wte: round(old + round(row sum)) (K4's
    slot += src with the rounded lookup gradient as src)."""
    gw, _ = embed_bwd(tokens, dout, gwte_old.shape[0], dtype)
    return _narrow(_widen(gwte_old, dtype) + _widen(gw, dtype), dtype)
