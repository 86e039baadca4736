"""ctypes binding of libchunkstar_b200.so (declared in include/chunkstar_b200.h).

There is deliberately no fallback: if the library is missing or a call
fails, this raises.  Structures mirror the header field for field.
"""

import ctypes
import os
from typing import Optional

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchunkstar_b200.so")

CS_FP16, CS_BF16, CS_FP32 = 0, 1, 2
CS_EINVAL, CS_EALIGN, CS_ETOOMANY, CS_EUNAVAIL, CS_EINPROGRESS = -1, -2, -3, -4, -5


class CsAdamHyper(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double),
                ("beta2", ctypes.c_double), ("eps", ctypes.c_double),
                ("weight_decay", ctypes.c_double), ("adamw", ctypes.c_int32)]


class CsStepState(ctypes.Structure):
    _fields_ = [("beta1_pow", ctypes.c_double), ("beta2_pow", ctypes.c_double),
                ("step", ctypes.c_int64), ("loss_scale", ctypes.c_float),
                ("good_steps", ctypes.c_int32), ("grad_scale", ctypes.c_float),
                ("step_size", ctypes.c_float), ("sqrt_bc2", ctypes.c_float),
                ("skip", ctypes.c_int32), ("grad_norm", ctypes.c_float),
                ("sumsq", ctypes.c_float)]


class CsAdamItem(ctypes.Structure):
    _fields_ = [("p16", ctypes.c_void_p), ("p32", ctypes.c_void_p),
                ("m", ctypes.c_void_p), ("v", ctypes.c_void_p), ("n", ctypes.c_int64)]


class CsGradItem(ctypes.Structure):
    _fields_ = [("g16", ctypes.c_void_p), ("n", ctypes.c_int64)]


class CsPackItem(ctypes.Structure):
    _fields_ = [("chunk", ctypes.c_void_p), ("offset", ctypes.c_int64),
                ("src", ctypes.c_void_p), ("n", ctypes.c_int64)]


#: every symbol the header declares, with (restype, argtypes)
SIGNATURES = {
    "cs_version": (ctypes.c_char_p, []),
    "cs_last_error": (ctypes.c_char_p, []),
    "cs_launch_count": (ctypes.c_int64, []),
    "cs_host_threads": (ctypes.c_int, [ctypes.c_int]),
    "cs_num_sms": (ctypes.c_int, []),
    "cs_adam_chunks": (ctypes.c_int, [ctypes.POINTER(CsAdamItem), ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(CsAdamHyper), ctypes.c_void_p,
                                      ctypes.c_void_p]),
    "cs_sumsq_scratch": (ctypes.c_int64, [ctypes.POINTER(CsGradItem), ctypes.c_int]),
    "cs_adam_variant": (ctypes.c_int, [ctypes.c_int]),
    "cs_grad_sumsq": (ctypes.c_int, [ctypes.POINTER(CsGradItem), ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int), ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_sumsq_finalize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "cs_step_state_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p]),
    "cs_adam_prepare": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(CsAdamHyper),
                                       ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]),
    "cs_pack": (ctypes.c_int, [ctypes.POINTER(CsPackItem), ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_void_p]),
    "cs_cast_pack": (ctypes.c_int, [ctypes.POINTER(CsPackItem), ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p]),
    "cs_master_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_void_p]),
    "cs_adam_chunks_host": (ctypes.c_int, [ctypes.POINTER(CsAdamItem), ctypes.c_int,
                                           ctypes.c_int, ctypes.POINTER(CsAdamHyper),
                                           ctypes.POINTER(CsStepState), ctypes.c_int]),
    "cs_grad_sumsq_host": (ctypes.c_int, [ctypes.POINTER(CsGradItem), ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_double), ctypes.c_int]),
    "cs_embed_fwd_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_int]),
    "cs_embed_bwd_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "cs_embed_fwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                    ctypes.c_void_p]),
    "cs_embed_bwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "cs_layernorm_supported": (ctypes.c_int, [ctypes.c_int]),
    "cs_layernorm_fwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                        ctypes.c_float, ctypes.c_int, ctypes.c_void_p]),
    "cs_layernorm_bwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p]),
    "cs_gemm_gelu": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_int64, ctypes.c_void_p]),
    "cs_gemm_res": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_void_p]),
    "cs_xent_fwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]),
    "cs_xent_bwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_float, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]),
    "cs_comm_version": (ctypes.c_int, []),
    "cs_comm_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "cs_comm_init": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p)]),
    "cs_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "cs_allgather": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_reduce_scatter_avg": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_allreduce": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p]),
    "cs_comm_check": (ctypes.c_int, [ctypes.c_void_p]),
    "cs_adam_chunks_host_oop": (ctypes.c_int, [ctypes.POINTER(CsAdamItem),
                                               ctypes.POINTER(CsAdamItem), ctypes.c_int,
                                               ctypes.c_int, ctypes.POINTER(CsAdamHyper),
                                               ctypes.POINTER(CsStepState), ctypes.c_int]),
    "cs_comm_abort": (ctypes.c_int, [ctypes.c_void_p]),
}

_lib: Optional[ctypes.CDLL] = None


class NativeError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load the library (once).  Raises if it is absent — no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    # torch first: it brings its own libcudart / libcublas / libcublasLt
    # (same SONAMEs as the toolkit's).  Whichever copy is loaded first serves
    # the whole process; if this library pulled the toolkit's libcublasLt in
    # before torch, torch's libcublas would run against a libcublasLt of
    # another version (CUBLAS_STATUS_INVALID_VALUE in its first GEMM).
    import torch  # noqa: F401
    if not os.path.exists(LIB_PATH):
        raise NativeError("libchunkstar_b200.so not built (%s); run "
                          "`python -m paper_2108_05818_b200._build` — the chunk step "
                          "has no CPU fallback" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().cs_last_error().decode(errors="replace")
        raise NativeError("%s failed (rc=%d): %s" % (what, rc, msg))


def launch_count() -> int:
    return int(load().cs_launch_count())
