"""The C-ABI library builds for sm_100a, loads and exports the header's API.

No GPU needed: only symbol resolution, struct layout and argument errors.
"""

import ctypes
import os
import re
import subprocess


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chunkstar_b200.h")


def _declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cs_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = _declared_functions()
    for must in ("cs_adam_chunks", "cs_grad_sumsq", "cs_pack", "cs_cast_pack",
                 "cs_master_init", "cs_adam_prepare", "cs_adam_chunks_host"):
        assert must in names


def test_library_exports_every_declared_symbol(native_lib):
    from paper_2108_05818_b200 import _native
    for name in _declared_functions():
        assert hasattr(native_lib, name), name
        assert name in _native.SIGNATURES, "binding missing for %s" % name


def test_library_targets_sm100a():
    from paper_2108_05818_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header(tmp_path, native_lib):
    from paper_2108_05818_b200 import _native as N
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "chunkstar_b200.h"\n'
                   'int main(void){\n'
                   ' printf("%zu %zu %zu %zu %zu\\n", sizeof(CsAdamHyper), sizeof(CsStepState),'
                   ' sizeof(CsAdamItem), sizeof(CsGradItem), sizeof(CsPackItem));\n'
                   ' printf("%zu %zu %zu %zu\\n", offsetof(CsStepState, loss_scale),'
                   ' offsetof(CsStepState, grad_scale), offsetof(CsStepState, skip),'
                   ' offsetof(CsStepState, sumsq));\n return 0; }\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    sizes, offs = subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")[:2]
    assert [int(x) for x in sizes.split()] == [
        ctypes.sizeof(N.CsAdamHyper), ctypes.sizeof(N.CsStepState), ctypes.sizeof(N.CsAdamItem),
        ctypes.sizeof(N.CsGradItem), ctypes.sizeof(N.CsPackItem)]
    assert [int(x) for x in offs.split()] == [
        N.CsStepState.loss_scale.offset, N.CsStepState.grad_scale.offset,
        N.CsStepState.skip.offset, N.CsStepState.sumsq.offset]
    assert ctypes.sizeof(N.CsStepState) <= 64


def test_argument_errors_are_reported(native_lib):
    from paper_2108_05818_b200 import _native as N
    rc = native_lib.cs_pack(None, -1, N.CS_FP16, 0, None)
    assert rc == -1 and b"invalid" in native_lib.cs_last_error()
    rc = native_lib.cs_master_init(None, None, None, None, 7, 4, None)
    assert rc == -1
    assert native_lib.cs_version().startswith(b"chunkstar_b200")


def test_argument_errors_of_model_side_entry_points(native_lib):
    """Validation happens before any CUDA call (no GPU needed)."""
    from paper_2108_05818_b200 import _native as N
    lib = native_lib
    assert lib.cs_embed_fwd(None, 4, 2, None, None, 100, 12, None, N.CS_FP16, None) == -1  # H % 8
    assert b"hidden" in lib.cs_last_error()
    assert lib.cs_embed_bwd(None, None, 5, 2, None, 10, 16, None, None, 0, N.CS_FP16,
                            None) == -1                                          # n % S
    assert lib.cs_embed_fwd_host(None, 1, 1, None, None, 10, 16, None, N.CS_FP16, 1) == -1
    assert lib.cs_embed_bwd_host(None, 3, 2, None, 10, 16, None, None, N.CS_BF16, 1, None) == -1
    # collectives: arguments are checked before NCCL is even loaded
    assert lib.cs_allgather(None, None, 4, N.CS_FP16, None, None) == -1
    assert lib.cs_reduce_scatter_avg(None, None, 4, N.CS_BF16, None, None) == -1
    assert lib.cs_allreduce(None, 1, N.CS_FP32, 0, None, None) == -1
    assert lib.cs_comm_init(b"\0" * 128, 2, 2, None) == -1                        # rank >= n
    assert lib.cs_comm_unique_id(None) == -1
    assert lib.cs_comm_destroy(None) == 0
    assert lib.cs_layernorm_supported(2048) == 1 and lib.cs_layernorm_supported(100) == 0
    assert lib.cs_layernorm_fwd(None, None, None, None, 4, 100, 1e-5, N.CS_FP16, None) == -1
    assert lib.cs_xent_fwd(None, None, 4, 10, 7, None, None, None) != 0           # dtype
