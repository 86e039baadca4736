"""bench.py contract on a small model: the N=1 line and the N>1 path
(torchrun, 2 ranks sharing cuda:0 over gloo — NCCL refuses two ranks on one
device; the NCCL launch differs only in the backend name)."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--layers", "2", "--hidden", "256", "--heads", "4", "--seq", "128", "--vocab", "512",
         "--batch", "2", "--cap", str(1 << 18), "--steps", "3", "--warmup", "3",
         "--no-cpu-baseline", "--no-offload-probe", "--no-c5"]


def _line(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_line():
    res = subprocess.run([sys.executable, "bench.py", *SMALL], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    d = _line(res.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["achieved"] > 0


def test_bench_offload_probe_fields():
    """The side measurement with every optimizer triplet in host DRAM: chunk
    moves against the idle pinned peak and against the ceiling measured
    beside the host Adam in the same run."""
    args = [a for a in SMALL if a != "--no-offload-probe"]
    res = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    probe = _line(res.stdout)["offload_probe"]
    assert probe["ms_per_step"] > 0 and probe["host_adam_gelem_per_s"] > 0
    for key in ("d2h", "h2d"):
        m = probe["chunk_moves"][key]
        assert m["copies"] > 0 and m["achieved_gbs"] > 0 and 0 < m["frac"]
        assert m["ceiling_beside_host_adam_gbs"] > 0 and m["frac_of_that_ceiling"] > 0


def test_bench_two_ranks_gloo_same_device():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 200),
           "bench.py", "--gpus", "2", "--dist-backend", "gloo", "--same-device", *SMALL]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, (res.stdout + res.stderr)[-3000:]
    d = _line(res.stdout)
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 4
    cps = d["collectives_per_step"]
    assert cps["ledger_bytes_per_rank"] == cps["closed_form_bytes_per_rank"] > 0
    assert "collectives" in d
    ins = d["collectives"]["in_step"]
    assert ins["all_gather"]["per_step"] > 0 and ins["reduce_scatter_avg"]["per_step"] > 0
    assert ins["all_gather"]["mean_ms"] > 0


def test_library_loaded_before_torch_keeps_torch_cublas_working():
    """build() loads the library before any torch CUDA work (then smoke() runs
    in the same process): torch's cuBLAS must still be the one in use."""
    code = ("import __graft_entry__ as g; from paper_2108_05818_b200 import _native; "
            "_native.load(); import torch; a = torch.randn(256, 256, device='cuda').half(); "
            "print(float((a @ a).float().abs().sum()) > 0)")
    res = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0 and res.stdout.strip().endswith("True"), res.stderr[-2000:]
