"""Physical out-of-memory inside a real step becomes the reference's
infeasible verdict (`/root/reference/pkg/src/chunkstar/engine.py:349-352`:
OOMError -> IterationReport(feasible=False, failure_reason="GPU_OOM")).

The accounting is given a roomy budget, so it never raises; the CUDA caching
allocator is capped just above what the model's weights and chunk payloads
use, so the real forward's activations fail to allocate
(torch.OutOfMemoryError).  The trainer must record an infeasible report for
that iteration, join its host work and refuse further steps.
"""

import gc

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec  # noqa: E402
from paper_2108_05818_b200.model import build_gpt_schema  # noqa: E402


def test_allocator_oom_in_a_step_is_an_infeasible_report():
    from paper_2108_05818_b200.trainer import ChunkTrainer, StepInfeasible
    gc.collect()
    torch.cuda.empty_cache()
    schema = build_gpt_schema(layers=2, hidden_dim=256, heads=4, seq_len=256, vocab=4096,
                              batch=64, context_bytes=1 << 20)
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=1 << 18),
                      HardwareSpec(gpu_count=1, gpu_bytes=8 << 30), dtype=torch.float16,
                      seed=0, embedding_placement="gpu")
    toks = torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1))
    total = torch.cuda.get_device_properties(0).total_memory
    # room for what exists now plus a little: the activations of B=64 x S=256
    # (hundreds of MB) cannot fit
    cap = torch.cuda.memory_reserved() + (64 << 20)
    torch.cuda.set_per_process_memory_fraction(cap / total)
    try:
        with pytest.raises(StepInfeasible) as info:
            tr.step_host(toks)
    finally:
        torch.cuda.set_per_process_memory_fraction(1.0)
    rep = info.value.report
    assert rep is tr.reports[-1] and rep.iteration == 0
    assert rep.feasible is False and rep.failure_reason == "GPU_OOM"
    assert rep.failure_moment is not None and rep.failure_moment >= 0
    assert info.value.cause is not None
    rep.validate_conservation()
    with pytest.raises(RuntimeError, match="infeasible"):
        tr.step_host(toks)
    tr.close()
    del tr, info
    gc.collect()
    torch.cuda.empty_cache()


def test_accounting_oom_is_an_infeasible_report_too():
    """A budget too small for the layout: the accounting's own OOMError, the
    same StepInfeasible with the reference's verdict."""
    from paper_2108_05818_b200.trainer import ChunkTrainer, StepInfeasible
    schema = build_gpt_schema(layers=2, hidden_dim=128, heads=4, seq_len=64, vocab=512,
                              batch=2, context_bytes=1 << 20)
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=1 << 16),
                      HardwareSpec(gpu_count=1, gpu_bytes=1 << 20), dtype=torch.float16,
                      seed=0, embedding_placement="gpu")
    toks = torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1))
    with pytest.raises(StepInfeasible) as info:
        tr.step_host(toks)
    rep = info.value.report
    assert rep.feasible is False and rep.failure_reason == "GPU_OOM"
    assert info.value.cause is None
    tr.close()
