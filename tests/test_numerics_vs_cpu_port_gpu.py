"""End-to-end numerics of C1 ("ledger parity plus numeric parity
of N=5 steps"): the real fp16 chunk-managed B200 step against the CPU port of
the same iteration (oracle/cpu_step.py: fp32 torch-CPU forward/backward of
the same reference-shaped GPT + the C-oracle chunk Adam on fp16 gradients),
started from the trainer's own initial weights, same batches, same loss
scale.  The Adam arithmetic itself is bit-exact (tests/test_kernels_gpu.py,
every in-step launch in tests/test_step_gpu.py); what this test bounds is the
fp16 model's deviation from an fp32 model over five steps:

* loss at every step within 2e-3 relative;
* fp32 masters after 5 steps: the GPU-minus-CPU difference is below 1 % of
  the update the 5 steps made (mean absolute), and max |diff| <= 2 * 5 * lr
  (an Adam step moves a weight by at most ~lr; a sign flip of a tiny gradient
  costs at most that).  Measured on B200: losses equal to 4-5 digits, mean
  |diff| 3.0e-7 vs mean |update| 2.3e-4 (0.13 %).
"""

import gzip
import json
import os

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decisions.json.gz")
STEPS, LR, SCALE = 5, 1e-4, 2.0 ** 16


def test_c1_five_steps_match_fp32_cpu_port(oracle_lib):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from oracle import numerics as O
    from oracle.cpu_step import CpuGPT
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.chunks import ChunkKind
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer

    with gzip.open(GOLDEN, "rt") as f:
        c = json.load(f)["cases"]["tiny_cap256Ki"]
    schema = build_gpt_schema(**c["schema"])
    tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                      dtype=torch.float16, seed=0, hyper=K.AdamHyper(lr=LR),
                      init_loss_scale=SCALE, dynamic_loss_scale=False,
                      embedding_placement="gpu")
    ex = tr.executor
    # the trainer's fp32 initial weights -> the CPU port's model
    cpu = CpuGPT(schema.layers, schema.hidden_dim, schema.heads, schema.vocab, schema.seq_len)
    cpu_params = list(cpu.blocks.parameters())
    assert len(cpu_params) == len(ex.shapes)
    init = {}
    with torch.no_grad():
        for tid, p in enumerate(cpu_params):
            pos, off, n = ex.offsets[tid]
            w = ex.init32[pos][off:off + n].view(p.shape)
            p.copy_(w)
            init[tid] = w.clone()
        (wte, wte32, _, _), (wpe, wpe32, _, _) = ex.embedding
        cpu.wte.copy_(wte32.view(cpu.wte.shape).cpu())
        cpu.wpe.copy_(wpe32.view(cpu.wpe.shape).cpu())
    state = {i: (np.zeros(p.numel(), np.float32), np.zeros(p.numel(), np.float32))
             for i, p in enumerate(cpu.parameters())}
    os_state = O.step_state(SCALE)
    g = torch.Generator().manual_seed(77)
    batches = [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
               for _ in range(STEPS)]
    gpu_losses, cpu_losses = [], []
    with sdpa_kernel(SDPBackend.MATH):
        for b in batches:
            gpu_losses.append(tr.step_host(b))
            cpu.zero_grad(set_to_none=True)
            loss = cpu(b[:, :-1], b[:, 1:])
            (loss * SCALE).backward()
            cpu_losses.append(float(loss))
            os_state.sumsq = 1.0
            O.adam_prepare(os_state, LR, 0.9, 0.999)
            for i, p in enumerate(cpu.parameters()):
                g16 = p.grad.detach().reshape(-1).half().numpy().view(np.uint16).copy()
                m, v = state[i]
                O.adam(g16, p.data.reshape(-1).numpy(), m, v, p.numel(), O.FP16, LR, 0.9, 0.999,
                       1e-8, 0.0, False, os_state, 4)
    np.testing.assert_allclose(gpu_losses, cpu_losses, rtol=2e-3)
    upd, dif, mx = [], [], 0.0
    cs = tr.sim.chunk_set
    for tid, p in enumerate(cpu_params):
        pos, off, n = ex.offsets[tid]
        master = tr.local_chunk_payload(pos, ChunkKind.PARAM_FP32)[off:off + n].cpu()
        mine = master.view(p.shape)
        upd.append((mine - init[tid]).abs().mean().item())
        d = (mine - p.detach()).abs()
        dif.append(d.mean().item())
        mx = max(mx, d.max().item())
    print("losses gpu %s cpu %s; mean |update| %.3g, mean |gpu-cpu| %.3g, max %.3g"
          % (np.round(gpu_losses, 5), np.round(cpu_losses, 5), np.mean(upd), np.mean(dif), mx))
    assert np.mean(dif) < 0.01 * np.mean(upd), (np.mean(dif), np.mean(upd))
    assert mx <= 2 * STEPS * LR, mx
    assert cs.positions > 1
