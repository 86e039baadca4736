"""CPU port of the chunk-managed GPT training step — TEST INFRASTRUCTURE /
BASELINE ONLY (bench.py's ``cpu_baseline`` and ``--impl reference`` legs).

The reference (`/root/reference`) is an accounting simulator: it has no CPU
*numerics* to time.  Its CPU path for this step is therefore
restated here as the natural host implementation of the same iteration:

* the reference's decision engine (layout, FSM, eviction, placement, DP
  protocol) runs for the iteration — this build's accounting core, which is
  decision-identical to the reference (tests/test_decisions_golden.py);
* the reference-shaped GPT (same eight tensors per layer, `model.py:163-191`)
  forward + backward in fp32 with torch on the host cores;
* the chunk Adam by the C oracle (oracle/cs_oracle.c, OpenMP) on every
  parameter: fp16 gradients (the chunk reuse) -> fp32 master/m/v -> fp16.

``kind`` is "port" (the reference has nothing to compile).
"""

import time
from typing import Dict, Optional

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from . import numerics as O


class _Block(nn.Module):
    def __init__(self, H: int, heads: int):
        super().__init__()
        self.heads = heads
        lin = lambda o, i: nn.Linear(i, o, bias=False)
        self.q, self.k, self.v, self.o = lin(H, H), lin(H, H), lin(H, H), lin(H, H)
        self.i1, self.i2 = lin(2 * H, H), lin(2 * H, H)
        self.o1, self.o2 = lin(H, 2 * H), lin(H, 2 * H)

    def forward(self, h):
        B, S, H = h.shape
        a = F.layer_norm(h, (H,))
        sp = lambda t: t.view(B, S, self.heads, H // self.heads).transpose(1, 2)
        att = F.scaled_dot_product_attention(sp(self.q(a)), sp(self.k(a)), sp(self.v(a)),
                                             is_causal=True)
        h = h + self.o(att.transpose(1, 2).reshape(B, S, H))
        b = F.layer_norm(h, (H,))
        g1 = F.gelu(self.i1(b), approximate="tanh")
        g2 = F.gelu(self.i2(b), approximate="tanh")
        return h + self.o1(g1) + self.o2(g2)


class CpuGPT(nn.Module):
    def __init__(self, layers: int, H: int, heads: int, vocab: int, seq: int):
        super().__init__()
        self.wte = nn.Parameter(torch.randn(vocab, H) * 0.02)
        self.wpe = nn.Parameter(torch.randn(seq, H) * 0.02)
        self.blocks = nn.ModuleList([_Block(H, heads) for _ in range(layers)])
        for p in self.blocks.parameters():
            nn.init.normal_(p, std=0.02)

    def forward(self, tok, tgt):
        B, S = tok.shape
        h = F.embedding(tok, self.wte) + self.wpe[:S]
        for blk in self.blocks:
            h = blk(h)
        logits = F.linear(F.layer_norm(h, (h.shape[-1],)), self.wte)
        return F.cross_entropy(logits.view(B * S, -1), tgt.reshape(B * S))


class CpuChunkStep:
    """One process, host cores only.  ``step()`` returns seconds."""

    def __init__(self, schema, sample_batch: int = 1, threads: Optional[int] = None,
                 seed: int = 0, lr: float = 1e-4):
        import os
        self.threads = threads or os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        torch.manual_seed(seed)
        self.schema = schema
        self.sample_batch = sample_batch
        self.model = CpuGPT(schema.layers, schema.hidden_dim, schema.heads, schema.vocab,
                            schema.seq_len)
        self.state: Dict[int, tuple] = {}
        for i, p in enumerate(self.model.parameters()):
            n = p.numel()
            self.state[i] = (np.zeros(n, np.float32), np.zeros(n, np.float32))
        self.os = O.step_state(1.0)
        self.lr = lr
        g = torch.Generator().manual_seed(seed)
        self.tokens = torch.randint(0, schema.vocab, (sample_batch, schema.seq_len + 1),
                                    generator=g)
        self._engine = None
        try:  # the decision engine of the same iteration (accounting-only)
            import paper_2108_05818_b200 as cs
            sim = cs.Simulator(schema, cs.HardwareSpec(gpu_count=1), cs.PolicySpec(
                capacity_elems=64 << 20))
            self._sim = sim
        except Exception:
            self._sim = None

    def step(self) -> float:
        t0 = time.perf_counter()
        if self._sim is not None:
            it = len(getattr(self, "_reports", []))
            plan = self._sim._plan_builder() if it == 0 else None
            rep = self._sim.engine.run_iteration(it, warmup=(it == 0), plan_builder=plan)
            self._reports = getattr(self, "_reports", []) + [rep]
        self.model.zero_grad(set_to_none=True)
        tok = self.tokens
        loss = self.model(tok[:, :-1], tok[:, 1:])
        loss.backward()
        self.os.sumsq = 1.0
        O.adam_prepare(self.os, self.lr, 0.9, 0.999)
        for i, p in enumerate(self.model.parameters()):
            g16 = p.grad.detach().reshape(-1).half().numpy().view(np.uint16).copy()
            p32 = p.data.reshape(-1).numpy()  # fp32 master is the CPU model's parameter
            m, v = self.state[i]
            O.adam(g16, p32, m, v, p32.size, O.FP16, self.lr, 0.9, 0.999, 1e-8, 0.0, False,
                   self.os, self.threads)
        return time.perf_counter() - t0

    @property
    def tokens_per_step(self) -> int:
        return self.sample_batch * self.schema.seq_len
