"""Seeded random configurations through the REAL B200 step.

Beyond the 13 golden configurations: for each seed a random tiny GPT (layers,
hidden, sequence, batch), chunk capacity, dtype, eviction strategy, optimizer
state placement, activation checkpointing, Adam / AdamW hyper-parameters
(learning rate, weight decay) and a GPU budget just above the
smallest feasible one (found with the accounting-only engine, so the run
evicts).  Properties checked on every configuration:

* decisions: every iteration's transfer / collective ledger and memory
  samples equal an accounting-only ``Simulator`` run of the same
  configuration (the accounting core is pinned to the reference by
  tests/test_decisions_golden.py);
* the executor moved exactly the billed chunk bytes;
* odd seeds delay every chunk move on its copy stream (H2D targets NaN until
  the bytes land), so any consumer not ordered after a move's event breaks
  the bit-identity below;
* every K1 launch of the tight-budget run equals the C oracle byte for byte
  (random lr, betas, weight decay, Adam / AdamW);
* numerics: the tight-budget run — with a random embedding placement
  (plan / host / device operator), synchronous, asynchronous or speculative
  host Adam —
  is bit-identical to an all-resident run of the same model (deterministic
  attention backend).
"""

import random

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec  # noqa: E402
from paper_2108_05818_b200.memory import EvictionStrategy  # noqa: E402
from paper_2108_05818_b200.model import build_gpt_schema  # noqa: E402

ITERS = 3


def _config(seed):
    r = random.Random(seed)
    H = r.choice([128, 256])
    schema = dict(layers=r.choice([2, 3, 4]), hidden_dim=H, heads=4,
                  seq_len=r.choice([64, 128]), batch=r.choice([2, 4]), vocab=r.choice([512, 4096]),
                  context_bytes=2 << 20)
    cap = r.choice([2 * H * H, 4 * H * H, 8 * H * H])
    policy = dict(capacity_elems=cap, checkpointing=r.random() < 0.4,
                  os_placement=r.choice(["auto", "auto", "cpu", "gpu"]),
                  eviction=r.choice([EvictionStrategy.LATEST_NEXT_USE,
                                     EvictionStrategy.LIST_ORDER]))
    dtype = r.choice([torch.float16, torch.bfloat16])
    run = dict(embedding_placement=r.choice(["plan", "cpu", "gpu"]),
               async_host_adam=r.random() < 0.5)
    run["speculative_host_adam"] = run["async_host_adam"] and r.random() < 0.7
    wd = r.choice([0.0, 0.0, 0.01, 0.1])
    hyper = dict(lr=r.choice([1e-4, 1e-3]), betas=r.choice([(0.9, 0.999), (0.9, 0.95)]),
                 weight_decay=wd, adamw=wd > 0 and r.random() < 0.5)
    return schema, policy, dtype, r.uniform(1.05, 1.4), run, hyper


def _feasible(schema, policy, gpu_bytes):
    from paper_2108_05818_b200.scenario import Simulator
    sim = Simulator(build_gpt_schema(**schema), HardwareSpec(gpu_count=1, gpu_bytes=gpu_bytes),
                    PolicySpec(**policy))
    run = sim.run(ITERS)
    return all(r.feasible for r in run.reports), run


def _tight_budget(schema, policy, slack):
    lo, hi = 1 << 20, 1 << 34
    while hi - lo > (256 << 10):
        mid = (lo + hi) // 2
        if _feasible(schema, policy, mid)[0]:
            hi = mid
        else:
            lo = mid
    return int(hi * slack)


def _rows(r):
    return ([(t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason) for t in r.transfers],
            [(c.iteration, c.group_id, c.kind, c.bytes) for c in r.collectives],
            [(s.moment, s.device, s.used_bytes, s.chunk_bytes, s.non_model_bytes)
             for s in r.samples])


@pytest.mark.parametrize("seed", range(24))
def test_random_config_real_step(seed):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    from paper_2108_05818_b200 import kernels as K
    schema_kw, policy, dtype, slack, knobs, hyper = _config(seed)
    budget = _tight_budget(schema_kw, policy, slack)
    ok, ref = _feasible(schema_kw, policy, budget)
    assert ok
    schema = build_gpt_schema(**schema_kw)
    g = torch.Generator().manual_seed(seed)
    toks = [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
            for _ in range(ITERS)]
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for name, gpu_bytes in (("tight", budget), ("resident", 180 * 10 ** 9)):
            kw = knobs if name == "tight" else {}
            tr = ChunkTrainer(schema, PolicySpec(**policy),
                              HardwareSpec(gpu_count=1, gpu_bytes=gpu_bytes), dtype=dtype, seed=0,
                              untied_head=True, hyper=K.AdamHyper(**hyper), **kw)
            if name == "tight":  # every K1 launch of the tight run replayed by the C oracle
                from oracle import step_check
                rec = step_check.arm(tr)
                if seed % 2:  # chunk moves land late; H2D targets read NaN until then
                    tr.executor.copy_delay_cycles = 1_000_000
            losses = [tr.step_host(t) for t in toks]
            tr.finish_host_work()
            if name == "tight":
                step_check.disarm(tr)
                assert rec["mismatch"] == [], (seed, rec["mismatch"][:3])
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            out[name] = (losses, params, tr)
    losses, params, tr = out["tight"]
    assert all(np.isfinite(losses))
    for mine, theirs in zip(tr.reports, ref.reports):
        assert _rows(mine) == _rows(theirs), (seed, mine.iteration)
    rows = [t for r in tr.reports for t in r.transfers if t.chunk_id != "embedding"]
    st = tr.executor.stats
    assert st.h2d_bytes - st.prefetch_discarded_bytes == sum(
        t.bytes for t in rows if (t.src, t.dst) == ("cpu", "gpu"))
    assert st.d2h_bytes == sum(t.bytes for t in rows if (t.src, t.dst) == ("gpu", "cpu"))
    assert out["resident"][0] == losses
    for a, b in zip(out["resident"][1], params):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
