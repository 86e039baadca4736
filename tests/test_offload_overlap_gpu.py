"""Chunk moves issued ahead of the accounting's decision, through the REAL step.

Two physical schedules that the ledger does not see (the rows stay at the
moments the reference bills them):

* pre-eviction: an optimizer-state chunk the last iteration evicted before
  ADAM is copied D2H right after this ADAM's K1 (the D2H direction is idle
  while ADAM's fetches fill H2D); the eviction in the next forward adopts the
  landed copy;
* early ADAM fetches: ADAM's fetches of GPU-placed positions are issued in the
  backward as soon as the last iteration's per-moment GPU usage leaves room.

On seeded tight-budget configurations (tests/test_fuzz_step_gpu.py's
generator) run for six iterations: every ledger row equals the
accounting-only engine's, the executor moves exactly the billed bytes
(pre-evictions count when adopted), every K1 launch equals the C oracle byte
for byte, and the result is bit-identical to an all-resident run — with
chunk moves landing late on odd seeds, and with a mispredicting schedule
(every optimizer-state chunk pre-evicted, most copies discarded when K1
rewrites the chunk).
"""

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec  # noqa: E402
from paper_2108_05818_b200.model import build_gpt_schema  # noqa: E402

from test_fuzz_step_gpu import _config, _rows, _tight_budget  # noqa: E402

ITERS = 6
SEEDS = [1, 4, 6, 9, 13, 16, 20]  # configurations whose ledger evicts chunks
EARLY = {1, 6, 16, 20}  # ... and whose backward leaves room for early ADAM fetches


def _run(seed, mispredict=False):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.chunks import ChunkKind
    from paper_2108_05818_b200.scenario import Simulator
    from paper_2108_05818_b200.trainer import ChunkTrainer
    from oracle import step_check
    schema_kw, policy, dtype, slack, knobs, hyper = _config(seed)
    budget = _tight_budget(schema_kw, policy, slack)
    schema = build_gpt_schema(**schema_kw)
    ref = Simulator(schema, HardwareSpec(gpu_count=1, gpu_bytes=budget),
                    PolicySpec(**policy)).run(ITERS)
    assert ref.feasible
    g = torch.Generator().manual_seed(seed)
    toks = [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
            for _ in range(ITERS)]
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for name, gpu_bytes in (("tight", budget), ("resident", 180 * 10 ** 9)):
            kw = knobs if name == "tight" else {}
            tr = ChunkTrainer(schema, PolicySpec(**policy),
                              HardwareSpec(gpu_count=1, gpu_bytes=gpu_bytes), dtype=dtype,
                              seed=0, untied_head=True, hyper=K.AdamHyper(**hyper), **kw)
            ex = tr.executor
            if name == "tight":
                rec = step_check.arm(tr)
                if seed % 2:
                    ex.copy_delay_cycles = 1_000_000
                if mispredict:  # every optimizer-state chunk is "predicted" evicted
                    base = ex.set_prefetch_schedule

                    def wrong(*a, **k):
                        base(*a, **k)
                        ex._preevict_ids |= {c.chunk_id for c in tr.sim.chunk_set.chunks.values()
                                             if c.list_kind is not ChunkKind.PARAM_FP16}
                    ex.set_prefetch_schedule = wrong
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
    os_evicted_before_adam = any(
        t.src == "gpu" and t.reason == "evict" and t.bytes > 0
        and tr.sim.chunk_set.chunks[t.chunk_id].list_kind is not ChunkKind.PARAM_FP16
        and t.moment < 2 * tr._events[-1].index + 1
        for t in tr.reports[-1].transfers if isinstance(t.chunk_id, int))
    print("seed %d: preevict hits %d, early ADAM fetches %d" % (
        seed, st.preevict_hits, st.adam_prefetch_early))
    return st, os_evicted_before_adam


@pytest.mark.parametrize("seed", SEEDS)
def test_preevict_and_early_adam_fetch(seed):
    st, os_evicted = _run(seed)
    if os_evicted:
        assert st.preevict_hits > 0, seed
        assert st.preevict_discarded == 0, seed  # the schedule is at its fixed point
    if seed in EARLY:
        assert st.adam_prefetch_early > 0 and st.adam_prefetch_oom == 0, seed


@pytest.mark.parametrize("seed", [1, 6, 16])
def test_mispredicted_preevictions_are_discarded(seed):
    st, _ = _run(seed, mispredict=True)
    assert st.preevict_discarded > 0, seed


def test_long_offload_run_holds_memory_constant():
    """15 iterations of a tight-budget configuration with pre-evictions and
    early ADAM fetches (seed 6's generator, chunk moves landing late): HBM
    allocated, pinned host bytes held by the executor and the slab pool stop
    growing once the schedule is at its fixed point, and nothing is ever
    discarded (the prediction holds every iteration)."""
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.trainer import ChunkTrainer
    schema_kw, policy, dtype, slack, knobs, hyper = _config(6)
    budget = _tight_budget(schema_kw, policy, slack)
    schema = build_gpt_schema(**schema_kw)
    tr = ChunkTrainer(schema, PolicySpec(**policy), HardwareSpec(gpu_count=1, gpu_bytes=budget),
                      dtype=dtype, seed=0, untied_head=True, hyper=K.AdamHyper(**hyper), **knobs)
    tr.executor.copy_delay_cycles = 200_000
    g = torch.Generator().manual_seed(6)
    marks = []
    for i in range(15):
        tr.step_host(torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1),
                                   generator=g))
        tr.finish_host_work()
        torch.cuda.synchronize()
        ex = tr.executor
        pinned = sum(t.numel() * t.element_size() for t in ex.payload["cpu"].values()) + \
            ex._free_host_bytes
        marks.append((torch.cuda.memory_allocated(), pinned, ex.slabs.slab_bytes,
                      len(ex._preevicted), len(ex._side_use)))
    st = tr.executor.stats
    assert st.preevict_hits > 0 and st.preevict_discarded == 0
    assert st.adam_prefetch_oom == 0
    assert st.adam_prefetch_early > 0
    print("early ADAM fetches", st.adam_prefetch_early, "pre-evictions", st.preevict_hits)
    steady = marks[5:]
    assert len({m[0] for m in steady}) == 1, marks      # HBM allocated
    assert len({m[1] for m in steady}) == 1, marks      # pinned payloads + free list
    assert len({m[2] for m in steady}) == 1, marks      # slab pool high-water mark
    assert max(m[4] for m in steady) <= max(m[4] for m in marks[:5]) + 8, marks
