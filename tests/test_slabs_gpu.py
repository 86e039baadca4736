"""HBM slab pool for chunk payloads (slabs.py): stream-ordered recycling."""

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def test_slab_recycled_after_enqueued_work_on_another_stream():
    from paper_2108_05818_b200.slabs import SlabPool
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    pool = SlabPool(torch.device("cuda", 0), [s1, s2])
    n = 1 << 24
    a = pool.take(n, torch.float16, s1)
    with torch.cuda.stream(s1):
        a.fill_(1.0)
        for _ in range(20):          # keep s1 busy writing the slab
            a.mul_(1.0)
    assert pool.give(a)
    b = pool.take(n, torch.float16, s2)
    assert b.data_ptr() == a.data_ptr() and pool.reuses == 1 and pool.allocs == 1
    with torch.cuda.stream(s2):
        b.fill_(2.0)
    torch.cuda.synchronize()
    assert bool((b == 2.0).all())
    # other sizes / dtypes never alias a free slab of another kind
    assert pool.give(b)
    c = pool.take(n, torch.float32, s1)
    assert c.data_ptr() != b.data_ptr() and pool.allocs == 2
    assert not pool.give(torch.empty(n, dtype=torch.float16, device="cuda"))  # not a slab
    assert pool.trim() == n * 2 and pool.free_tensors() == []


def test_eviction_run_recycles_chunk_slabs():
    """A tight-budget run (evictions, host Adam) reuses slabs instead of
    asking the caching allocator, and holds no more slabs than the
    sum of every chunk of the run."""
    import gzip
    import json
    import os
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    with gzip.open(os.path.join(os.path.dirname(__file__), "golden", "decisions.json.gz"),
                   "rt") as f:
        c = json.load(f)["cases"]["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                      dtype=torch.float16, seed=0)
    g = torch.Generator().manual_seed(1)
    for _ in range(4):
        tr.step_host(torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1),
                                   generator=g))
    pool = tr.executor.slabs
    assert pool.reuses > pool.allocs > 0
    cs = tr.sim.chunk_set
    every_chunk = sum(ch.bytes for ch in cs.chunks.values()) if isinstance(cs.chunks, dict) \
        else sum(ch.bytes for ch in cs.chunks)
    assert pool.slab_bytes < every_chunk
