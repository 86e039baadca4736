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


def test_side_events_order_only_the_slabs_own_copies():
    """give(side_events=...): the next taker waits for the slab's own copy on
    a side stream (its bytes are read before they are overwritten) but not
    for unrelated work queued behind it on that stream."""
    from paper_2108_05818_b200.slabs import SlabPool
    compute, d2h = torch.cuda.current_stream(), torch.cuda.Stream()
    pool = SlabPool(torch.device("cuda", 0), [compute, d2h], max_free=4)
    n = 1 << 24
    a = pool.take(n, torch.float16, compute)
    a.fill_(3.0)
    host = torch.empty(n, dtype=torch.float16, pin_memory=True)
    d2h.wait_stream(compute)
    with torch.cuda.stream(d2h):
        torch.cuda._sleep(20_000_000)            # the copy lands late ...
        host.copy_(a, non_blocking=True)
        own = torch.cuda.Event()
        own.record(d2h)
        torch.cuda._sleep(400_000_000)           # ... and unrelated work queues behind it
    assert pool.give(a, [own])
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(compute)
    b = pool.take(n, torch.float16, compute)
    assert b.data_ptr() == a.data_ptr()
    b.fill_(7.0)                                  # must not reach the copy's source early
    t1.record(compute)
    t1.synchronize()
    assert bool((host == 3.0).all())              # the copy read the slab before the refill
    slept = t0.elapsed_time(t1)
    # the taker waited for the late copy (~20M cycles) but not for the 400M-cycle tail
    ev_tail = torch.cuda.Event(enable_timing=True)
    ev_tail.record(d2h)
    ev_tail.synchronize()
    assert slept < 0.5 * t0.elapsed_time(ev_tail), (slept, t0.elapsed_time(ev_tail))


def test_side_events_free_to_the_allocator_in_compute_order():
    """Beyond max_free a slab goes back to the caching allocator; with side
    events the compute stream waits for them first, so a later allocation
    on the compute stream cannot overwrite bytes a copy still reads."""
    from paper_2108_05818_b200.slabs import SlabPool
    compute, d2h = torch.cuda.current_stream(), torch.cuda.Stream()
    pool = SlabPool(torch.device("cuda", 0), [compute, d2h], max_free=0)
    n = 1 << 24
    a = pool.take(n, torch.float16, compute)
    a.fill_(5.0)
    host = torch.empty(n, dtype=torch.float16, pin_memory=True)
    d2h.wait_stream(compute)
    with torch.cuda.stream(d2h):
        torch.cuda._sleep(50_000_000)
        host.copy_(a, non_blocking=True)
        own = torch.cuda.Event()
        own.record(d2h)
    assert pool.give(a, [own])
    del a
    c = torch.empty(n, dtype=torch.float16, device="cuda")  # may reuse the block
    c.fill_(9.0)
    torch.cuda.synchronize()
    assert bool((host == 5.0).all())
