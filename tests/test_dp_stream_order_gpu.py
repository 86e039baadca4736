"""The ZeRO executor under NCCL's completion semantics, made adversarial.

With NCCL a collective completes on a stream: ``work.wait()`` only orders the
caller's stream after it, and nothing in the receive buffer is valid before
that point.  Gloo (what the multi-rank tests on one GPU must use) blocks the
host instead, which hides any executor read that is not stream-ordered after
its collective.  ``StreamOrderedComm`` exchanges over gloo but lands every
result LATE: on a side stream, after a ~1 ms spin, with the receive buffer
poisoned (NaN) in the meantime.  A gather slot read before its ``wait()``, a
reduce-scatter output consumed early, or a group slab recycled while the
collective still writes it turns into NaN losses, skipped steps or a ledger /
loss mismatch.  Chunk moves are delayed the same way (the executor's
``copy_delay_cycles`` knob).  Cases follow tests/test_dp_step_gpu.py.
"""

import gzip
import json
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decisions.json.gz")
ITERS = 3


class _Work:
    def __init__(self, event):
        self.event = event

    def wait(self):
        if os.environ.get("CS_TEST_DROP_WAITS") == "1":  # mutation check: must fail
            return
        torch.cuda.current_stream().wait_event(self.event)


class StreamOrderedComm:
    """ChunkComm's interface; results land on the device late (see module doc)."""

    def __init__(self, delay_cycles: int = 2_000_000):
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.side = torch.cuda.Stream()
        self.delay = delay_cycles
        self.calls = []
        self.keep = []  # pinned staging buffers, alive until their copies ran

    def _land(self, dst, host, async_op):
        self.side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.side):
            dst.fill_(float("nan"))           # nothing is valid before wait()
            torch.cuda._sleep(self.delay)
            dst.copy_(host, non_blocking=True)
        dst.record_stream(self.side)
        ev = torch.cuda.Event()
        ev.record(self.side)
        self.keep = [k for k in self.keep if not k[0].query()] + [(ev, host)]
        work = _Work(ev)
        if async_op:
            return work
        work.wait()
        return None

    def all_gather_slab(self, slab, async_op=False, src=None):
        cap = slab.numel() // self.world
        self.calls.append(("all_gather", slab.numel() * slab.element_size()))
        mine = (slab[self.rank * cap:(self.rank + 1) * cap] if src is None
                else src[:cap]).cpu()  # after the contribution's writes
        out = torch.empty(slab.numel(), dtype=slab.dtype)
        dist.all_gather_into_tensor(out, mine)
        return self._land(slab, out.pin_memory(), async_op)

    def reduce_scatter_avg(self, out, slab, async_op=False):
        self.calls.append(("reduce_scatter", slab.numel() * slab.element_size()))
        host = slab.cpu()
        res = torch.empty(out.numel(), dtype=out.dtype)
        dist.reduce_scatter_tensor(res, host, op=dist.ReduceOp.AVG)
        return self._land(out, res.pin_memory(), async_op)

    def all_reduce_sum(self, t):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM)
        t.copy_(h)

    def all_reduce_avg(self, t):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.AVG)
        t.copy_(h)


def _case(name):
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)["cases"][name]


def _batches(schema, rank, n):
    g = torch.Generator().manual_seed(77 + rank)
    return [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
            for _ in range(n)]


def _worker(rank, world, port, outdir, case, place, async_adam):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
        from paper_2108_05818_b200.model import build_gpt_schema
        from paper_2108_05818_b200.trainer import ChunkTrainer
        c = _case(case)
        schema = build_gpt_schema(**c["schema"])
        comm = StreamOrderedComm()
        tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                          dtype=torch.float16, seed=0, embedding_placement=place,
                          untied_head=True if place != "plan" else None,
                          async_host_adam=async_adam, comm=comm)
        assert tr.nproc == world and tr.rank == rank and tr.executor.comm is comm
        tr.executor.copy_delay_cycles = 1_000_000  # chunk moves land late as well
        losses = [tr.step_host(b) for b in _batches(schema, rank, ITERS)]
        tr.finish_host_work()
        torch.cuda.synchronize()
        st = tr.step_state()
        reports = [{"transfers": [[t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason]
                                  for t in r.transfers],
                    "collectives": [[x.iteration, x.group_id, x.kind, x.bytes, x.includes_padding]
                                    for x in r.collectives]} for r in tr.reports]
        torch.save({"losses": losses, "reports": reports, "applied": int(st.step),
                    "calls": len(comm.calls), "prefetch": tr.executor.stats.gather_prefetch_hits},
                   os.path.join(outdir, "rank%d.pt" % rank))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world,place,async_adam", [
    ("tiny_p2", 2, "plan", False), ("tiny_p4_tight", 4, "plan", False),
    ("tiny_p8", 8, "plan", False), ("tiny_p2_ckpt", 2, "plan", False),
    ("tiny_p2", 2, "gpu", False), ("tiny_p4_tight", 4, "cpu", True)])
def test_zero_step_with_late_landing_collectives(case, world, place, async_adam):
    with tempfile.TemporaryDirectory() as d:
        port = 30300 + world * 10 + (place == "gpu") + 2 * async_adam + os.getpid() % 50 * 40
        mp.spawn(_worker, args=(world, port, d, case, place, async_adam), nprocs=world,
                 join=True)
        res = [torch.load(os.path.join(d, "rank%d.pt" % r), weights_only=False)
               for r in range(world)]
    c = _case(case)
    for r in range(world):
        assert all(np.isfinite(res[r]["losses"])), res[r]["losses"]
        assert res[r]["applied"] == ITERS            # no step skipped on poisoned grads
        assert res[r]["calls"] > 0 and res[r]["prefetch"] > 0
        for mine, theirs in zip(res[r]["reports"], c["ranks"][str(r)]["iterations"]):
            assert mine["transfers"] == theirs["transfers"], r
            assert mine["collectives"] == theirs["collectives"], r

    # one rank on the concatenated batch, as in tests/test_dp_step_gpu.py
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    kw = dict(c["schema"])
    kw["batch"] = kw["batch"] * world
    tr = ChunkTrainer(build_gpt_schema(**kw), PolicySpec(**c["policy"]),
                      HardwareSpec(gpu_count=1, gpu_bytes=180 * 10**9), dtype=torch.float16,
                      seed=0, embedding_placement=place,
                      untied_head=True if place != "plan" else None)
    schema1 = build_gpt_schema(**c["schema"])
    per_rank = [_batches(schema1, r, ITERS) for r in range(world)]
    single = [tr.step_host(torch.cat([per_rank[r][i] for r in range(world)]))
              for i in range(ITERS)]
    mean_dp = [float(np.mean([res[r]["losses"][i] for r in range(world)])) for i in range(ITERS)]
    np.testing.assert_allclose(mean_dp, single, rtol=2e-3)
