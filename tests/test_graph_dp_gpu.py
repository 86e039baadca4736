"""CUDA-graph capture of the ZeRO step (``graph_multi_rank``), checked on one GPU.

NCCL refuses two ranks on one device and gloo collectives are host calls,
so neither can run inside a stream capture here.  ``MirrorComm`` stands in
for NCCL's completion semantics without a peer: every collective runs on a
side stream forked from the caller's stream (as torch's NCCL process group
does), lands late (a spin first, the receive buffer poisoned with NaN until
then) and is joined only by ``work.wait()`` (or at once for a synchronous
call).  Its peers are mirrors of this rank: a gathered remote slot receives
a copy of this rank's own contribution, a reduce-scatter's average over p
identical contributions is this rank's slot, an all-reduce sum is p times
the value.  That is not training the reference's model, but it is
deterministic, so an eagerly executed run and a run whose steady state is a
captured graph must agree bit for bit -- and a capture-illegal call in the
ZeRO path (a host wait, an event query, a collective whose Work is never
joined before the capture ends) fails the capture outright.  The decision
ledgers must still equal the reference's for this rank.
"""

import gzip
import json
import os

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decisions.json.gz")
STEPS = 8


class _Work:
    def __init__(self, event):
        self.event = event

    def wait(self):
        if os.environ.get("CS_TEST_DROP_WAITS") == "1":  # mutation check: must fail
            return
        torch.cuda.current_stream().wait_event(self.event)


class MirrorComm:
    """ChunkComm's interface for rank ``rank`` of ``world`` mirrored ranks."""

    def __init__(self, world: int, rank: int, delay_cycles: int = 200_000):
        self.world, self.rank = world, rank
        self.side = torch.cuda.Stream()
        self.delay = delay_cycles
        self.calls = []
        self.keep = []

    def _run(self, dst, fill, async_op):
        self.side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.side):
            dst.fill_(float("nan"))       # nothing is valid before wait()
            torch.cuda._sleep(self.delay)
            fill()
        ev = torch.cuda.Event()
        ev.record(self.side)
        work = _Work(ev)
        if async_op:
            return work
        work.wait()
        return None

    def all_gather_slab(self, slab, async_op=False, src=None):
        cap = slab.numel() // self.world
        self.calls.append(("all_gather", slab.numel() * slab.element_size()))
        mine = slab[self.rank * cap:(self.rank + 1) * cap] if src is None else src[:cap]
        if src is None:  # in place: keep the contribution before the poison
            mine = mine.clone()
            self.keep.append(mine)  # read on the side stream: never recycled early

        def fill():
            slab.view(self.world, cap).copy_(mine.unsqueeze(0).expand(self.world, cap))
        return self._run(slab, fill, async_op)

    def reduce_scatter_avg(self, out, slab, async_op=False):
        cap = out.numel()
        self.calls.append(("reduce_scatter", slab.numel() * slab.element_size()))
        if out.data_ptr() == slab[self.rank * cap:].data_ptr():
            return self._run(out[:0], lambda: None, async_op)  # in place: already the mean
        slot = slab[self.rank * cap:(self.rank + 1) * cap]
        return self._run(out, lambda: out.copy_(slot), async_op)

    def all_reduce_sum(self, t):
        self._run(t[:0], lambda: t.mul_(self.world), False)

    def all_reduce_avg(self, t):
        pass

    def check(self):
        pass


def _case(name):
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)["cases"][name]


def _run(case, rank, graph):
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = _case(case)
    schema = build_gpt_schema(**c["schema"])
    comm = MirrorComm(c["nproc"], rank)
    tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                      dtype=torch.float16, seed=0, comm=comm, cuda_graph=graph,
                      graph_multi_rank=graph)
    assert tr.nproc == c["nproc"] and tr.rank == rank
    g = torch.Generator().manual_seed(91 + rank)
    batches = [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
               for _ in range(4)]
    losses = [tr.step_host(batches[i % 4]) for i in range(STEPS)]
    torch.cuda.synchronize()
    from paper_2108_05818_b200.chunks import ChunkKind
    params = torch.cat([tr.local_chunk_payload(pos, kind).float().cpu()
                        for pos in tr.sim.local for kind in ChunkKind])
    reports = [([[t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason] for t in r.transfers],
                [[x.iteration, x.group_id, x.kind, x.bytes, x.includes_padding]
                 for x in r.collectives]) for r in tr.reports]
    out = {"losses": losses, "params": params, "reports": reports,
           "captured": tr._graph is not None, "calls": len(comm.calls),
           "state": tr.step_state()}
    tr.close()
    return out


@pytest.mark.parametrize("case,rank", [("tiny_p2", 0), ("tiny_p2", 1), ("tiny_p8", 7),
                                       ("tiny_p2_ckpt", 1)])
def test_captured_zero_step_matches_eager(case, rank):
    eager = _run(case, rank, graph=False)
    graph = _run(case, rank, graph=True)
    assert not eager["captured"] and graph["captured"]
    assert all(l == l for l in eager["losses"]), eager["losses"]
    # bit-identical: every loss and every parameter the run ends with
    assert graph["losses"] == eager["losses"]
    assert torch.equal(graph["params"], eager["params"])
    assert bytes(graph["state"]) == bytes(eager["state"])  # step, loss scale, scalars
    # the captured steps replayed their collectives: the eager run issued them
    # every step, the graph run only until (and including) the capture
    assert eager["calls"] > graph["calls"] > 0
    ref = _case(case)["ranks"][str(rank)]["iterations"]
    for runs in (eager, graph):
        for (tr, co), theirs in zip(runs["reports"], ref):
            assert tr == theirs["transfers"] and co == theirs["collectives"]
        # steady state: every later iteration repeats the reference's last one
        for tr, co in runs["reports"][len(ref):]:
            assert tr == ref[-1]["transfers"]
            assert [x[1:] for x in co] == [x[1:] for x in ref[-1]["collectives"]]
