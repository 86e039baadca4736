"""Multi-rank ZeRO chunk-group data path on CPU (gloo, world size 2 and 4).

The product executor (paper_2108_05818_b200/payload.py) owns the DP data
path: group slabs, remote members as slot views, in-place all-gather with a
zero phantom slot, reduce-scatter(avg) fed from the BWD slab plus the local
chunk's grads.  Here a test double overrides only its device primitives
(payload allocation and copies become host tensors, the Adam kernels become
the C oracle) and the REAL gather / reduce-scatter / binding code runs over
gloo while the accounting engine drives the iteration.

Every rank writes fake, exactly-representable gradients
g = ((rank + 1) + (e mod 7)) * 2^-10 into each BWD operator's parameter
views.  A single-process replay of the same training (mean gradient, oracle
Adam per tensor) gives the truth; every rank must observe exactly the true
parameters at every FWD and BWD operator of every iteration, and each
rank's own chunks must hold the true parameters at the end.
"""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
from paper_2108_05818_b200.gpt import reference_tensor_shapes
from paper_2108_05818_b200.model import CPU, Phase, build_gpt_schema, param_tensor_specs
from paper_2108_05818_b200.payload import ChunkComm, ChunkPayloadExecutor
from paper_2108_05818_b200.scenario import Simulator

LR, B1, B2, EPS = 1e-3, 0.9, 0.999, 1e-8
ITERS = 3


def _schema():
    return build_gpt_schema(layers=2, hidden_dim=64, heads=4, seq_len=16, vocab=100, batch=2,
                            context_bytes=1000)


CAP = 3 * 64 * 64  # 5 positions per layer -> 10 positions, padded tail at p=4


def _init_values(numel: int, tid: int) -> np.ndarray:
    e = np.arange(numel, dtype=np.float64)
    return (np.sin(e * 0.37 + tid) * 0.02).astype(np.float32)


def _fake_grad(numel: int, rank: int) -> np.ndarray:
    e = np.arange(numel)
    return (((rank + 1) + (e % 7)) * 2.0 ** -10).astype(np.float16)


class _NoSlabs:
    """Host double of the HBM slab pool: payloads are plain host tensors."""

    def give(self, t, side_events=None):
        return False

    def owns(self, t):
        return False

    def free_tensors(self):
        return []


class HostDoubleExecutor(ChunkPayloadExecutor):
    """Device primitives on the host; everything else is the product code."""

    def _setup_device(self, init_loss_scale):
        from oracle import numerics as O
        self.O = O
        self.compute = self.copy_stream = self.state = None
        self.slabs = _NoSlabs()
        self.os_state = O.step_state(1.0)
        self.observed = []

    def _alloc(self, chunk, device):
        return torch.empty(chunk.capacity_elems, dtype=self._elem_dtype(chunk))

    def _alloc_for_copy(self, chunk):
        return self._alloc(chunk, "gpu")

    def _transfer(self, s, d, src, dst, prior):
        d.copy_(s)
        self.stats.copies += 1
        return None

    def on_compute_start(self, ev, chunks):
        super().on_compute_start(ev, chunks)
        for tid in ev.tensor_refs:
            view = self.params[tid].data
            self.observed.append((self._iteration, ev.phase.value, tid,
                                  view.reshape(-1).view(torch.int16).clone()))
            if ev.phase is Phase.BWD:
                g = _fake_grad(view.numel(), self.rank)
                view.reshape(-1).copy_(torch.from_numpy(g))

    def on_adam_begin(self, iteration, plan=None):
        self._gather_prefetched.clear()
        self.wait_collectives()  # as the product: reduce-scatters into local chunks landed
        self.os_state.sumsq = 1.0
        self.O.adam_prepare(self.os_state, LR, B1, B2)

    def init_optimizer_state(self, position, device):
        p32, m, v = (self.tensor(c, device) for c in self.chunk_set.os_triplet(position))
        src = self.init32.pop(position)
        p32.copy_(src)
        m.zero_()
        v.zero_()

    def adam_position(self, position, device):
        cs = self.chunk_set
        param = cs.param_chunk(position)
        n = param.used_elems
        p16 = self.tensor(param, device)
        p32, m, v = (self.tensor(c, device) for c in cs.os_triplet(position))
        self.O.adam(p16.view(torch.int16).numpy().view(np.uint16), p32.numpy(), m.numpy(),
                    v.numpy(), n, self.O.FP16, LR, B1, B2, EPS, 0.0, False, self.os_state)

    def _flush_adam(self):
        self._pending, self._pending_ids = [], set()


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        schema = _schema()
        ex = HostDoubleExecutor("cpu", torch.float16, K.AdamHyper(lr=LR), comm=ChunkComm())
        ex._iteration = 0
        sim = Simulator(schema, HardwareSpec(gpu_count=world, gpu_bytes=10 ** 9,
                                             cpu_bytes=10 ** 10),
                        PolicySpec(capacity_elems=CAP), nproc=world, rank=rank,
                        payload_backend=ex, collective_backend=ex, executor=ex)
        shapes = reference_tensor_shapes(schema)
        params = [torch.nn.Parameter(torch.empty(0, dtype=torch.float16)) for _ in shapes]
        ex.attach(sim.chunk_set, sim.partition, rank, params, shapes)
        ex._placeholder = torch.empty(0, dtype=torch.float16)
        for pos in sim.local:
            chunk = sim.chunk_set.param_chunk(pos)
            p32 = torch.zeros(CAP)
            for t in chunk.tensors:
                p32[t.offset_elems:t.offset_elems + t.numel] = torch.from_numpy(
                    _init_values(t.numel, t.tensor_id))
            ex.payload[CPU][chunk.chunk_id] = p32.half()
            ex.init32[pos] = p32
        for it in range(ITERS):
            ex._iteration = it
            rep = sim.engine.run_iteration(it, warmup=(it == 0),
                                           plan_builder=sim._plan_builder() if it == 0 else None)
            assert rep.feasible
            ex.gather_depth = 2  # as the trainer: prefetch gathers from the previous log
        final = {}
        for pos in sim.local:
            chunk = sim.chunk_set.param_chunk(pos)
            dev = "gpu" if ex.has(chunk, "gpu") else "cpu"
            buf = ex.tensor(chunk, dev)
            for t in chunk.tensors:
                final[t.tensor_id] = buf[t.offset_elems:t.offset_elems + t.numel].view(
                    torch.int16).clone()
        torch.save({"observed": ex.observed, "final": final,
                    "gathers": ex.stats.gathers, "reduce_scatters": ex.stats.reduce_scatters,
                    "gather_prefetch_hits": ex.stats.gather_prefetch_hits,
                    "collectives": [(c.group_id, c.kind) for r in [rep] for c in r.collectives]},
                    os.path.join(outdir, "rank%d.pt" % rank))
    finally:
        dist.destroy_process_group()


def _truth(schema, world):
    """Single-process replay: params (fp16 bits) seen at each iteration, and final."""
    from oracle import numerics as O
    specs = param_tensor_specs(schema)
    state = {s.tensor_id: [_init_values(s.numel, s.tensor_id), np.zeros(s.numel, np.float32),
                           np.zeros(s.numel, np.float32)] for s in specs}
    p16 = {tid: st[0].astype(np.float16).view(np.int16) for tid, st in state.items()}
    seen = []
    os_ = O.step_state(1.0)
    for it in range(ITERS):
        seen.append({tid: v.copy() for tid, v in p16.items()})
        os_.sumsq = 1.0
        O.adam_prepare(os_, LR, B1, B2)
        for s in specs:
            e = np.arange(s.numel)
            g = (((world + 1) / 2.0 + (e % 7)) * 2.0 ** -10).astype(np.float16)
            g16 = g.view(np.uint16).copy()
            p32, m, v = state[s.tensor_id]
            O.adam(g16, p32, m, v, s.numel, O.FP16, LR, B1, B2, EPS, 0.0, False, os_)
            p16[s.tensor_id] = g16.view(np.int16)
    return seen, p16


@pytest.mark.parametrize("world", [2, 4])
def test_zero_chunk_groups_over_gloo(world, oracle_lib):
    schema = _schema()
    port = 29600 + world + (os.getpid() % 200)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, d), nprocs=world, join=True)
        results = [torch.load(os.path.join(d, "rank%d.pt" % r), weights_only=False)
                   for r in range(world)]
    seen, final = _truth(schema, world)
    n_tensors = len(param_tensor_specs(schema))
    for r, res in enumerate(results):
        assert res["gathers"] > 0 and res["reduce_scatters"] > 0
        assert res["gather_prefetch_hits"] > 0  # async gathers issued ahead were adopted
        checked = 0
        for it, phase, tid, bits in res["observed"]:
            np.testing.assert_array_equal(bits.numpy(), seen[it][tid],
                                          err_msg="rank %d it %d %s tensor %d" % (r, it, phase, tid))
            checked += 1
        assert checked == ITERS * 2 * n_tensors  # every tensor, FWD and BWD, every iteration
        for tid, bits in res["final"].items():
            np.testing.assert_array_equal(bits.numpy(), final[tid])
    # every rank issued the same collective sequence
    assert len({tuple(res["collectives"]) for res in results}) == 1
    owned = sorted(t for res in results for t in res["final"])
    assert owned == list(range(n_tensors))
