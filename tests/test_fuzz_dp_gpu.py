"""Seeded random configurations through the REAL multi-rank ZeRO step (p
ranks sharing cuda:0 over gloo).  For each seed: random tiny GPT, capacity,
world size p in {2, 3, 4}, eviction strategy, checkpointing, optimizer-state
placement and a per-rank GPU budget just above the smallest feasible one for
every rank (found with the accounting-only engine, so gathered remote chunks
get evicted).  Every rank's transfer and collective ledgers must equal the
accounting-only engine of that rank (pinned to the reference on random
configurations by tests/test_decisions_fuzz.py), and every rank must move
exactly the bytes it bills.  Odd seeds run with collectives that land late on a
side stream with NaN-poisoned receive buffers (tests/test_dp_stream_order_gpu.py),
so every read of collective results must be stream-ordered as under NCCL."""

import os
import random
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

ITERS = 3


def _config(seed):
    r = random.Random(500 + seed)
    H = r.choice([128, 256])
    schema = dict(layers=r.choice([2, 3, 4]), hidden_dim=H, heads=4, seq_len=r.choice([64, 128]),
                  batch=r.choice([2, 4]), vocab=r.choice([512, 4096]), context_bytes=2 << 20)
    policy = dict(capacity_elems=r.choice([2, 4]) * H * H, checkpointing=r.random() < 0.4,
                  os_placement=r.choice(["auto", "auto", "cpu"]),
                  eviction=r.choice(["latest_next_use", "list_order"]))
    return schema, policy, r.choice([2, 3, 4]), r.uniform(1.05, 1.3)


def _sim(schema, policy, world, rank, gpu_bytes):
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.memory import EvictionStrategy
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.scenario import Simulator
    pol = PolicySpec(**dict(policy, eviction=EvictionStrategy(policy["eviction"])))
    return Simulator(build_gpt_schema(**schema), HardwareSpec(gpu_count=world, gpu_bytes=gpu_bytes),
                     pol, nproc=world, rank=rank).run(ITERS)


def _budget(schema, policy, world, slack):
    lo, hi = 1 << 20, 1 << 34
    while hi - lo > (256 << 10):
        mid = (lo + hi) // 2
        if all(all(r.feasible for r in _sim(schema, policy, world, k, mid).reports)
               for k in range(world)):
            hi = mid
        else:
            lo = mid
    return int(hi * slack)


def _rows(r):
    return ([[t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason] for t in r.transfers],
            [[c.iteration, c.group_id, c.kind, c.bytes, c.includes_padding]
             for c in r.collectives])


def _worker(rank, world, port, outdir, schema_kw, policy, budget, late=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
        from paper_2108_05818_b200.memory import EvictionStrategy
        from paper_2108_05818_b200.model import build_gpt_schema
        from paper_2108_05818_b200.trainer import ChunkTrainer
        schema = build_gpt_schema(**schema_kw)
        pol = PolicySpec(**dict(policy, eviction=EvictionStrategy(policy["eviction"])))
        comm = None
        if late:  # collectives that land late on a side stream (NCCL-style completion)
            from test_dp_stream_order_gpu import StreamOrderedComm
            comm = StreamOrderedComm()
        tr = ChunkTrainer(schema, pol, HardwareSpec(gpu_count=world, gpu_bytes=budget),
                          dtype=torch.float16, seed=0, comm=comm)
        g = torch.Generator().manual_seed(rank)
        losses = [tr.step_host(torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1),
                                             generator=g)) for _ in range(ITERS)]
        tr.finish_host_work()
        st = tr.executor.stats
        torch.save({"rows": [_rows(r) for r in tr.reports], "losses": losses,
                    "applied": int(tr.step_state().step),
                    "h2d": st.h2d_bytes - st.prefetch_discarded_bytes, "d2h": st.d2h_bytes},
                   os.path.join(outdir, "rank%d.pt" % rank))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", range(8))
def test_random_config_real_zero_step(seed):
    schema, policy, world, slack = _config(seed)
    budget = _budget(schema, policy, world, slack)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, 29300 + seed * 10 + os.getpid() % 50 * 50, d, schema,
                                policy, budget, seed % 2 == 1), nprocs=world, join=True)
        res = [torch.load(os.path.join(d, "rank%d.pt" % k), weights_only=False)
               for k in range(world)]
    for k in range(world):
        ref = _sim(schema, policy, world, k, budget)
        assert res[k]["rows"] == [_rows(r) for r in ref.reports], (seed, k)
        assert all(x == x and abs(x) < 1e4 for x in res[k]["losses"]) and \
            res[k]["applied"] == ITERS, (seed, k, res[k]["losses"])
        billed = [t for r in ref.reports for t in r.transfers if t.chunk_id != "embedding"]
        assert res[k]["h2d"] == sum(t.bytes for t in billed if (t.src, t.dst) == ("cpu", "gpu"))
        assert res[k]["d2h"] == sum(t.bytes for t in billed if (t.src, t.dst) == ("gpu", "cpu"))
