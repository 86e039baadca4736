"""Long-horizon ZeRO run: p ranks sharing cuda:0 over gloo for --steps steps
on a learnable stream, against one rank on the concatenated batch.  Reports
the per-step mean-of-ranks loss vs the single-rank loss, and HBM in use at
the start / end of the run (a slab or group-buffer leak would grow it).

    python scripts/dp_long.py [--world 2] [--steps 100]
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KW = dict(layers=4, hidden_dim=512, heads=8, seq_len=256, vocab=8192, batch=4)
# untied LM head everywhere: the embedding placement rule depends on the batch
# (per rank vs concatenated), and a tied head would make it a different model


def stream(steps, world, batch):
    import torch
    g = torch.Generator().manual_seed(11)
    table = torch.randint(0, 8192, (8192, 4), generator=g)
    out = []
    for _ in range(steps):
        st = torch.empty(world * batch, 257, dtype=torch.int64)
        st[:, 0] = torch.randint(0, 8192, (world * batch,), generator=g)
        for t in range(256):
            st[:, t + 1] = table[st[:, t], torch.randint(0, 4, (world * batch,), generator=g)]
        out.append(st)
    return out


def worker(rank, world, port, outdir, steps, budget):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2108_05818_b200 import kernels as K
        from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
        from paper_2108_05818_b200.model import build_gpt_schema
        from paper_2108_05818_b200.trainer import ChunkTrainer
        schema = build_gpt_schema(**KW)
        tr = ChunkTrainer(schema, PolicySpec(capacity_elems=4 * 512 * 512),
                          HardwareSpec(gpu_count=world, gpu_bytes=budget), seed=0,
                          hyper=K.AdamHyper(lr=3e-4, betas=(0.9, 0.95)), untied_head=True)
        data = stream(steps, world, KW["batch"])
        losses, mem = [], []
        for i, b in enumerate(data):
            losses.append(tr.step_host(b[rank * KW["batch"]:(rank + 1) * KW["batch"]]))
            if i in (5, steps - 1):
                tr.finish_host_work()
                torch.cuda.synchronize()
                mem.append(torch.cuda.memory_allocated())
        st = tr.executor.stats
        torch.save({"losses": losses, "mem": mem, "gathers": st.gathers,
                    "reduce_scatters": st.reduce_scatters, "copies": st.copies},
                   os.path.join(outdir, "r%d.pt" % rank))
    finally:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--budget-mb", type=int, default=0, help="per-rank GPU budget (0: roomy)")
    ap.add_argument("--tight", action="store_true",
                    help="budget 20%% above the smallest feasible one for every rank")
    a = ap.parse_args()
    import torch
    import torch.multiprocessing as mp
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    budget = a.budget_mb << 20 if a.budget_mb else 180 * 10 ** 9
    if a.tight:
        from paper_2108_05818_b200.scenario import Simulator
        schema = build_gpt_schema(**KW)

        def ok(b):
            return all(all(r.feasible for r in Simulator(
                schema, HardwareSpec(gpu_count=a.world, gpu_bytes=b),
                PolicySpec(capacity_elems=4 * 512 * 512), nproc=a.world, rank=k).run(3).reports)
                for k in range(a.world))
        lo, hi = 1 << 20, 1 << 34
        while hi - lo > (1 << 18):
            mid = (lo + hi) // 2
            hi, lo = (mid, lo) if ok(mid) else (hi, mid)
        budget = int(hi * 1.2)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(a.world, 29450 + os.getpid() % 100, d, a.steps, budget),
                 nprocs=a.world, join=True)
        res = [torch.load(os.path.join(d, "r%d.pt" % r), weights_only=False)
               for r in range(a.world)]
    kw = dict(KW, batch=KW["batch"] * a.world)
    tr = ChunkTrainer(build_gpt_schema(**kw), PolicySpec(capacity_elems=4 * 512 * 512),
                      HardwareSpec(gpu_count=1, gpu_bytes=180 * 10 ** 9), seed=0,
                      hyper=K.AdamHyper(lr=3e-4, betas=(0.9, 0.95)), untied_head=True)
    single = [tr.step_host(b) for b in stream(a.steps, a.world, KW["batch"])]
    mean_dp = [sum(r["losses"][i] for r in res) / a.world for i in range(a.steps)]
    rel = [abs(x - y) / abs(y) for x, y in zip(mean_dp, single)]
    print(json.dumps({"world": a.world, "steps": a.steps, "budget_bytes": budget,
                      "single_first_last": [single[0], single[-1]],
                      "dp_mean_first_last": [mean_dp[0], mean_dp[-1]],
                      "max_rel_diff": max(rel), "mean_rel_diff": sum(rel) / len(rel),
                      "hbm_in_use_step5_vs_last": [r["mem"] for r in res],
                      "gathers": [r["gathers"] for r in res],
                      "reduce_scatters": [r["reduce_scatters"] for r in res],
                      "copies": [r["copies"] for r in res]}), flush=True)


if __name__ == "__main__":
    main()
