"""Long-horizon placement invariance: one process, the same model, data and
seeds under three placements — all resident, every optimizer triplet in host
DRAM (host Adam, async), and a GPU budget just above the smallest feasible
one (evictions) — for --steps steps with a deterministic attention backend.
The loss trajectories and final parameters must be bit-identical.

    python scripts/placement_invariance_long.py [--steps 150]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=150)
    a = ap.parse_args()
    import torch
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.scenario import Simulator
    from paper_2108_05818_b200.trainer import ChunkTrainer
    kw = dict(layers=4, hidden_dim=1024, heads=8, seq_len=512, vocab=50304, batch=16)
    schema = build_gpt_schema(**kw)
    cap = 4 << 20
    lo, hi = 1 << 24, 1 << 36
    while hi - lo > (1 << 22):   # smallest feasible GPU budget (accounting only)
        mid = (lo + hi) // 2
        run = Simulator(schema, HardwareSpec(gpu_count=1, gpu_bytes=mid, cpu_bytes=150 * 10 ** 9),
                        PolicySpec(capacity_elems=cap)).run(3)
        ok = all(r.feasible for r in run.reports)
        hi, lo = (mid, lo) if ok else (hi, mid)
    tight = int(hi * 1.15)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(7)
    active = torch.randperm(50304, device=dev, generator=g)[:2048]
    table = torch.randint(0, 2048, (2048, 4), device=dev, generator=g)
    batches = []
    for _ in range(a.steps):
        st = torch.empty(16, 513, dtype=torch.int64, device=dev)
        st[:, 0] = torch.randint(0, 2048, (16,), device=dev, generator=g)
        for t in range(512):
            st[:, t + 1] = table[st[:, t], torch.randint(0, 4, (16,), device=dev, generator=g)]
        batches.append(active[st].cpu())
    runs = {}
    configs = {"resident": (PolicySpec(capacity_elems=cap), None),
               "host_optimizer_state": (PolicySpec(capacity_elems=cap, os_placement="cpu"), None),
               "tight_budget": (PolicySpec(capacity_elems=cap),
                                HardwareSpec(gpu_count=1, gpu_bytes=tight, cpu_bytes=150 * 10 ** 9))}
    with sdpa_kernel(SDPBackend.MATH):
        for name, (pol, hw) in configs.items():
            tr = ChunkTrainer(schema, pol, hw, seed=0, hyper=K.AdamHyper(lr=3e-4, betas=(0.9, 0.95)))
            losses = [tr.step_host(b) for b in batches]
            tr.finish_host_work()
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            st = tr.executor.stats
            runs[name] = (losses, params)
            print(json.dumps({"config": name, "first_loss": losses[0], "last_loss": losses[-1],
                              "host_adam_items": st.host_adam_items, "chunk_copies": st.copies,
                              "h2d_gb": round(st.h2d_bytes / 1e9, 2),
                              "d2h_gb": round(st.d2h_bytes / 1e9, 2),
                              "skipped": a.steps - int(tr.step_state().step)}), flush=True)
            del tr
            torch.cuda.empty_cache()
    base = runs["resident"]
    out = {"steps": a.steps, "tight_budget_bytes": tight}
    for name, (losses, params) in runs.items():
        out[name] = {"losses_identical": losses == base[0],
                     "params_identical": all(torch.equal(x.view(torch.int16), y.view(torch.int16))
                                             for x, y in zip(params, base[1]))}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
