"""Training demo of the chunk-managed step on a learnable synthetic task.

Tokens follow a fixed random Markov chain over a random subset of the
vocabulary (every token has K equally likely successors), so the achievable
loss is ln(K) while a model that learned nothing sits at ln(V).  The 1B GPT (or --layers/--hidden) trains for --steps
with fp16 chunks, dynamic loss scaling, chunk Adam and CUDA-graph replay;
prints one JSON line per --every steps and a summary.

    python scripts/train_demo.py [--steps 300] [--layers 20] [--hidden 2048] [--batch 16]
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--layers", type=int, default=20)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--vocab", type=int, default=50304)
    ap.add_argument("--succ", type=int, default=4, help="successors per token (loss floor ln K)")
    ap.add_argument("--active", type=int, default=2048,
                    help="tokens the chain visits (a random subset of the vocabulary)")
    ap.add_argument("--lr", type=float, default=3e-4)
    ap.add_argument("--every", type=int, default=25)
    ap.add_argument("--os", default="auto", choices=["auto", "cpu", "gpu"],
                    help="optimizer-state placement policy")
    ap.add_argument("--gpu-gb", type=float, default=0.0,
                    help="accounting GPU budget in GB (0: 90%% of HBM) — small values evict")
    ap.add_argument("--deterministic", action="store_true",
                    help="deterministic attention backend (bit-comparable runs)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--ckpt", action="store_true", help="activation checkpointing")
    a = ap.parse_args()
    import torch
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1234)
    vocab_ids = torch.randperm(a.vocab, device=dev, generator=g)[:a.active]
    table = torch.randint(0, a.active, (a.active, a.succ), device=dev, generator=g)

    def batch():
        state = torch.empty(a.batch, a.seq + 1, dtype=torch.int64, device=dev)
        state[:, 0] = torch.randint(0, a.active, (a.batch,), device=dev, generator=g)
        for t in range(a.seq):
            pick = torch.randint(0, a.succ, (a.batch,), device=dev, generator=g)
            state[:, t + 1] = table[state[:, t], pick]
        return vocab_ids[state]

    schema = build_gpt_schema(layers=a.layers, hidden_dim=a.hidden, heads=a.heads,
                              seq_len=a.seq, vocab=a.vocab, batch=a.batch)
    from paper_2108_05818_b200.config import HardwareSpec
    hw = (HardwareSpec(gpu_count=1, gpu_bytes=int(a.gpu_gb * 1e9), cpu_bytes=150 * 10 ** 9)
          if a.gpu_gb else None)
    cap = 64 << 20 if a.hidden >= 2048 else 4 * a.hidden * a.hidden
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=cap, os_placement=a.os,
                                         checkpointing=a.ckpt), hw, seed=0,
                      dtype=torch.bfloat16 if a.dtype == "bf16" else torch.float16,
                      hyper=K.AdamHyper(lr=a.lr, betas=(0.9, 0.95)), cuda_graph=not a.no_graph)
    if a.deterministic:  # keep the context object alive for the whole run
        from torch.nn.attention import SDPBackend, sdpa_kernel
        deterministic_ctx = sdpa_kernel(SDPBackend.MATH)
        deterministic_ctx.__enter__()
    t0 = time.perf_counter()
    losses = []
    for i in range(a.steps):
        loss = float(tr.step(batch()).item())
        losses.append(loss)
        if (i + 1) % a.every == 0 or i == 0:
            st = tr.step_state()
            print(json.dumps({"step": i + 1, "loss": round(loss, 4),
                              "loss_scale": st.loss_scale, "applied_steps": int(st.step),
                              "grad_norm": round(float(st.grad_norm), 4),
                              "cuda_graph": tr._graph is not None}), flush=True)
    st = tr.step_state()
    print(json.dumps({"summary": True, "model": "GPT L%d H%d" % (a.layers, a.hidden),
                      "steps": a.steps, "first_loss": round(losses[0], 4),
                      "last10_mean_loss": round(sum(losses[-10:]) / 10, 4),
                      "ln_vocab": round(math.log(a.vocab), 4),
                      "ln_successors_floor": round(math.log(a.succ), 4),
                      "skipped_steps": a.steps - int(st.step), "final_loss_scale": st.loss_scale,
                      "wall_s": round(time.perf_counter() - t0, 1),
                      "all_finite": all(math.isfinite(x) for x in losses),
                      "host_adam_items": tr.executor.stats.host_adam_items,
                      "chunk_copies": tr.executor.stats.copies,
                      "losses": [round(x, 6) for x in losses]}), flush=True)


if __name__ == "__main__":
    main()
