"""Host-side profile of eager chunk-managed steps (where the enqueue time goes).

    python scripts/profile_host.py [batch] [steps] [sweep-config]

Runs the 1B bench model (or a scripts/configs_sweep.py configuration)
eagerly (no CUDA graph) and prints cProfile's top functions by own time over
`steps` steps after warm-up."""

import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    if len(sys.argv) > 3:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from configs_sweep import CONFIGS
        c = CONFIGS[sys.argv[3]]
        B = c["batch"]
        schema = build_gpt_schema(layers=c["layers"], hidden_dim=c["hidden"], heads=c["heads"],
                                  seq_len=1024, vocab=50304, batch=B)
        pol = PolicySpec(capacity_elems=c["cap"], os_placement=c["os"],
                         checkpointing=c.get("ckpt", False))
    else:
        schema = build_gpt_schema(layers=20, hidden_dim=2048, heads=16, seq_len=1024,
                                  vocab=50304, batch=B)
        pol = PolicySpec(capacity_elems=64 << 20)
    tr = ChunkTrainer(schema, pol, seed=0, hyper=K.AdamHyper(lr=1e-4))
    tok = torch.randint(0, 50304, (B, 1025)).cuda()
    for _ in range(3):
        tr.step(tok)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for _ in range(steps):
        tr.step(tok)
    pr.disable()
    host = (time.perf_counter() - t0) / steps
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) / steps
    print("host enqueue %.1f ms/step, wall %.1f ms/step" % (host * 1e3, tot * 1e3))
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
    pstats.Stats(pr).sort_stats("cumtime").print_stats(30)


if __name__ == "__main__":
    main()
