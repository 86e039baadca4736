"""GPU idle gaps of eager steps (torch.profiler kernel timeline): where does
an eager step lose time against the graph-replayed one?

    python scripts/gpu_gaps.py [batch]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    arg = sys.argv[1] if len(sys.argv) > 1 else "32"
    if arg.isdigit():
        B = int(arg)
        schema = build_gpt_schema(layers=20, hidden_dim=2048, heads=16, seq_len=1024,
                                  vocab=50304, batch=B)
        pol = PolicySpec(capacity_elems=64 << 20)
    else:  # a scripts/configs_sweep.py configuration
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from configs_sweep import CONFIGS
        c = CONFIGS[arg]
        B = c["batch"]
        schema = build_gpt_schema(layers=c["layers"], hidden_dim=c["hidden"], heads=c["heads"],
                                  seq_len=1024, vocab=50304, batch=B)
        pol = PolicySpec(capacity_elems=c["cap"], os_placement=c["os"],
                         checkpointing=c.get("ckpt", False))
    tr = ChunkTrainer(schema, pol, seed=0, hyper=K.AdamHyper(lr=1e-4))
    tok = torch.randint(0, 50304, (B, 1025)).cuda()
    for _ in range(3):
        tr.step(tok)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            tr.step(tok)
        torch.cuda.synchronize()
    kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                   if e.device_type == torch.autograd.DeviceType.CUDA],
                  key=lambda x: x[0])
    busy, gaps = 0.0, []
    t_end = kern[0][1]
    for s, e, n in kern:
        if s > t_end:
            gaps.append((s - t_end, n))
        busy += max(0, e - max(s, t_end)) if e > t_end else 0
        t_end = max(t_end, e)
    span = kern[-1][1] - kern[0][0]
    print("kernels %d, span %.1f ms, busy %.1f ms, idle %.1f ms (2 steps)"
          % (len(kern), span / 1e3, busy / 1e3, (span - busy) / 1e3))
    gaps.sort(reverse=True)
    print("largest gaps (us, next kernel):")
    for g, n in gaps[:15]:
        print("  %8.1f  %s" % (g, n[:100]))
    small = [g for g, _ in gaps if g < 50]
    print("gaps < 50 us: %d totalling %.1f ms" % (len(small), sum(small) / 1e3))
    agg = {}
    for s_, e_, n in kern:
        key = n[:60]
        a = agg.setdefault(key, [0.0, 0])
        a[0] += (e_ - s_) / 1e3
        a[1] += 1
    print("per-kernel time in these steps (ms, launches):")
    for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
        print("  %8.3f %5d  %s" % (t / 2, c // 2, k))


if __name__ == "__main__":
    main()
