"""HBM bandwidth by read:write mix on this B200, beside the chunk kernels of
the same mix — the roofline for write-heavy kernels (K4 accumulate reads
4 B / writes 2 B per element; K6 state birth reads 2 B / writes 12 B).

Streams (4 GiB-class buffers, far beyond the 126 MB L2, CUDA events, best
of 5): read-only (torch sum of fp16), write-only (fill_), copy 1:1
(copy_), plus K2 (read only), K3 pack (1:1), K4 (2:1), K5 cast+pack
(4 B read : 2 B write), K6 (1:6).  Prints one JSON line per stream.

    python scripts/hbm_mix.py
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2108_05818_b200 import kernels as K  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    n = 1 << 30  # elements
    dev = "cuda"
    h = torch.randn(n, device=dev).half()
    h2 = torch.empty_like(h)
    f32 = torch.empty(n, device=dev)
    m = torch.empty(n, device=dev)
    v = torch.empty(n, device=dev)
    scratch = torch.empty(K.sumsq_scratch([(h, n)]), device=dev)
    item_sums = torch.empty(1, dtype=torch.float64, device=dev)
    out = torch.empty((), device=dev, dtype=torch.float32)
    rows = [
        ("read_only torch.sum fp16", lambda: torch.sum(h, dim=0, dtype=torch.float32, out=out),
         2, 0),
        ("write_only fill_ fp32", lambda: f32.fill_(1.0), 0, 4),
        ("copy_ fp16 1:1", lambda: h2.copy_(h), 2, 2),
        ("K2 grad_sumsq", lambda: K.grad_sumsq([(h, n)], scratch, item_sums), 2, 0),
        ("K3 pack", lambda: K.pack([(h2, 0, h, n)]), 2, 2),
        ("K4 accumulate", lambda: K.pack([(h2, 0, h, n)], accumulate=True), 4, 2),
        ("K5 cast_pack", lambda: K.cast_pack([(h2, 0, f32, n)]), 4, 2),
        ("K6 master_init", lambda: K.master_init(f32, m, v, h, n), 2, 12),
    ]
    for name, fn, rb, wb in rows:
        ms = timed(fn)
        gbs = (rb + wb) * n / (ms * 1e-3) / 1e9
        print(json.dumps({"stream": name, "read_B_per_elem": rb, "write_B_per_elem": wb,
                          "ms": round(ms, 3), "gbs": round(gbs, 1)}), flush=True)


if __name__ == "__main__":
    main()
