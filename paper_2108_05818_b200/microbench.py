"""C5 microbench: chunk kernels K1-K6 at 1M-1G elements, HBM GB/s vs roofline.

Algorithmic bytes per element: K1 Adam 28, K2 sumsq 2,
K3 pack 4, K4 accumulate 6, K5 cast+pack 6, K6 state birth 14 (fp16 src).
Each kernel is timed with CUDA events around a CUDA-graph replay of
``iters`` back-to-back launches after warm-up (device time, no host launch
cost); inputs >= 8M elements exceed the 126 MB L2 between iterations,
smaller ones partly hit L2.

    python -m paper_2108_05818_b200.microbench [--sizes 20,22,...] [--iters N]
"""

import argparse
import json
import os
from typing import Callable, Dict, List

import torch

from . import kernels as K

BYTES_PER_ELEM = {"adam": 28, "sumsq": 2, "pack": 4, "accumulate": 6, "cast_pack": 6,
                  "master_init": 14}


def measured_peak_gbs() -> float:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def time_launch(fn: Callable[[], None], iters: int, warmup: int = 3) -> float:
    """Average DEVICE milliseconds per call: the ``iters`` calls are captured
    once into a CUDA graph and replayed between CUDA events, so small sizes
    measure the kernel, not the Python/ctypes launch path."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        for _ in range(iters):
            fn()
    graph.replay()  # warm replay
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    graph.replay()
    end.record()
    torch.cuda.synchronize()
    return start.elapsed_time(end) / iters


def bench_size(n: int, iters: int, dtype=torch.float16) -> Dict[str, float]:
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    p16 = (torch.randn(n, device=dev, generator=g) * 1e-3).to(dtype)
    p32 = torch.randn(n, device=dev, generator=g) * 0.02
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    hyper = K.AdamHyper(lr=1e-4)
    state = K.StepState(dev)
    state.sumsq().fill_(1.0)
    K.adam_prepare(state, hyper)
    partials = torch.empty(K.sumsq_partials(), device=dev)
    src16 = (torch.randn(n, device=dev, generator=g)).to(dtype)
    src32 = torch.randn(n, device=dev, generator=g)
    out = {}
    ms = time_launch(lambda: K.adam_chunks([(p16, p32, m, v, n)], hyper, state), iters)
    out["adam"] = ms
    out["sumsq"] = time_launch(lambda: K.grad_sumsq([(p16, n)], partials), iters)
    out["pack"] = time_launch(lambda: K.pack([(p16, 0, src16, n)]), iters)
    out["accumulate"] = time_launch(lambda: K.pack([(p16, 0, src16, n)], accumulate=True), iters)
    out["cast_pack"] = time_launch(lambda: K.cast_pack([(p16, 0, src32, n)]), iters)
    out["master_init"] = time_launch(lambda: K.master_init(p32, m, v, p16, n), iters)
    return out


def run(sizes_log2: List[int], iters: int) -> List[dict]:
    peak = measured_peak_gbs()
    rows = []
    for lg in sizes_log2:
        n = 1 << lg
        times = bench_size(n, iters)
        for name, ms in times.items():
            gbs = BYTES_PER_ELEM[name] * n / (ms * 1e-3) / 1e9
            rows.append({"kernel": name, "n": n, "ms": round(ms, 5), "gbs": round(gbs, 1),
                         "frac_of_measured_peak": round(gbs / peak, 4)})
        torch.cuda.empty_cache()
    return rows


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20,22,24,26,28,30")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--adam-variants", default="",
                    help="comma list of cs_adam_variant ids: time K1 for each")
    args = ap.parse_args()
    if args.adam_variants:
        from . import _native as N
        peak = measured_peak_gbs()
        for v in [int(x) for x in args.adam_variants.split(",")]:
            N.load().cs_adam_variant(v)
            for lg in [int(s) for s in args.sizes.split(",")]:
                n = 1 << lg
                ms = bench_size(n, args.iters)["adam"]
                gbs = 28 * n / (ms * 1e-3) / 1e9
                print(json.dumps({"kernel": "adam", "variant": v, "n": n, "ms": round(ms, 5),
                                  "gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak, 4)}))
        return
    rows = run([int(s) for s in args.sizes.split(",")], args.iters)
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
