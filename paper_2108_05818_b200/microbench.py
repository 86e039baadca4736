"""C5 microbench (BASELINE.json configs[4]): chunk kernels K1-K6 at
1M-1G elements, HBM GB/s vs roofline, beside CPU Adam arms.

Algorithmic bytes per element: K1 Adam 28, K2 sumsq 2,
K3 pack 4, K4 accumulate 6, K5 cast+pack 6, K6 state birth 14 (fp16 src).

GPU arm: every timed launch is preceded by an L2 flush (a read of a
buffer twice the 126 MB L2: cold and clean), and bracketed by CUDA events on its stream;
the flush's ~0.1 ms of device work hides the host launch, so the events
see the kernel alone, cold.  Sizes below ~4M elements are latency-bound
(a few microseconds of launch ramp against < 10 us of traffic) and are
labelled so; the roofline fraction is meaningful from 16M elements up.

CPU arms (SURVEY §8d CPU baseline items 2-3), same element counts, same
algorithmic bytes per element, host DRAM:

* ``cpu_torch_fused``: torch-CPU fused Adam (``torch.optim.Adam(fused=True)``
  over the fp32 master) with the chunk path's casts — fp16 gradients widened
  to fp32 before, the fp16 parameter copy narrowed after;
* ``cpu_host_k1``: this build's own host K1 (``cs_adam_chunks_host``, AVX2 +
  OpenMP), the kernel that runs CPU-placed optimizer triplets;
* ``cpu_torch``: torch-CPU restatements of K2-K6 (fp32 sum of squares in
  double, fp16 copy, widen-add-narrow accumulate, fp32 -> fp16 cast, state
  birth).

Thread counts are reported with every CPU row.

    python -m paper_2108_05818_b200.microbench [--sizes 20,22,...] [--iters N] [--cpu]
"""

import argparse
import json
import os
import time
from typing import Callable, Dict, List, Optional

import torch

from . import kernels as K

BYTES_PER_ELEM = {"adam": 28, "sumsq": 2, "pack": 4, "accumulate": 6, "cast_pack": 6,
                  "master_init": 14}
L2_BYTES = 126 << 20
#: below this many algorithmic bytes per call, a fixed ~7-15 us of launch and
#: event cost (one launch for K1/K3-K6, three for the canonical K2) is >= 5 %
#: of the time at the HBM peak: such rows are reported as latency-bound
LATENCY_BOUND_BELOW_BYTES = 256 << 20


def measured_peak_gbs() -> float:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


class L2Flush:
    """Reads a buffer of 2 x L2 so the next launch starts cold AND clean: the
    previous launch's dirty lines are written back during the flush, and L2
    is left holding clean lines (a write flush would leave 126 MB of dirty
    lines whose write-back the next, timed launch would pay: at 2^20 elements
    that is several times the kernel's own traffic)."""

    def __init__(self, device="cuda"):
        self.buf = torch.ones(2 * L2_BYTES // 4, dtype=torch.float32, device=device)
        self.out = torch.empty((), dtype=torch.float32, device=device)

    def __call__(self) -> None:
        torch.sum(self.buf, dim=0, out=self.out)


def time_launch(fn: Callable[[], None], iters: int, flush: Optional[L2Flush],
                warmup: int = 2) -> float:
    """Average DEVICE milliseconds per cold call (see the module doc)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    pairs = []
    for _ in range(iters):
        if flush is not None:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        pairs.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in pairs) / iters


def bench_size(n: int, iters: int, dtype=torch.float16, flush: Optional[L2Flush] = None,
               kernels=tuple(BYTES_PER_ELEM)) -> Dict[str, float]:
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
    scratch = torch.empty(K.sumsq_scratch([(p16, n)]), device=dev)
    item_sums = torch.empty(1, dtype=torch.float64, device=dev)
    fns = {"adam": lambda: K.adam_chunks([(p16, p32, m, v, n)], hyper, state),
           "sumsq": lambda: K.grad_sumsq([(p16, n)], scratch, item_sums)}
    if any(k in kernels for k in ("pack", "accumulate", "cast_pack", "master_init")):
        src16 = (torch.randn(n, device=dev, generator=g)).to(dtype)
        src32 = torch.randn(n, device=dev, generator=g)
        fns.update({"pack": lambda: K.pack([(p16, 0, src16, n)]),
                    "accumulate": lambda: K.pack([(p16, 0, src16, n)], accumulate=True),
                    "cast_pack": lambda: K.cast_pack([(p16, 0, src32, n)]),
                    "master_init": lambda: K.master_init(p32, m, v, p16, n)})
    return {k: time_launch(fns[k], iters, flush) for k in kernels}


def run(sizes_log2: List[int], iters: int, kernels=tuple(BYTES_PER_ELEM)) -> List[dict]:
    peak = measured_peak_gbs()
    flush = L2Flush()
    rows = []
    for lg in sizes_log2:
        n = 1 << lg
        times = bench_size(n, iters, flush=flush, kernels=kernels)
        for name, ms in times.items():
            gbs = BYTES_PER_ELEM[name] * n / (ms * 1e-3) / 1e9
            rows.append({"arm": "gpu", "kernel": name, "n": n, "ms": round(ms, 5),
                         "gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak, 4),
                         "regime": ("latency-bound" if BYTES_PER_ELEM[name] * n < LATENCY_BOUND_BELOW_BYTES
                                    else "hbm"),
                         "l2": "read-flushed before every launch (cold, clean)"})
        torch.cuda.empty_cache()
    return rows


# ---- CPU arms ------------------------------------------------------------------------


def _cpu_inputs(n: int):
    g = torch.Generator().manual_seed(0)
    g16 = (torch.randn(n, generator=g) * 1e-3).half()
    p32 = torch.randn(n, generator=g) * 0.02
    m = torch.randn(n, generator=g) * 1e-4
    v = torch.rand(n, generator=g) * 1e-7
    return g16, p32, m, v


def cpu_torch_fused_adam(n: int, iters: int = 2) -> dict:
    """torch-CPU fused Adam with the chunk path's casts, all host threads."""
    g16, p32, m, v = _cpu_inputs(n)
    p = torch.nn.Parameter(p32)
    opt = torch.optim.Adam([p], lr=1e-4, betas=(0.9, 0.999), eps=1e-8, fused=True)
    p16 = torch.empty(n, dtype=torch.float16)
    times = []
    for k in range(iters + 1):
        t0 = time.perf_counter()
        p.grad = g16.float()          # fp16 grad chunk widened on the fly
        opt.step()
        p16.copy_(p.detach())         # fp32 master narrowed into the fp16 chunk
        if k:
            times.append(time.perf_counter() - t0)
    s = min(times)
    return {"arm": "cpu_torch_fused", "kernel": "adam", "n": n, "ms": round(s * 1e3, 3),
            "gbs": round(28 * n / s / 1e9, 2), "gelem_per_s": round(n / s / 1e9, 4),
            "threads": torch.get_num_threads()}


def cpu_host_k1(n: int, iters: int = 2, threads: int = 0) -> dict:
    """This build's host K1 (AVX2/F16C + OpenMP) over pinned host buffers."""
    from . import _native as N
    g16, p32, m, v = _cpu_inputs(n)
    if torch.cuda.is_available():  # the buffers CPU-placed triplets live in
        g16, p32, m, v = (t.pin_memory() for t in (g16, p32, m, v))
    st = N.CsStepState()
    st.grad_scale, st.step_size, st.sqrt_bc2, st.skip = 1.0, 1e-4, 0.03, 0
    hyper = K.AdamHyper(lr=1e-4)
    times = []
    for k in range(iters + 1):
        t0 = time.perf_counter()
        K.adam_chunks_host([(g16, p32, m, v, n)], hyper, st, threads)
        if k:
            times.append(time.perf_counter() - t0)
    s = min(times)
    return {"arm": "cpu_host_k1", "kernel": "adam", "n": n, "ms": round(s * 1e3, 3),
            "gbs": round(28 * n / s / 1e9, 2), "gelem_per_s": round(n / s / 1e9, 4),
            "threads": int(N.load().cs_host_threads(threads))}


def cpu_torch_chunk_ops(n: int, iters: int = 2) -> List[dict]:
    """torch-CPU restatements of K2-K6 on host buffers, all threads (SURVEY
    §8d CPU baseline item 3: the cast and copy of pack / cast)."""
    g = torch.Generator().manual_seed(0)
    src16 = (torch.randn(n, generator=g)).half()
    src32 = torch.randn(n, generator=g)
    dst16 = torch.zeros(n, dtype=torch.float16)
    p32, m, v = torch.empty(n), torch.empty(n), torch.empty(n)
    ops = {
        "sumsq": lambda: src16.float().square().sum(dtype=torch.float64),
        "pack": lambda: dst16.copy_(src16),
        "accumulate": lambda: dst16.copy_(dst16.float().add_(src16.float())),
        "cast_pack": lambda: dst16.copy_(src32),
        "master_init": lambda: (p32.copy_(src16), m.zero_(), v.zero_()),
    }
    rows = []
    for name, fn in ops.items():
        times = []
        for k in range(iters + 1):
            t0 = time.perf_counter()
            fn()
            if k:
                times.append(time.perf_counter() - t0)
        s = min(times)
        rows.append({"arm": "cpu_torch", "kernel": name, "n": n, "ms": round(s * 1e3, 3),
                     "gbs": round(BYTES_PER_ELEM[name] * n / s / 1e9, 2),
                     "threads": torch.get_num_threads()})
    return rows


def run_cpu(sizes_log2: List[int]) -> List[dict]:
    rows = []
    for lg in sizes_log2:
        n = 1 << lg
        it = 1 if n >= (1 << 29) else 2
        rows.append(cpu_torch_fused_adam(n, it))
        rows.append(cpu_host_k1(n, it))
        rows.extend(cpu_torch_chunk_ops(n, it))
    return rows


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20,22,24,26,28,30")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--cpu", action="store_true", help="also run the CPU Adam arms")
    ap.add_argument("--kernels", default=",".join(BYTES_PER_ELEM))
    args = ap.parse_args()
    sizes = [int(s) for s in args.sizes.split(",")]
    for r in run(sizes, args.iters, tuple(args.kernels.split(","))):
        print(json.dumps(r), flush=True)
    if args.cpu:
        for r in run_cpu(sizes):
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
