"""Host-DRAM ceilings the host Adam is measured against (one JSON line each).

* torch copy of 1 GiB fp32 (read + write streams), all threads;
* in-place read-modify-write of four fp32 streams (the host Adam's access
  pattern without its arithmetic: 16 B read + 16 B written per element);
* the host Adam itself (cs_adam_chunks_host, 28 B per element) at 4, 8, 12
  and 16 threads.

    python scripts/host_bw.py
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2108_05818_b200 import _native as N  # noqa: E402
from paper_2108_05818_b200 import kernels as K  # noqa: E402


def timed(fn, reps=5):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps


def main():
    n = 1 << 28
    torch.set_num_threads(os.cpu_count())
    a = torch.empty(n).normal_()
    b = torch.empty_like(a)
    dt = timed(lambda: b.copy_(a))
    print(json.dumps({"case": "torch copy fp32 1 GiB", "threads": torch.get_num_threads(),
                      "gbs": round(2 * n * 4 / dt / 1e9, 1)}), flush=True)
    m = 1 << 26
    bufs = [torch.ones(m) for _ in range(4)]
    dt = timed(lambda: [x.mul_(1.0000001) for x in bufs])
    print(json.dumps({"case": "in-place RMW, four fp32 streams of 64 Mi (sequential)",
                      "threads": torch.get_num_threads(),
                      "gbs": round(4 * m * 8 / dt / 1e9, 1)}), flush=True)
    items = [(torch.empty(m, dtype=torch.float16).fill_(1e-3), torch.full((m,), 0.02),
              torch.zeros(m), torch.zeros(m), m) for _ in range(4)]
    prev = N.CsStepState(beta1_pow=1.0, beta2_pow=1.0, step=0, loss_scale=1.0)
    st = K.speculate_step_scalars(prev, K.AdamHyper(lr=1e-4))
    for th in (4, 8, 12, 16):
        dt = timed(lambda: K.adam_chunks_host(items, K.AdamHyper(lr=1e-4), st, th), reps=3)
        print(json.dumps({"case": "host Adam (cs_adam_chunks_host), 4 x 64 Mi", "threads": th,
                          "gelem_per_s": round(4 * m / dt / 1e9, 2),
                          "gbs": round(28 * 4 * m / dt / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
