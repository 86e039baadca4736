"""Host-link copies against host-DRAM traffic: why chunk moves beside the
host Adam run below the pinned-memcpy peak.

Times 128 MiB pinned<->HBM copies (the fp16 chunk of the 1B model) on a side
stream, one direction at a time and both at once, (a) with the host idle,
(b) while the host Adam (cs_adam_chunks_host, the executor's worker team)
streams four 64 Mi-element positions in a loop, (c) into destination buffers
the CPU has just written (dirty in its caches).  Prints one JSON line per case.

    python scripts/host_link_contention.py [--threads 12]
"""

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2108_05818_b200 import _native as N  # noqa: E402
from paper_2108_05818_b200 import kernels as K  # noqa: E402

N16 = 64 << 20          # elements of one chunk
REPS = 64


def timed_copies(pairs, stream):
    """Issue every (dst, src) copy on ``stream``; GB/s over the whole batch."""
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record()
        for d, s in pairs:
            d.copy_(s, non_blocking=True)
        b.record()
    return a, b, sum(d.numel() * d.element_size() for d, _ in pairs)


def run_case(name, dirs, host, dev, items, adam_threads, dirty=False):
    streams = {"h2d": torch.cuda.Stream(), "d2h": torch.cuda.Stream()}
    stop = threading.Event()
    started = threading.Event()
    rate = []

    def adam_loop():
        prev = N.CsStepState(beta1_pow=1.0, beta2_pow=1.0, step=0, loss_scale=1.0)
        st = K.speculate_step_scalars(prev, K.AdamHyper(lr=1e-4))
        n = 0
        t0 = time.perf_counter()
        while not stop.is_set():
            K.adam_chunks_host(items, K.AdamHyper(lr=1e-4), st, adam_threads)
            n += sum(it[4] for it in items)
            started.set()
        rate.append(n / (time.perf_counter() - t0) / 1e9)

    th = None
    if items:
        th = threading.Thread(target=adam_loop)
        th.start()
        started.wait()
    if dirty:
        for t in host:
            t.fill_(1.0)
    res = {}
    evs = []
    for d in dirs:
        pairs = ([(dev[i % len(dev)], host[i % len(host)]) for i in range(REPS)] if d == "h2d"
                 else [(host[i % len(host)], dev[i % len(dev)]) for i in range(REPS)])
        evs.append((d,) + timed_copies(pairs, streams[d]))
    torch.cuda.synchronize()
    for d, a, b, nb in evs:
        res[d] = round(nb / (a.elapsed_time(b) * 1e-3) / 1e9, 1)
    if th is not None:
        stop.set()
        th.join()
    out = {"case": name, "gbs": res, "host_adam_threads": adam_threads if items else 0}
    if rate:
        out["host_adam_gelem_per_s"] = round(rate[0], 2)
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0, help="host Adam team (0: the executor's)")
    args = ap.parse_args()
    ht = K.host_threads(0)
    team = args.threads or max(1, ht - max(2, ht // 4))
    host = [torch.empty(N16, dtype=torch.float16, pin_memory=True) for _ in range(4)]
    dev = [torch.empty(N16, dtype=torch.float16, device="cuda") for _ in range(4)]
    for t in host:
        t.zero_()
    items = [(torch.empty(N16, dtype=torch.float16).fill_(1e-3), torch.full((N16,), 0.02),
              torch.zeros(N16), torch.zeros(N16), N16) for _ in range(4)]
    for case, dirs in (("h2d", ["h2d"]), ("d2h", ["d2h"]), ("both", ["h2d", "d2h"])):
        run_case(case + "_idle", dirs, host, dev, None, team)
        run_case(case + "_dirty_dst", dirs, host, dev, None, team, dirty=True)
        run_case(case + "_host_adam", dirs, host, dev, items, team)
    print(json.dumps({"host_threads": ht, "worker_team": team}))


if __name__ == "__main__":
    main()
