"""Freeze the REFERENCE's decisions on seeded random configurations.

Complements gen_decision_golden.py (13 hand-picked cases) with 80 random
ones: model shape, chunk capacity, world size and rank, GPU / host budgets
from roomy to infeasible, eviction strategy, soft-limit fraction, optimizer
state placement and activation checkpointing.  Each case runs the unmodified
reference (/root/reference, build container only) through its own wiring
(``run_rank`` of gen_decision_golden) and stores the same digest; a case the
reference rejects stores the exception's class name instead.

Run from the repo root:  python tests/golden/gen_decision_fuzz.py
"""

import gzip
import importlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from gen_decision_golden import REF_SRC, digest, run_rank  # noqa: E402

OUT = os.path.join(HERE, "decisions_fuzz.json.gz")
N_CASES = 80
MI = 1 << 20


def random_case(seed):
    r = random.Random(1000 + seed)
    H = r.choice([64, 128, 192, 256])
    skw = dict(layers=r.randint(1, 6), hidden_dim=H, heads=4, seq_len=r.choice([32, 64, 128]),
               batch=r.randint(1, 8), vocab=r.choice([128, 1000, 50304]),
               context_bytes=r.choice([0, 1 * MI, 2 * MI, 4 * MI]))
    cap = r.choice([2, 3, 4, 6, 8, 16]) * H * H
    nproc = r.choice([1, 1, 2, 3, 4, 8])
    ranks = list(range(nproc)) if nproc <= 4 else [0, r.randrange(1, nproc), nproc - 1]
    gpu_bytes = int(r.choice([0.5, 1, 2, 4, 8, 16, 64, 10 ** 4]) * MI * r.uniform(1, 4))
    hkw = dict(gpu_count=nproc, gpu_bytes=gpu_bytes)
    if r.random() < 0.3:
        hkw["cpu_bytes"] = int(r.choice([8, 32, 256]) * MI * nproc)
    pkw = dict(capacity_elems=cap, checkpointing=r.random() < 0.3,
               os_placement=r.choice(["auto", "auto", "cpu", "gpu"]),
               eviction=r.choice(["latest_next_use", "list_order"]),
               limit_fraction=r.choice([0.8, 0.8, 0.6, 1.0]))
    return skw, hkw, pkw, nproc, ranks, 3


def main() -> None:
    sys.path.insert(0, REF_SRC)
    cs = importlib.import_module("chunkstar")
    for mod in ("model", "config", "scenario", "chunks", "parallel", "memory", "engine",
                "profiler"):
        importlib.import_module("chunkstar." + mod)
    assert cs.__file__.startswith(REF_SRC), cs.__file__
    out = {"reference": REF_SRC, "cases": {}}
    n_feasible = n_error = 0
    for seed in range(N_CASES):
        skw, hkw, pkw, nproc, ranks, iters = random_case(seed)
        pkw_ref = dict(pkw, eviction=cs.memory.EvictionStrategy(pkw["eviction"]))
        entry = {"schema": skw, "hardware": hkw, "policy": pkw, "nproc": nproc,
                 "iterations": iters, "ranks": {}}
        for rank in ranks:
            try:
                sim, reports, plan = run_rank(cs, "fuzz%d" % seed, skw, hkw, pkw_ref, nproc,
                                              rank, iters)
                entry["ranks"][str(rank)] = digest(sim, reports, plan)
                n_feasible += all(it["feasible"] for it in
                                  entry["ranks"][str(rank)]["iterations"])
            except Exception as e:  # the reference rejects the configuration
                entry["ranks"][str(rank)] = {"error": type(e).__name__}
                n_error += 1
        out["cases"]["fuzz%02d" % seed] = entry
    with gzip.open(OUT, "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", n_feasible, "feasible rank runs,",
          n_error, "rejected")


if __name__ == "__main__":
    main()
