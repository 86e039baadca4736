"""Freeze ledger CSV files written by the REFERENCE's own writers
(`chunkstar/reports.py`) for two configs, as byte-parity fixtures for
paper_2108_05818_b200.ledgers.  Run from the repo root:
    python tests/golden/gen_ledger_golden.py
"""

import importlib
import json
import os
import sys
import tempfile

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ledgers")
MI = 1 << 20
CASES = {
    "tiny_tight": (dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                        context_bytes=2 * MI), dict(gpu_count=1, gpu_bytes=24 * MI),
                   dict(capacity_elems=MI // 4), 1),
    "tiny_p4_tight": (dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                           context_bytes=2 * MI), dict(gpu_count=4, gpu_bytes=20 * MI),
                      dict(capacity_elems=MI // 4), 4),
}


def main():
    sys.path.insert(0, REF_SRC)
    cs = importlib.import_module("chunkstar")
    reports = importlib.import_module("chunkstar.reports")
    for name, (skw, hkw, pkw, nproc) in CASES.items():
        sim = cs.Simulator(cs.build_gpt_schema(**skw), cs.HardwareSpec(**hkw),
                           cs.PolicySpec(**pkw), nproc)
        run = sim.run(3)
        d = os.path.join(OUT, name)
        os.makedirs(d, exist_ok=True)
        reports.write_layout_csv(run, d)
        reports.write_moments_csv(run, d)
        reports.write_transfers_csv(run, d)
        reports.write_collectives_csv(run, d)
        chunk_block = {"plan": reports._plan_block(run),
                       "iterations": [reports._iteration_block(r) for r in run.reports]}
        with open(os.path.join(d, "chunk_block.json"), "w") as f:
            f.write(reports.render_json(chunk_block))
        print(name, sorted(os.listdir(d)))


if __name__ == "__main__":
    main()
