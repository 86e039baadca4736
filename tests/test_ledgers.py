"""Ledger wire formats are byte-identical to the reference's writers
(fixtures from tests/golden/gen_ledger_golden.py)."""

import os

import pytest

from paper_2108_05818_b200 import ledgers
from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.scenario import Simulator

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ledgers")
MI = 1 << 20
CASES = {
    "tiny_tight": (dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                        context_bytes=2 * MI), dict(gpu_count=1, gpu_bytes=24 * MI),
                   dict(capacity_elems=MI // 4), 1),
    "tiny_p4_tight": (dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                           context_bytes=2 * MI), dict(gpu_count=4, gpu_bytes=20 * MI),
                      dict(capacity_elems=MI // 4), 4),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_ledger_files_byte_identical_to_reference_writers(name, tmp_path):
    skw, hkw, pkw, nproc = CASES[name]
    sim = Simulator(build_gpt_schema(**skw), HardwareSpec(**hkw), PolicySpec(**pkw), nproc)
    run = sim.run(3)
    ledgers.write_ledgers(str(tmp_path), run.reports, run.layout_rows, run.plan)
    for fname in ("layout.csv", "moments_chunk.csv", "transfers_chunk.csv",
                  "collectives_chunk.csv"):
        with open(os.path.join(GOLD, name, fname), "rb") as f:
            ref = f.read()
        with open(tmp_path / fname, "rb") as f:
            mine = f.read()
        assert mine == ref, fname
    block = ledgers.render_json(ledgers.chunk_summary(run.reports, run.plan))
    with open(os.path.join(GOLD, name, "chunk_block.json")) as f:
        assert block == f.read()
