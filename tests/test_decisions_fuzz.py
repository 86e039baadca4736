"""Decision parity on 80 seeded random configurations (model shape, chunk
capacity, world size / rank, budgets from roomy to infeasible, eviction
strategy, soft limit, optimizer-state placement, checkpointing) against the
REFERENCE's frozen decisions (tests/golden/gen_decision_fuzz.py): layout,
plan, every ledger row, samples, final FSM states and copies — and the same
rejection where the reference rejects a configuration."""

import gzip
import json
import os

import pytest

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
from paper_2108_05818_b200.memory import EvictionStrategy
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.scenario import Simulator
from test_decisions_golden import _digest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decisions_fuzz.json.gz")
with gzip.open(GOLDEN, "rt") as _f:
    CASES = json.load(_f)["cases"]
PARAMS = [(name, rank) for name, case in CASES.items() for rank in case["ranks"]]


@pytest.mark.parametrize("name,rank", PARAMS)
def test_random_config_matches_reference(name, rank):
    case = CASES[name]
    ref = case["ranks"][rank]
    pkw = dict(case["policy"], eviction=EvictionStrategy(case["policy"]["eviction"]))
    try:
        sim = Simulator(build_gpt_schema(**case["schema"]), HardwareSpec(**case["hardware"]),
                        PolicySpec(**pkw), nproc=case["nproc"], rank=int(rank))
        result = sim.run(case["iterations"])
    except Exception as e:
        assert ref.get("error") == type(e).__name__, (name, rank, repr(e))
        return
    assert "error" not in ref, (name, rank, ref)
    mine = json.loads(json.dumps(_digest(sim, result.reports, result.plan)))
    assert mine["layout"] == ref["layout"]
    assert mine["plan"] == ref["plan"]
    assert len(mine["iterations"]) == len(ref["iterations"])
    for a, b in zip(mine["iterations"], ref["iterations"]):
        for key in b:
            assert a[key] == b[key], (name, rank, b["iteration"], key)
    assert mine["final_states"] == ref["final_states"]
    assert mine["final_copies"] == ref["final_copies"]


def test_fuzz_covers_feasible_and_infeasible_runs():
    feas = [all(it["feasible"] for it in r["iterations"])
            for c in CASES.values() for r in c["ranks"].values() if "error" not in r]
    assert sum(feas) >= 50 and len(feas) - sum(feas) >= 10, (sum(feas), len(feas))
