"""Decision parity: this build's engine vs the REFERENCE's frozen ledgers.

tests/golden/decisions.json.gz was produced by importing the unmodified
reference (tests/golden/gen_decision_golden.py).  Layout rows, placement
plan, every transfer-ledger row (moment, chunk, src, dst, bytes, reason),
every collective row, the per-moment samples and the final FSM states /
copies must be identical for every rank of every case.
"""

import gzip
import json
import os

import pytest

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.scenario import Simulator

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decisions.json.gz")

with gzip.open(GOLDEN, "rt") as _f:
    CASES = json.load(_f)["cases"]

PARAMS = [(name, rank) for name, case in CASES.items() for rank in case["ranks"]]


def _digest(sim, reports, plan):
    def samples(r):
        return [[s.moment, s.device, s.used_bytes, s.chunk_bytes, s.non_model_bytes]
                for s in r.samples]
    return {
        "layout": [list(row) for row in sim.chunk_set.layout_rows()],
        "plan": None if plan is None else {
            "gpu_margin_bytes": plan.gpu_margin_bytes,
            "peak_non_model_bytes": plan.peak_non_model_bytes,
            "working_set_bytes": plan.working_set_bytes,
            "os_positions_on_gpu": list(plan.os_positions_on_gpu),
            "embedding_device": plan.embedding_device},
        "iterations": [{
            "iteration": r.iteration, "warmup": r.warmup, "feasible": r.feasible,
            "failure_reason": r.failure_reason, "failure_moment": r.failure_moment,
            "transfers": [[t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason]
                          for t in r.transfers],
            "collectives": [[c.iteration, c.group_id, c.kind, c.bytes, c.includes_padding]
                            for c in r.collectives],
            "cpu_to_gpu_bytes": r.cpu_to_gpu_bytes, "gpu_to_cpu_bytes": r.gpu_to_cpu_bytes,
            "intra_gpu_collective_bytes": r.intra_gpu_collective_bytes,
            "peak_gpu_bytes": r.peak_gpu_bytes, "peak_cpu_bytes": r.peak_cpu_bytes,
            "samples": samples(r) if len(r.samples) <= 2000 else None,
        } for r in reports],
        "final_states": {str(c.chunk_id): [t.state.value for t in c.tensors]
                         for c in sim.chunk_set.chunks.values()},
        "final_copies": {str(c.chunk_id): list(c.copies)
                         for c in sim.chunk_set.chunks.values()},
    }


@pytest.mark.parametrize("name,rank", PARAMS)
def test_engine_matches_reference_ledgers(name, rank):
    case = CASES[name]
    schema = build_gpt_schema(**case["schema"])
    sim = Simulator(schema, HardwareSpec(**case["hardware"]), PolicySpec(**case["policy"]),
                    nproc=case["nproc"], rank=int(rank))
    result = sim.run(case["iterations"])
    mine = json.loads(json.dumps(_digest(sim, result.reports, result.plan)))
    ref = case["ranks"][rank]
    assert mine["layout"] == ref["layout"]
    assert mine["plan"] == ref["plan"]
    assert len(mine["iterations"]) == len(ref["iterations"])
    for it_mine, it_ref in zip(mine["iterations"], ref["iterations"]):
        for key in it_ref:
            assert it_mine[key] == it_ref[key], (name, rank, it_ref["iteration"], key)
    assert mine["final_states"] == ref["final_states"]
    assert mine["final_copies"] == ref["final_copies"]


def test_collective_order_is_rank_invariant():
    """Every rank issues the same (group, kind) sequence: a 1:1 NCCL mapping
    cannot deadlock."""
    for name, case in CASES.items():
        seqs = {tuple((c[1], c[2]) for it in r["iterations"] for c in it["collectives"])
                for r in case["ranks"].values()}
        assert len(seqs) == 1, name
