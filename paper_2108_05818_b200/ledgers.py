"""Ledger wire formats: the parity artefacts between the oracle and real runs.

Column schemas and ordering follow the reference's report writers
(`/root/reference/pkg/src/chunkstar/reports.py:170-232`, schema version 1):

    layout.csv                tensor_id,kind,chunk_id,offset_elems,numel
    moments_<strategy>.csv    iteration,moment,device,used_bytes,chunk_bytes,non_model_bytes
    transfers_<strategy>.csv  iteration,moment,chunk_id,src,dst,bytes,reason
    collectives_<strategy>.csv iteration,group_id,kind,bytes,includes_padding(0/1)

and the per-run chunk block of ``summary.json`` (plan + per-iteration
totals, sorted keys, 2-space indent).  Files are deterministic (no time or
host data), so a real B200 run and the reference simulator on the same
config can be diffed byte for byte.  The writers take any sequence of
``IterationReport`` — from ``Simulator.run`` or from ``ChunkTrainer.reports``.
"""

import csv
import io
import json
import os
from typing import Dict, IO, Iterable, List, Optional, Sequence, Tuple

from .engine import IterationReport
from .profiler import PlacementPlan

SCHEMA_VERSION = 1

_COLUMNS = {
    "layout": ("tensor_id", "kind", "chunk_id", "offset_elems", "numel"),
    "moments": ("iteration", "moment", "device", "used_bytes", "chunk_bytes",
                "non_model_bytes"),
    "transfers": ("iteration", "moment", "chunk_id", "src", "dst", "bytes", "reason"),
    "collectives": ("iteration", "group_id", "kind", "bytes", "includes_padding"),
}


def _rows(kind: str, reports: Sequence[IterationReport]) -> Iterable[list]:
    for r in reports:
        if kind == "moments":
            for s in r.samples:
                yield [r.iteration, s.moment, s.device, s.used_bytes, s.chunk_bytes,
                       s.non_model_bytes]
        elif kind == "transfers":
            for t in r.transfers:
                yield [r.iteration, t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason]
        elif kind == "collectives":
            for c in r.collectives:
                yield [c.iteration, c.group_id, c.kind, c.bytes, int(c.includes_padding)]


def _csv_text(header: Sequence[str], rows: Iterable[Sequence]) -> str:
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(header)
    for row in rows:
        w.writerow(list(row))
    return buf.getvalue()


def ledger_csv(kind: str, reports: Sequence[IterationReport]) -> str:
    """``kind`` in moments / transfers / collectives."""
    return _csv_text(_COLUMNS[kind], _rows(kind, reports))


def layout_csv(layout_rows: Sequence[Tuple[int, str, int, int, int]]) -> str:
    return _csv_text(_COLUMNS["layout"], layout_rows)


def plan_block(plan: Optional[PlacementPlan]) -> Optional[Dict]:
    if plan is None:
        return None
    return {"gpu_margin_bytes": plan.gpu_margin_bytes,
            "peak_non_model_bytes": plan.peak_non_model_bytes,
            "working_set_bytes": plan.working_set_bytes,
            "os_positions_on_gpu": list(plan.os_positions_on_gpu),
            "os_chunks_on_gpu": plan.os_chunks_on_gpu,
            "embedding_device": plan.embedding_device}


def iteration_block(r: IterationReport) -> Dict:
    return {"iteration": r.iteration, "warmup": r.warmup, "feasible": r.feasible,
            "failure_reason": r.failure_reason, "failure_moment": r.failure_moment,
            "cpu_to_gpu_bytes": r.cpu_to_gpu_bytes, "gpu_to_cpu_bytes": r.gpu_to_cpu_bytes,
            "collective_bytes": r.intra_gpu_collective_bytes,
            "peak_gpu_bytes": r.peak_gpu_bytes, "peak_cpu_bytes": r.peak_cpu_bytes}


def chunk_summary(reports: Sequence[IterationReport], plan: Optional[PlacementPlan]) -> Dict:
    return {"plan": plan_block(plan), "iterations": [iteration_block(r) for r in reports]}


def render_json(payload: Dict) -> str:
    return json.dumps(payload, sort_keys=True, indent=2) + "\n"


def write_ledgers(out_dir: str, reports: Sequence[IterationReport], layout_rows,
                  plan: Optional[PlacementPlan] = None, strategy: str = "chunk",
                  extra_summary: Optional[Dict] = None) -> List[str]:
    """Write layout / moments / transfers / collectives CSVs and a summary."""
    os.makedirs(out_dir, exist_ok=True)
    files = {"layout.csv": layout_csv(layout_rows)}
    for kind in ("moments", "transfers", "collectives"):
        files["%s_%s.csv" % (kind, strategy)] = ledger_csv(kind, reports)
    summary = {"schema_version": SCHEMA_VERSION, "kind": "run",
               "outcomes": {strategy: chunk_summary(reports, plan)}}
    if extra_summary:
        summary.update(extra_summary)
    files["summary.json"] = render_json(summary)
    paths = []
    for name, text in files.items():
        path = os.path.join(out_dir, name)
        with open(path, "w", encoding="utf-8", newline="") as fh:
            fh.write(text)
        paths.append(path)
    return paths


class TraceWriter:
    """JSON-lines moment trace; pass ``.emit`` as the engine's ``trace_fn``."""

    def __init__(self, handle: IO[str]):
        self._handle = handle

    def emit(self, record: Dict) -> None:
        self._handle.write(json.dumps(record, sort_keys=True) + "\n")
