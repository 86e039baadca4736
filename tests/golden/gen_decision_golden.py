"""Freeze the REFERENCE's decisions (layout, transfer and collective ledgers,
placement plan, FSM end states) as golden fixtures.

Imports the unmodified reference from /root/reference/pkg/src (available in
the build container only; the fixtures travel, the reference does not) and
runs its own Simulator wiring (`scenario.py:105-182`) — for ranks other than
0 the same wiring is assembled by hand from the reference's classes, as its
test fixture does (`tests/conftest.py:27-70`), because `Simulator`
hard-codes rank 0.

Run from the repo root:  python tests/golden/gen_decision_golden.py
"""

import gzip
import json
import os
import sys

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "decisions.json.gz")

# (name, schema kwargs, hardware kwargs, policy kwargs, nproc, ranks, iterations)
MI = 1 << 20
CASES = [
    # C1 tiny GPT, p=1: all-resident and two chunk sizes
    ("tiny_cap1Mi", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4),
     dict(gpu_count=1, gpu_bytes=180 * 10**9), dict(capacity_elems=MI), 1, [0], 3),
    ("tiny_cap256Ki", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4),
     dict(gpu_count=1, gpu_bytes=180 * 10**9), dict(capacity_elems=MI // 4), 1, [0], 3),
    # tight GPU budget: eviction + partial OS placement on the host
    ("tiny_tight", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                        context_bytes=2 * MI),
     dict(gpu_count=1, gpu_bytes=24 * MI), dict(capacity_elems=MI // 4), 1, [0], 4),
    ("tiny_os_cpu", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                         context_bytes=2 * MI),
     dict(gpu_count=1, gpu_bytes=64 * MI), dict(capacity_elems=MI // 4, os_placement="cpu"),
     1, [0], 3),
    # ZeRO chunk groups, every rank (tail group padded at p=4 and p=8)
    ("tiny_p2", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4),
     dict(gpu_count=2, gpu_bytes=180 * 10**9), dict(capacity_elems=MI // 4), 2, [0, 1], 3),
    ("tiny_p4_tight", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                           context_bytes=2 * MI),
     dict(gpu_count=4, gpu_bytes=20 * MI), dict(capacity_elems=MI // 4), 4, [0, 1, 2, 3], 3),
    ("tiny_p8", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4),
     dict(gpu_count=8, gpu_bytes=180 * 10**9), dict(capacity_elems=MI // 4), 8,
     list(range(8)), 3),
    ("tiny_p2_ckpt", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4),
     dict(gpu_count=2, gpu_bytes=180 * 10**9),
     dict(capacity_elems=MI // 4, checkpointing=True), 2, [0, 1], 3),
    # activation checkpointing on one rank under a tight budget (RE_FWD events)
    ("tiny_ckpt_tight", dict(layers=4, hidden_dim=256, heads=4, seq_len=128, batch=4,
                             context_bytes=2 * MI),
     dict(gpu_count=1, gpu_bytes=14 * MI), dict(capacity_elems=MI // 4, checkpointing=True),
     1, [0], 3),
    # C2 1B on one B200, chunk-size sweep
    ("gpt1b_cap32Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=16),
     dict(gpu_count=1, gpu_bytes=180 * 10**9), dict(capacity_elems=32 * MI), 1, [0], 3),
    ("gpt1b_cap64Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=16),
     dict(gpu_count=1, gpu_bytes=180 * 10**9), dict(capacity_elems=64 * MI), 1, [0], 3),
    ("gpt1b_cap256Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=16),
     dict(gpu_count=1, gpu_bytes=180 * 10**9), dict(capacity_elems=256 * MI), 1, [0], 3),
    # C2 at the configuration bench.py measures: per-GPU batch 32, where the
    # plan computes the embedding on the GPU (`profiler.py:70-74`), chunk-size
    # sweep; 160 GB is the accounting budget the GPU test runs the real step at
    ("gpt1b_b32_cap32Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=32),
     dict(gpu_count=1, gpu_bytes=160 * 10**9), dict(capacity_elems=32 * MI), 1, [0], 3),
    ("gpt1b_b32_cap64Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=32),
     dict(gpu_count=1, gpu_bytes=160 * 10**9), dict(capacity_elems=64 * MI), 1, [0], 3),
    ("gpt1b_b32_cap128Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=32),
     dict(gpu_count=1, gpu_bytes=160 * 10**9), dict(capacity_elems=128 * MI), 1, [0], 3),
    ("gpt1b_b32_cap256Mi", dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, batch=32),
     dict(gpu_count=1, gpu_bytes=160 * 10**9), dict(capacity_elems=256 * MI), 1, [0], 3),
    # the C3 model on one GPU (scripts/configs_sweep.py "4b_gpu")
    ("gpt4b_p1", dict(layers=64, hidden_dim=2304, heads=16, seq_len=1024, batch=8),
     dict(gpu_count=1, gpu_bytes=160 * 10**9), dict(capacity_elems=64 * MI), 1, [0], 3),
    # the C4 model on one GPU (configs_sweep "12b_mixed" / "12b_ckpt"): without
    # checkpointing the plan splits the optimizer triplets between HBM and host
    # DRAM and the fp16 chunks are evicted and refetched every iteration
    ("gpt12b_p1_mixed", dict(layers=60, hidden_dim=4096, heads=32, seq_len=1024, batch=8),
     dict(gpu_count=1, gpu_bytes=160 * 10**9, cpu_bytes=1500 * 10**9),
     dict(capacity_elems=64 * MI), 1, [0], 3),
    ("gpt12b_p1_ckpt", dict(layers=60, hidden_dim=4096, heads=32, seq_len=1024, batch=8),
     dict(gpu_count=1, gpu_bytes=160 * 10**9, cpu_bytes=1500 * 10**9),
     dict(capacity_elems=64 * MI, checkpointing=True), 1, [0], 3),
    # C3 4B ZeRO at p=8 (ranks 0 and 7)
    ("gpt4b_p8", dict(layers=64, hidden_dim=2304, heads=16, seq_len=1024, batch=8),
     dict(gpu_count=8, gpu_bytes=180 * 10**9), dict(capacity_elems=64 * MI), 8, [0, 7], 3),
    # C4 12B at p=8 with optimizer state in pinned host DRAM
    ("gpt12b_p8_os_cpu", dict(layers=60, hidden_dim=4096, heads=32, seq_len=1024, batch=8),
     dict(gpu_count=8, gpu_bytes=180 * 10**9, cpu_bytes=2000 * 10**9),
     dict(capacity_elems=64 * MI, os_placement="cpu"), 8, [0], 3),
]


def run_rank(cs, name, skw, hkw, pkw, nproc, rank, iterations):
    """The reference Simulator's wiring for one rank."""
    schema = cs.model.build_gpt_schema(**skw)
    hw = cs.config.HardwareSpec(**hkw)
    policy = cs.config.PolicySpec(**pkw)
    if rank == 0:
        sim = cs.scenario.Simulator(schema, hw, policy, nproc)
        result = sim.run(iterations)
        return sim, result.reports, result.plan
    timeline = cs.model.build_event_timeline(schema, checkpointing=policy.checkpointing)
    chunk_set = cs.chunks.build_model_chunk_lists(schema, capacity_elems=policy.capacity_elems)
    partition = cs.parallel.partition_chunks(chunk_set, nproc)
    local = partition.local_positions(rank)
    chunk_set.init_on_cpu(local, kinds=(cs.chunks.ChunkKind.PARAM_FP16,))
    pools = {cs.model.GPU: cs.memory.DevicePool(cs.model.GPU, hw.gpu_bytes),
             cs.model.CPU: cs.memory.DevicePool(cs.model.CPU, hw.cpu_bytes // nproc)}
    manager = cs.memory.MemoryManager(pools, policy.eviction)
    manager.register_chunks(chunk_set.chunks.values())
    manager.add_extra_model_bytes(cs.model.CPU, chunk_set.embedding.fp16_bytes)
    dp = cs.parallel.DpRuntime(chunk_set, partition, manager, rank=rank)
    engine = cs.engine.Engine(chunk_set, timeline, manager, schema=schema, dp=dp,
                              limit_fraction=policy.limit_fraction)
    engine.embedding_device = cs.profiler.embedding_compute_device(schema)
    gpu_cap = pools[cs.model.GPU].capacity_bytes

    def build(stats):
        return cs.profiler.compute_placement_plan(stats, chunk_set, gpu_cap, schema,
                                                  local_positions=local,
                                                  os_placement=policy.os_placement)

    class _S:
        pass
    s = _S()
    s.chunk_set, s.engine, s.dp, s.partition = chunk_set, engine, dp, partition
    # Simulator.run's own first check (`scenario.py:141-147, 163-168`): a host
    # too small for its shard of the layout is infeasible at moment 0
    cpu_pool = pools[cs.model.CPU]
    if cpu_pool.used_bytes > cpu_pool.capacity_bytes:
        return s, [cs.engine.IterationReport(iteration=0, warmup=True, feasible=False,
                                             failure_reason="CPU_OOM", failure_moment=0)], None
    reports = [engine.run_iteration(0, warmup=True, plan_builder=build)]
    for i in range(1, iterations):
        if not reports[-1].feasible:
            break
        reports.append(engine.run_iteration(i, warmup=False))
    return s, reports, engine.plan


def digest(sim, reports, plan):
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
            # samples only for the small cases (they are 2 per moment)
            "samples": samples(r) if len(r.samples) <= 2000 else None,
        } for r in reports],
        "final_states": {str(c.chunk_id): [t.state.value for t in c.tensors]
                         for c in sim.chunk_set.chunks.values()},
        "final_copies": {str(c.chunk_id): list(c.copies)
                         for c in sim.chunk_set.chunks.values()},
    }


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import importlib
    cs = importlib.import_module("chunkstar")
    for mod in ("model", "config", "scenario", "chunks", "parallel", "memory", "engine",
                "profiler"):
        importlib.import_module("chunkstar." + mod)
    assert cs.__file__.startswith(REF_SRC), cs.__file__
    golden = {"reference": REF_SRC, "cases": {}}
    for name, skw, hkw, pkw, nproc, ranks, iters in CASES:
        entry = {"schema": skw, "hardware": hkw, "policy": pkw, "nproc": nproc,
                 "iterations": iters, "ranks": {}}
        for rank in ranks:
            sim, reports, plan = run_rank(cs, name, skw, hkw, pkw, nproc, rank, iters)
            entry["ranks"][str(rank)] = digest(sim, reports, plan)
        golden["cases"][name] = entry
        last = entry["ranks"][str(ranks[0])]["iterations"]
        print("%-18s ranks=%s feasible=%s transfers/iter=%s coll/iter=%s"
              % (name, ranks, [it["feasible"] for it in last],
                 [len(it["transfers"]) for it in last], [len(it["collectives"]) for it in last]))
    with gzip.open(OUT, "wt") as f:
        json.dump(golden, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
