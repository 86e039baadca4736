"""Benchmark of the chunk-managed GPT training step (PatrickStar) on B200.

Workload (BASELINE.json configs[1]): GPT-2 1B (L20 H2048, 16 heads,
S1024, V50304), fp16 chunks with dynamic loss scaling, all chunks
HBM-resident, per-GPU batch --batch (default 32, from C2's {4,8,16,32}: the
fastest), chunk capacity --cap
(default 64Mi elements).  A step = warm-up-planned chunk-managed forward +
backward + fused chunk Adam over one synthetic batch per GPU; N>1 ranks run
ZeRO chunk groups over NCCL (weak scaling: fixed per-GPU batch).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl chunk|reference]

Prints one JSON line (rank 0).  ``value`` = tokens/s over all ranks with
inputs already in HBM (CUDA events, max over ranks); ``e2e`` = the same
through ChunkTrainer.step_host_async (pinned host tokens H2D + loss D2H of
every step inside the timed region; step k's loss is read on the host once
step k+1 is enqueued, the usual lagged loss logging).  ``roofline`` = K1 fused chunk Adam timed in-region with
CUDA events on the compute stream.  ``cpu_baseline`` = the CPU port of the
step (oracle/cpu_step.py) on a bounded sample, rank 0 at N=1 only.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GPT tokens/sec & TFLOPS/GPU at 1/2/4/8 B200; chunk-Adam HBM GB/s vs peak"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chunk", choices=["chunk", "reference"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--cap", type=int, default=64 << 20)
    ap.add_argument("--layers", type=int, default=20)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--vocab", type=int, default=50304)
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--embedding-weights", default="hbm", choices=["hbm", "host"],
                    help="GPU-computed embedding state resident in HBM (default) or in host "
                         "DRAM with the reference's weight round trip realised")
    ap.add_argument("--no-graph", action="store_true",
                    help="eager steps only (no CUDA-graph replay of the steady state)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph-dp", action="store_true",
                    help="also capture the ZeRO step in a CUDA graph at N > 1 (opt-in: "
                         "unvalidated on multi-GPU hardware)")
    ap.add_argument("--dist-backend", default="nccl", help=argparse.SUPPRESS)
    ap.add_argument("--same-device", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-offload-probe", action="store_true",
                    help="skip the host-offload side measurement (chunk moves GB/s)")
    ap.add_argument("--cpu-sample-batch", type=int, default=1)
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the C5 microbench summary (K1-K6 1M-1G elements + CPU Adam arms)")
    ap.add_argument("--profile-step", action="store_true",
                    help="after warm-up run ONE step between cudaProfilerStart/Stop and exit "
                         "(for ncu --profile-from-start off); prints no bench line")
    return ap.parse_args()


def model_flops_per_step(B, S, L, H, V):
    """72·B·S·L·H²·(1 + S/(6H) + V/(12·L·H)) per GPU-batch."""
    return 72.0 * B * S * L * H * H * (1 + S / (6.0 * H) + V / (12.0 * L * H))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", 1382.7)), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def host_link_peak(dev, nbytes=1 << 30, iters=5):
    """Pinned cudaMemcpyAsync bandwidth H2D / D2H (GB/s), CUDA events."""
    import torch
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    devb = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {}
    for name, dst, src in (("h2d", devb, host), ("d2h", host, devb)):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            dst.copy_(src, non_blocking=True)
        b_.record()
        torch.cuda.synchronize()
        out[name] = nbytes * iters / (a.elapsed_time(b_) * 1e-3) / 1e9
    return out


def host_link_beside_host_adam(dev, threads, chunk=64 << 20, copies=16):
    """The same pinned copies (fp16 chunk-sized, 128 MiB, rotating over four
    buffers as the executor's drains and adam_copy do) while the host Adam
    (cs_adam_chunks_host, the executor's worker team) streams host DRAM:
    the link ceiling the offloaded step's moves can reach on this host."""
    import threading
    import torch
    from paper_2108_05818_b200 import _native as N
    from paper_2108_05818_b200 import kernels as K
    host = [torch.empty(chunk, dtype=torch.float16, pin_memory=True) for _ in range(4)]
    devb = [torch.empty(chunk, dtype=torch.float16, device=dev) for _ in range(4)]
    items = [(torch.empty(chunk, dtype=torch.float16).fill_(1e-3), torch.full((chunk,), 0.02),
              torch.zeros(chunk), torch.zeros(chunk), chunk) for _ in range(4)]
    st = K.speculate_step_scalars(N.CsStepState(beta1_pow=1.0, beta2_pow=1.0, step=0,
                                                loss_scale=1.0), K.AdamHyper(lr=1e-4))
    stop, started = threading.Event(), threading.Event()

    def adam_loop():
        while not stop.is_set():
            K.adam_chunks_host(items, K.AdamHyper(lr=1e-4), st, threads)
            started.set()

    th = threading.Thread(target=adam_loop)
    th.start()
    started.wait()
    out = {}
    try:
        for name in ("h2d", "d2h"):
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(copies):
                if name == "h2d":
                    devb[i % 4].copy_(host[i % 4], non_blocking=True)
                else:
                    host[i % 4].copy_(devb[i % 4], non_blocking=True)
            b_.record()
            torch.cuda.synchronize()
            out[name] = chunk * 2 * copies / (a.elapsed_time(b_) * 1e-3) / 1e9
    finally:
        stop.set()
        th.join()
    return out


def offload_probe(schema_kw, dev, steps=4, warmup=6):
    """The same 1B step with every optimizer triplet in pinned host DRAM
    (os_placement=cpu): grads D2H + host fused Adam + params H2D as
    `adam_copy` (`engine.py:249-251, 265-267`).  Reports the chunk moves'
    achieved host-link GB/s from copy-stream CUDA events."""
    import torch
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    peak = host_link_peak(dev)
    schema = build_gpt_schema(**schema_kw)
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=64 << 20, os_placement="cpu"),
                      seed=0, hyper=K.AdamHyper(lr=1e-4), time_copies=True)
    gen = torch.Generator().manual_seed(7)
    toks = [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1),
                          generator=gen).to(dev) for _ in range(2)]
    for i in range(warmup):
        tr.step(toks[i % 2])
    tr.finish_host_work()  # the warm-up's last host updates are not timed
    torch.cuda.synchronize()
    st = tr.executor.stats
    st.copy_events.clear()
    host0, items0 = st.host_adam_seconds, st.host_adam_items
    spec0 = (st.spec_issued, st.spec_committed, st.spec_discarded, st.spec_cancelled)
    pinned0 = torch.cuda.host_memory_stats().get("num_host_alloc", 0)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        tr.step(toks[i % 2])
    tr.finish_host_work()  # the last step's async host Adam is part of the step
    b_.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b_) / steps
    pinned_allocs = torch.cuda.host_memory_stats().get("num_host_alloc", 0) - pinned0
    spec = [x - y for x, y in zip((st.spec_issued, st.spec_committed, st.spec_discarded,
                                   st.spec_cancelled), spec0)]
    agg = {}
    for name, nbytes, e0, e1 in st.copy_events:
        t = e0.elapsed_time(e1)
        s = agg.setdefault(name, [0, 0.0, 0])
        s[0] += nbytes
        s[1] += t
        s[2] += 1
    moves = {}
    for name, (nbytes, t, n) in agg.items():
        key = "h2d" if name == "cpu>gpu" else "d2h"
        gbs = nbytes / (t * 1e-3) / 1e9 if t > 0 else None
        moves[key] = {"copies": n, "bytes": nbytes, "achieved_gbs": round(gbs, 1),
                      "peak_gbs": round(peak[key], 1), "frac": round(gbs / peak[key], 3)}
    try:  # after the trainer's timed steps: the host is otherwise idle
        beside = host_link_beside_host_adam(dev, tr.executor.worker_threads)
        for key, m in moves.items():
            m["ceiling_beside_host_adam_gbs"] = round(beside[key], 1)
            m["frac_of_that_ceiling"] = round(m["achieved_gbs"] / beside[key], 3)
    except Exception as e:  # reported, never fatal
        moves["ceiling_error"] = repr(e)[:200]
    rep = tr.reports[-1]
    out = {"workload": "GPT-1B step, os_placement=cpu (every optimizer triplet in pinned host "
                       "DRAM), B=%d" % schema.batch,
           "ms_per_step": round(ms, 2),
           "tokens_per_s": round(schema.batch * schema.seq_len / (ms * 1e-3), 1),
           "ledger_pcie_bytes_per_step": rep.pcie_bytes,
           "chunk_moves": moves,
           "host_adam_s_per_step": round((st.host_adam_seconds - host0) / steps, 4),
           "host_adam_gelem_per_s": round(
               sum(tr.sim.chunk_set.param_chunk(p).used_elems for p in tr.sim.local)
               / max((st.host_adam_seconds - host0) / steps, 1e-9) / 1e9, 3),
           "prefetch_hits": st.prefetch_hits, "prefetch_issued": st.prefetch_issued,
           "prefetch_discarded": st.prefetch_discarded,
           "async_host_adam": tr.executor.async_host_adam,
           "speculative_host_adam": {"enabled": tr.executor.speculative_host_adam,
                                     "issued_committed_discarded_cancelled": spec},
           "early_drains": st.early_drains,
           "pinned_host_allocs_during_timing": pinned_allocs,
           "worker_threads": tr.executor.worker_threads, "host_threads": tr.host_threads,
           "peak_source": "pinned cudaMemcpyAsync 1 GiB, host idle; ceiling_beside_host_adam: 128 MiB copies while the host Adam (worker team) streams host DRAM"}
    del tr
    torch.cuda.empty_cache()
    return out


def c5_probe(sizes=(20, 22, 24, 26, 28, 30), oracle_sizes=(20, 24)):
    """C5 (BASELINE.json configs[4]): K1 fused chunk Adam at 1M-1G elements,
    L2 flushed before every launch, HBM GB/s vs the measured peak; beside it
    the CPU Adam arms on the same element counts (torch-CPU fused Adam with
    the chunk casts, all threads; this build's host K1; the C oracle, one
    thread per core, at the small sizes only)."""
    import torch
    from paper_2108_05818_b200 import microbench as MB
    rows = MB.run(list(sizes), iters=5, kernels=("adam", "sumsq", "pack", "accumulate",
                                                  "cast_pack", "master_init"))
    torch.cuda.empty_cache()
    table = {}
    for r in rows:
        e = table.setdefault(str(r["n"]), {})
        e[r["kernel"]] = {"gpu_gbs": r["gbs"], "gpu_frac": r["frac_of_measured_peak"],
                          "regime": r["regime"]}
    for lg in sizes:
        n = 1 << lg
        it = 1 if n >= (1 << 29) else 2
        a = MB.cpu_torch_fused_adam(n, it)
        b = MB.cpu_host_k1(n, it)
        table[str(n)]["adam"].update({"cpu_torch_fused_gbs": a["gbs"],
                                      "cpu_torch_fused_threads": a["threads"],
                                      "cpu_host_k1_gbs": b["gbs"],
                                      "cpu_host_k1_threads": b["threads"]})
    for lg in oracle_sizes:  # the C restatement (checker), scalar
        import numpy as np
        import time as _t
        from oracle import numerics as O
        n = 1 << lg
        rng = np.random.default_rng(0)
        g = O.to_half_bits((rng.standard_normal(n) * 1e-3).astype(np.float32))
        p32 = (rng.standard_normal(n) * 0.02).astype(np.float32)
        m, v = np.zeros(n, np.float32), np.zeros(n, np.float32)
        st = O.step_state(1.0)
        O.adam_prepare(st, 1e-4, 0.9, 0.999)
        thr = len(os.sched_getaffinity(0))
        t0 = _t.perf_counter()
        O.adam(g, p32, m, v, n, O.FP16, 1e-4, 0.9, 0.999, 1e-8, 0.0, False, st, threads=thr)
        dt = _t.perf_counter() - t0
        table[str(n)]["adam"].update({"cpu_oracle_gbs": round(28 * n / dt / 1e9, 3),
                                      "cpu_oracle_threads": thr})
    return {"kernels_bytes_per_elem": MB.BYTES_PER_ELEM, "peak_gbs": MB.measured_peak_gbs(),
            "l2": "flushed (a read of 2 x 126 MB: cold, clean) before every GPU launch",
            "cpu_arms": "torch.optim.Adam(fused=True) on CPU incl. fp16->fp32 grad and "
                        "fp32->fp16 param casts; cs_adam_chunks_host (AVX2+OpenMP); C oracle "
                        "(scalar C, OpenMP over the affinity mask)", "rows": table}


NVLINK_PEAK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md; 900 nominal)


def collective_probe(dev, cap, dtype, world, iters=5, warmup=2):
    """The chunk-group collectives of the step, timed alone: all-gather of a
    p x cap group slab and reduce-scatter(avg) back to one cap chunk
    (`parallel.py:196-264`), each issued synchronously on the current stream
    and bracketed by CUDA events there; max over ranks.  busbw = (p-1)*cap*
    elem_bytes / t against the measured 770 GB/s peer copy."""
    import torch
    import torch.distributed as dist
    slab = torch.empty(world * cap, dtype=dtype, device=dev).normal_()
    out = torch.empty(cap, dtype=dtype, device=dev)
    rank = dist.get_rank()
    mine = slab[rank * cap:(rank + 1) * cap]
    res = {}
    for name, fn in (("all_gather", lambda: dist.all_gather_into_tensor(slab, mine)),
                     ("reduce_scatter_avg",
                      lambda: dist.reduce_scatter_tensor(out, slab, op=dist.ReduceOp.AVG))):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        busbw = (world - 1) * cap * slab.element_size() / (ms * 1e-3) / 1e9
        res[name] = {"ms": round(ms, 4), "busbw_gbs": round(busbw, 1),
                     "frac": round(busbw / NVLINK_PEAK_GBS, 4)}
    res.update({"group_slab_bytes": world * cap * slab.element_size(), "p": world,
                "peak_gbs": NVLINK_PEAK_GBS,
                "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                "timing": "CUDA events on the issuing stream, %d back-to-back calls, max over "
                          "ranks" % iters})
    del slab, out
    return res


def collectives_in_step(durations, world, steps):
    """Per kind: count per step, mean ms and busbw of the chunk-group
    collectives as they ran inside the timed steps (overlapped with compute),
    busbw = (p-1) * slot bytes / duration, max over ranks."""
    import torch
    import torch.distributed as dist
    kinds = ("all_gather", "reduce_scatter_avg")
    agg = {k: [0, 0.0, 0] for k in kinds}  # count, ms, wire bytes
    src = "none"
    for kind, nbytes, ms, how in durations:
        a = agg.setdefault(kind, [0, 0.0, 0])
        a[0] += 1
        a[1] += ms
        a[2] += (world - 1) * nbytes // world
        src = how
    t = torch.tensor([agg[k][1] for k in kinds], dtype=torch.float64,
                     device=torch.cuda.current_device())
    if dist.get_backend() == "gloo":
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res = {}
    for i, k in enumerate(kinds):
        n, _, wire = agg[k]
        ms = float(t[i])
        busbw = wire / (ms * 1e-3) / 1e9 if ms > 0 else None
        res[k] = {"per_step": n / max(steps, 1), "mean_ms": round(ms / n, 4) if n else None,
                  "busbw_gbs": round(busbw, 1) if busbw else None,
                  "frac": round(busbw / NVLINK_PEAK_GBS, 4) if busbw else None}
    res["timing"] = ("Work.get_duration (NCCL-stream events)" if src == "work" else
                     "CUDA events from issue to completion (includes queueing behind earlier "
                     "collectives)")
    return res


def k1_traffic(elements):
    """Per-launch DRAM traffic of K1 from the committed `ncu --set full`
    capture of the same in-step launch (profiles/), scaled to this launch's
    element count when it differs; None if no capture is committed."""
    path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        per_elem = (d["dram_bytes_read"] + d["dram_bytes_write"]) / d["elements"]
        return round(per_elem * elements, 0), d["source"]
    except Exception:
        return None, None


def host_info():
    """What `cores` means on this host: logical CPUs in the affinity mask,
    SMT siblings per core, NUMA nodes (sysfs)."""
    cpus = sorted(os.sched_getaffinity(0))
    smt = 1
    try:
        with open("/sys/devices/system/cpu/cpu%d/topology/thread_siblings_list" % cpus[0]) as f:
            from paper_2108_05818_b200.hostres import parse_cpulist
            smt = len(parse_cpulist(f.read().strip()))
    except OSError:
        pass
    nodes = len([d for d in os.listdir("/sys/devices/system/node")
                 if d.startswith("node")]) if os.path.isdir("/sys/devices/system/node") else 1
    return {"logical_cpus": len(cpus), "threads_per_core": smt,
            "physical_cores": len(cpus) // max(smt, 1), "numa_nodes": nodes}


def cpu_baseline(schema_kw, sample_batch, steps=1):
    from oracle.cpu_step import CpuChunkStep
    from paper_2108_05818_b200.model import build_gpt_schema
    schema = build_gpt_schema(**schema_kw)
    runner = CpuChunkStep(schema, sample_batch=sample_batch)
    secs = [runner.step() for _ in range(steps)]
    t = min(secs)
    return {"value": round(runner.tokens_per_step / t, 3), "unit": UNIT,
            "cores": runner.threads, "kind": "port", "host": host_info(),
            "sample": "%d x %d tokens on the full %d-layer H%d model per step (fp32 torch-CPU "
                      "fwd/bwd + C-oracle chunk Adam over all %.2fB params + the decision "
                      "engine), best of %d" % (sample_batch, schema.seq_len, schema.layers,
                                               schema.hidden_dim,
                                               sum(p.numel() for p in runner.model.parameters())
                                               / 1e9, steps)}


REF_ENGINE_CODE = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
import chunkstar
from chunkstar.config import HardwareSpec, PolicySpec
from chunkstar.model import build_gpt_schema
from chunkstar.scenario import Simulator
assert chunkstar.__file__.startswith(sys.argv[1]), chunkstar.__file__
kw = json.loads(sys.argv[2])
schema = build_gpt_schema(**kw["schema"])
sim = Simulator(schema, HardwareSpec(gpu_count=1, gpu_bytes=kw["gpu_bytes"]),
                PolicySpec(capacity_elems=kw["cap"]), 1)
t0 = time.perf_counter()
warm = sim.engine.run_iteration(0, warmup=True, plan_builder=sim._plan_builder())
t1 = time.perf_counter()
secs = []
for i in range(1, 1 + kw["iters"]):
    a = time.perf_counter()
    r = sim.engine.run_iteration(i, warmup=False)
    secs.append(time.perf_counter() - a)
    assert r.feasible
print(json.dumps({"warmup_s": t1 - t0, "measured_s": secs, "events": len(sim.timeline.events),
                  "pcie_bytes": r.pcie_bytes}))
"""


def decision_engine_timing(args, iters=3):
    """SURVEY §8(d) CPU baseline item 1: the UNMODIFIED reference's
    `Engine.run_iteration` (`cs/engine.py:282-364`, installed under
    baseline/_ref) on the bench's timeline, one Python thread, beside this
    build's decision engine (accounting-only) on the same timeline."""
    import subprocess
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    schema = dict(layers=args.layers, hidden_dim=args.hidden, heads=args.heads,
                  seq_len=args.seq, vocab=args.vocab, batch=args.batch)
    kw = {"schema": schema, "cap": args.cap, "gpu_bytes": 160 * 10**9, "iters": iters}
    out = {"config": "GPT L%d H%d B%d cap %d, 160 GB accounting budget"
                     % (args.layers, args.hidden, args.batch, args.cap)}
    if os.path.isdir(os.path.join(ref_dir, "chunkstar")):
        res = subprocess.run([sys.executable, "-c", REF_ENGINE_CODE, ref_dir, json.dumps(kw)],
                             capture_output=True, text=True, timeout=900)
        if res.returncode == 0:
            d = json.loads(res.stdout.strip().splitlines()[-1])
            out["reference_ms_per_iteration"] = round(1e3 * min(d["measured_s"]), 2)
            out["reference_warmup_ms"] = round(1e3 * d["warmup_s"], 2)
            out["events"] = d["events"]
        else:
            out["reference_error"] = res.stderr[-300:]
    else:
        out["reference_error"] = "baseline/_ref not installed"
    from paper_2108_05818_b200.config import HardwareSpec, PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.scenario import Simulator
    sim = Simulator(build_gpt_schema(**schema), HardwareSpec(gpu_count=1, gpu_bytes=kw["gpu_bytes"]),
                    PolicySpec(capacity_elems=args.cap), 1)
    sim.engine.run_iteration(0, warmup=True, plan_builder=sim._plan_builder())
    secs = []
    for i in range(1, 1 + iters):
        a = time.perf_counter()
        sim.engine.run_iteration(i, warmup=False)
        secs.append(time.perf_counter() - a)
    out["this_build_ms_per_iteration"] = round(1e3 * min(secs), 2)
    out["threads"] = 1
    return out


def workload_config(args, world):
    """The workload both arms are measured on (the reference arm runs a
    bounded sample of it, described in its ``cpu_baseline.sample``)."""
    return {"workload": "GPT-2 1B chunk-managed training step (configs[1])",
            "model": "GPT L%d H%d heads%d S%d V%d (reference-shaped, 8 chunked "
                     "tensors/layer)" % (args.layers, args.hidden, args.heads, args.seq,
                                         args.vocab),
            "global_batch": world * args.batch, "per_gpu_batch": args.batch,
            "seq_len": args.seq, "chunk_capacity_elems": args.cap,
            "parallelism": "zero-chunk-dp%d" % world,
            "l2": "inputs larger than L2 (16 GB of chunk state streamed per step)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    schema_kw = dict(layers=args.layers, hidden_dim=args.hidden, heads=args.heads,
                     seq_len=args.seq, vocab=args.vocab, batch=args.batch)
    from oracle.cpu_step import CpuChunkStep
    from paper_2108_05818_b200.model import build_gpt_schema
    runner = CpuChunkStep(build_gpt_schema(**schema_kw), sample_batch=args.cpu_sample_batch)
    for _ in range(args.warmup):
        runner.step()
    secs = [runner.step() for _ in range(args.steps)]
    total = sum(secs)
    value = runner.tokens_per_step * len(secs) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(secs), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": workload_config(args, int(os.environ.get("WORLD_SIZE", "1"))),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": runner.threads,
                         "kind": "port", "host": host_info(),
                         "sample": "%d x %d tokens per step on the full model (fp32 "
                                   "torch-CPU fwd/bwd + C-oracle chunk Adam over every "
                                   "parameter + the decision engine): a bounded sample of "
                                   "the workload's %d x %d tokens per GPU"
                                   % (args.cpu_sample_batch, args.seq, args.batch, args.seq)},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    try:
        line["decision_engine"] = decision_engine_timing(args)
    except Exception as e:  # reported, never fatal
        line["decision_engine"] = {"error": repr(e)[:300]}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2108_05818_b200 import _native
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:  # test hook: several ranks on one GPU (gloo only)
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.dist_backend == "nccl":
            # per-collective start/end events on the NCCL stream: the in-step
            # durations of the chunk-group collectives (Work.get_duration)
            os.environ.setdefault("TORCH_NCCL_ENABLE_TIMING", "1")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    schema_kw = dict(layers=args.layers, hidden_dim=args.hidden, heads=args.heads,
                     seq_len=args.seq, vocab=args.vocab, batch=args.batch)
    schema = build_gpt_schema(**schema_kw)
    dtype = torch.float16 if args.dtype == "fp16" else torch.bfloat16
    trainer = ChunkTrainer(schema, PolicySpec(capacity_elems=args.cap), dtype=dtype, seed=0,
                           hyper=K.AdamHyper(lr=1e-4, betas=(0.9, 0.999), eps=1e-8),
                           cuda_graph=not args.no_graph, graph_multi_rank=args.graph_dp,
                           embedding_weights=args.embedding_weights)
    ex = trainer.executor
    B, S = args.batch, args.seq
    gen = torch.Generator().manual_seed(1000 + rank)
    pool = [torch.randint(0, args.vocab, (B, S + 1), generator=gen).pin_memory()
            for _ in range(4)]
    dev_pool = [t.to(dev) for t in pool]

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(max(args.warmup, 1)):
        trainer.step(dev_pool[i % 4])
    if trainer.cuda_graph:  # reach the fixed point and capture before timing
        while trainer._graph is None and trainer.iteration < args.warmup + 6:
            trainer.step(dev_pool[trainer.iteration % 4])
    torch.cuda.synchronize()
    barrier()
    if args.profile_step:
        torch.cuda.cudart().cudaProfilerStart()
        trainer.step(dev_pool[0])
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return

    # ---- timed region 1: device-resident inputs -> value -----------------------
    ex.record_k1 = True
    ex.k1_events.clear()
    if world > 1:  # in-step durations of the overlapped chunk-group collectives
        ex.time_collectives = True
        ex.coll_log.clear()
    moved0 = ex.stats.h2d_bytes - ex.stats.prefetch_discarded_bytes + ex.stats.d2h_bytes
    he = trainer.host_embedding
    emb_moved0 = he.h2d_bytes + he.d2h_bytes if he is not None else 0
    reports0 = len(trainer.reports)
    launches0 = _native.launch_count()
    clocks = ClockSampler(local_rank)
    clocks.start()
    torch.cuda.synchronize()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    t0.record()
    for k in range(args.steps):
        loss = trainer.step(dev_pool[k % 4])
    t1.record()
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = _native.launch_count() - launches0
    if trainer._graph is not None:  # library kernels replayed from the captured graph
        launches += trainer.graph_kernels_per_step * args.steps
    ms = t0.elapsed_time(t1) / args.steps
    in_step = None
    if world > 1:
        ex.time_collectives = False
        in_step = collectives_in_step(ex.collective_durations(), world, args.steps)
        ex.coll_log.clear()
    # chunk bytes the executor moved in the timed steps (a replayed graph
    # moves none: it is only captured once the schedule moves no chunk)
    moved = (ex.stats.h2d_bytes - ex.stats.prefetch_discarded_bytes + ex.stats.d2h_bytes
             - moved0) / args.steps
    emb_moved = ((he.h2d_bytes + he.d2h_bytes - emb_moved0) / args.steps
                 if he is not None else 0)
    billed = [r.pcie_bytes for r in trainer.reports[reports0:reports0 + args.steps]]
    ex.record_k1 = False
    k1_ms = [a.elapsed_time(b) for a, b, _ in ex.k1_events]
    k1_elems = [n for _, _, n in ex.k1_events]
    k1_note = "mean over the timed region's eager steps"
    if trainer._graph is not None and trainer.graph_k1 is not None:
        # every replay re-records the graph's K1 event nodes: read the last
        # timed replay, then sample further replays of the same step
        a, b, n = trainer.graph_k1
        k1_ms, k1_elems = [a.elapsed_time(b)], [n]
        for k in range(5):
            trainer.step(dev_pool[k % 4])
            torch.cuda.synchronize()
            k1_ms.append(a.elapsed_time(b))
            k1_elems.append(n)
        k1_note = ("mean of %d replays' K1 event-record nodes (last timed replay + %d "
                   "sampled replays of the same graph)" % (len(k1_ms), len(k1_ms) - 1))
    final_loss = float(loss.item())
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # ---- timed region 2: end to end through the public API -----------------------
    torch.cuda.synchronize()
    barrier()
    clocks2 = ClockSampler(local_rank)
    clocks2.start()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0 = time.perf_counter()
    d0.record()
    pending = None
    for k in range(args.steps):  # step k's loss is read once step k+1 is enqueued
        nxt = trainer.step_host_async(pool[k % 4])
        if pending is not None:
            pending.result()
        pending = nxt
    pending.result()
    d1.record()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - e0) * 1e3 / args.steps
    e2e_dev_ms = d0.elapsed_time(d1) / args.steps
    clk2 = clocks2.stop()
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    hbm_peak, bf16_peak, peak_src = measured_peaks()
    tokens_per_step = world * B * S
    flops = model_flops_per_step(B, S, args.layers, args.hidden, args.vocab)
    k1_avg_ms = sum(k1_ms) / len(k1_ms) if k1_ms else float("nan")
    k1_bytes = 28.0 * (sum(k1_elems) / len(k1_elems)) if k1_elems else 0.0
    k1_gbs = k1_bytes / (k1_avg_ms * 1e-3) / 1e9 if k1_ms else None
    st = trainer.step_state()
    traffic, traffic_src = k1_traffic(int(k1_bytes // 28))
    out = {
        "metric": METRIC, "value": round(tokens_per_step / (ms * 1e-3), 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": workload_config(args, world),
        "layout": {"positions": trainer.sim.chunk_set.positions,
                   "os_on_gpu": len(trainer.sim.engine.plan.os_positions_on_gpu)},
        "tflops_per_gpu": round(flops / (ms * 1e-3) / 1e12, 2),
        "tflops_frac_of_sustained_bf16": round(flops / (ms * 1e-3) / 1e12 / bf16_peak, 4),
        "roofline": {"kernel": "cs_adam_chunks (K1 fused chunk Adam)", "bound": "hbm",
                     "achieved": round(k1_gbs, 1) if k1_gbs else None, "peak": hbm_peak,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(k1_gbs / hbm_peak, 4) if k1_gbs else None,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": k1_bytes,
                     "elements_per_launch": int(k1_bytes // 28),
                     "avg_launch_ms": round(k1_avg_ms, 4),
                     "launch_ms_samples": [round(x, 4) for x in k1_ms],
                     "timing": k1_note,
                     "share_of_step": round(k1_avg_ms / ms, 4)},
        "e2e": {"value": round(tokens_per_step / (e2e_ms * 1e-3), 1), "unit": UNIT,
                "h2d_bytes_per_step": pool[0].numel() * pool[0].element_size(),
                "d2h_bytes_per_step": 4, "ms_per_step": round(e2e_ms, 3),
                "device_ms_per_step": round(e2e_dev_ms, 3),
                "sm_mhz": clk2.get("sm_mhz")},
        "pcie_per_step": {
            "ledger_billed_bytes": int(sum(billed) / max(len(billed), 1)),
            "physically_moved_chunk_bytes": int(moved),
            "physically_moved_embedding_bytes": int(emb_moved),
            "ledger_rows_not_realized": trainer.ledger_rows_not_realized(),
            "embedding_weights": trainer.embedding_weights,
            "note": "the reference bills a GPU-computed embedding's weights down at FWD and "
                    "weight grads up at BWD (engine.py:214-219); by default they stay resident "
                    "in HBM, charged to the GPU pool; --embedding-weights host realises the "
                    "round trip (DESIGN.md section 7)"},
        "gpu_resident_non_chunked_bytes": trainer.gpu_resident_bytes,
        "non_model": "measured" if trainer.tracer is not None else "analytic",
        "host_threads": trainer.host_threads,
        "gpu_launches": int(launches),
        "host_enqueue_ms_per_step": round(host_ms, 3),
        "cuda_graph": trainer._graph is not None,
        "clocks": clk,
        "final_loss": final_loss, "loss_scale": st.loss_scale, "adam_steps": int(st.step),
    }
    if world > 1:
        from paper_2108_05818_b200.parallel import CollectiveScheme, closed_form_volume
        rep = trainer.reports[-1]
        out["collectives_per_step"] = {
            "ledger_bytes_per_rank": int(sum(c.bytes for c in rep.collectives)),
            "count": len(rep.collectives),
            "closed_form_bytes_per_rank": int(closed_form_volume(
                world, trainer.sim.partition.padded_param_elems(args.cap),
                CollectiveScheme.CHUNK_COLLECTIVE))}
        del trainer, ex
        torch.cuda.empty_cache()
        try:
            out["collectives"] = collective_probe(dev, args.cap, dtype, world)
        except Exception as e:  # reported, never fatal
            out["collectives"] = {"error": repr(e)[:300]}
        out["collectives"]["in_step"] = in_step
    if world == 1 and not args.no_offload_probe:
        del trainer, ex
        torch.cuda.empty_cache()
        try:
            out["offload_probe"] = offload_probe(schema_kw, dev)
        except Exception as e:  # reported, never fatal
            out["offload_probe"] = {"error": repr(e)[:300]}
    if world == 1 and not args.no_c5:
        torch.cuda.empty_cache()
        try:
            out["c5"] = c5_probe()
        except Exception as e:  # reported, never fatal
            out["c5"] = {"error": repr(e)[:300]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(schema_kw, args.cpu_sample_batch)
        except Exception as e:  # reported, never fatal
            out["cpu_baseline"] = {"value": None, "error": repr(e)[:200]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
