"""Timeline of the all-host-optimizer-state step (bench offload probe config).

Records, for one steady-state step: the GPU start time of every timeline
event (CUDA event on the compute stream), every chunk copy's GPU window
(copy-stream events) and every host Adam job's host window, relative to the
step start.  Prints a compact JSON summary; ``--ab`` alternates early
gradient drain on/off and prints ms/step for each.

    python scripts/offload_timeline.py [--batch 32] [--ab 3]
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

from paper_2108_05818_b200 import kernels as K  # noqa: E402
from paper_2108_05818_b200.config import PolicySpec  # noqa: E402
from paper_2108_05818_b200.model import build_gpt_schema  # noqa: E402
from paper_2108_05818_b200.trainer import ChunkTrainer  # noqa: E402


MODELS = {"1b": dict(layers=20, hidden_dim=2048, heads=16),
          "12b": dict(layers=60, hidden_dim=4096, heads=32)}


def make(batch, env, model="1b", os_placement="cpu"):
    os.environ.update(env)
    schema = build_gpt_schema(**MODELS[model], seq_len=1024, vocab=50304, batch=batch)
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=64 << 20, os_placement=os_placement),
                      seed=0, hyper=K.AdamHyper(lr=1e-4), time_copies=True)
    gen = torch.Generator().manual_seed(7)
    toks = [torch.randint(0, schema.vocab, (batch, 1025), generator=gen).cuda() for _ in range(2)]
    return tr, toks


def timed_steps(tr, toks, steps, warmup=6):
    for i in range(warmup):
        tr.step(toks[i % 2])
    tr.finish_host_work()
    torch.cuda.synchronize()
    hs0 = torch.cuda.host_memory_stats()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record()
    for i in range(steps):
        tr.step(toks[i % 2])
        evs[i + 1].record()
    tr.finish_host_work()
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    hs1 = torch.cuda.host_memory_stats()
    per = [round(evs[i].elapsed_time(evs[i + 1]), 1) for i in range(steps)]
    pinned = {k: hs1[k] - hs0.get(k, 0) for k in hs1
              if isinstance(hs1[k], (int, float)) and hs1[k] != hs0.get(k, 0)
              and ("alloc" in k or "free" in k or "time" in k.lower())}
    timed_steps.last = {"per_step_enqueue_boundaries_ms": per, "pinned_delta": pinned}
    return evs[0].elapsed_time(end) / steps


def timeline(tr, toks):
    eng, ex = tr.sim.engine, tr.executor
    marks = []
    s0, f0 = eng.start_event, eng.finish_event

    def start(ev):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((ev.index, ev.name, "start", time.perf_counter(), e))
        s0(ev)

    def finish(ev):
        f0(ev)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((ev.index, ev.name, "finish", time.perf_counter(), e))

    jobs = []
    r0 = ex._run_host_adam

    def run_host_adam(job, item, state):
        t = time.perf_counter()
        r0(job, item, state)
        jobs.append((job.cids[0], t, time.perf_counter()))

    for i in range(3):
        tr.step(toks[i % 2])
    tr.finish_host_work()
    torch.cuda.synchronize()
    for i in range(2):  # steady state: the host work of the previous step still runs
        tr.step(toks[i % 2])
    rs0 = ex._run_spec

    def run_spec(waits, item_in, item_out, state):
        t = time.perf_counter()
        rs0(waits, item_in, item_out, state)
        jobs.append(("spec", t, time.perf_counter()))

    blocks = []
    j0 = ex._join

    def join(cid):
        t = time.perf_counter()
        j0(cid)
        dt = time.perf_counter() - t
        if dt > 1e-3:
            blocks.append(("join", cid, t, t + dt))

    wr0 = ex.wait_ready

    def wait_ready(chunk, device):
        t = time.perf_counter()
        wr0(chunk, device)
        dt = time.perf_counter() - t
        if dt > 1e-3:
            blocks.append(("wait_ready_" + device, chunk.chunk_id, t, t + dt))

    eng.start_event, eng.finish_event, ex._run_host_adam = start, finish, run_host_adam
    ex._run_spec = run_spec
    ex._join, ex.wait_ready = join, wait_ready
    retries0 = torch.cuda.memory_stats().get("num_alloc_retries", 0)
    ex.stats.copy_events.clear()
    samples = []
    stop = threading.Event()
    main_id = threading.get_ident()

    def sampler():  # poor man's profiler of the enqueueing thread
        while not stop.is_set():
            f = sys._current_frames().get(main_id)
            stack = []
            while f is not None and len(stack) < 12:
                stack.append("%s:%d:%s" % (os.path.basename(f.f_code.co_filename), f.f_lineno,
                                           f.f_code.co_name))
                f = f.f_back
            samples.append((time.perf_counter(), stack))
            time.sleep(0.002)

    th = threading.Thread(target=sampler, daemon=True)
    z = torch.cuda.Event(enable_timing=True)
    z.record()
    hz = time.perf_counter()
    th.start()
    tr.step(toks[0])
    tr.step(toks[1])  # the next step's forward shows when the updated params land
    tr.finish_host_work()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    eng.start_event, eng.finish_event, ex._run_host_adam = s0, f0, r0
    ex._run_spec = rs0
    ex._join, ex.wait_ready = j0, wr0
    retries = torch.cuda.memory_stats().get("num_alloc_retries", 0) - retries0
    ev = [(i, n, k, round((h - hz) * 1e3, 2), round(z.elapsed_time(e), 2))
          for i, n, k, h, e in marks]
    copies = [(name, round(z.elapsed_time(a), 2), round(z.elapsed_time(b), 2), nb)
              for name, nb, a, b in ex.stats.copy_events]
    host = [(cid, round((a - hz) * 1e3, 2), round((b - hz) * 1e3, 2)) for cid, a, b in jobs]
    blk = [(k, cid, round((a - hz) * 1e3, 2), round((b - hz) * 1e3, 2)) for k, cid, a, b in blocks]
    smp = [(round((t - hz) * 1e3, 1), st) for t, st in samples]
    return {"events": ev, "copies": copies, "host_adam": host, "host_blocks": blk,
            "main_thread_samples": smp,
            "alloc_retries_recorded": retries}


def _busy(windows):
    """Union length of [a, b) windows (ms)."""
    tot, end = 0.0, None
    for a, b in sorted(windows):
        if end is None or a > end:
            tot += b - a
            end = b
        elif b > end:
            tot += b - end
            end = b
    return round(tot, 1)


def summarize(res):
    """Per phase of the FIRST recorded step (GPU clock): window, bytes and
    busy time of each copy direction inside it, host-Adam busy time."""
    ev = res["events"]
    starts = {}
    for i, n, k, h, g in ev:
        starts.setdefault((i, k), []).append(g)
    first = lambda key: starts[key][0]
    idx = sorted({i for i, *_ in ev})
    adam = idx[-1]
    n_fwd = (len(idx) - 1) // 2
    bounds = {"fwd": (first((idx[0], "start")), first((idx[n_fwd], "start"))),
              "bwd": (first((idx[n_fwd], "start")), first((adam, "start"))),
              "adam": (first((adam, "start")), starts[(idx[0], "start")][1])}
    out = {"step_ms": round(bounds["adam"][1] - bounds["fwd"][0], 1)}
    for ph, (a, b) in bounds.items():
        d = {"window_ms": round(b - a, 1)}
        for kind in ("gpu>cpu", "cpu>gpu"):
            w = [(max(x, a), min(y, b)) for n, x, y, nb in res["copies"] if n == kind and y > a and x < b]
            nb = sum(nb for n, x, y, nb in res["copies"] if n == kind and a <= x < b)
            d[kind] = {"busy_ms": _busy(w), "gb_started": round(nb / 1e9, 2)}
        d["host_adam_busy_ms"] = _busy([(max(x, a), min(y, b)) for c, x, y in res["host_adam"]
                                        if y > a and x < b])
        out[ph] = d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--model", default="1b", choices=sorted(MODELS))
    ap.add_argument("--os", default="cpu", help="os_placement (auto|cpu|gpu)")
    ap.add_argument("--ab", type=int, default=0)
    ap.add_argument("--arms", default="", help="JSON list of env dicts for --ab")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "offload_timeline.json"))
    args = ap.parse_args()
    if args.ab:
        arms = [{"CS_EARLY_DRAIN": "1", "CS_SPEC_HOST_ADAM": "1", "CS_WORKER_THREADS": "0"},
                {"CS_EARLY_DRAIN": "1", "CS_SPEC_HOST_ADAM": "1", "CS_WORKER_THREADS": "10"},
                {"CS_EARLY_DRAIN": "1", "CS_SPEC_HOST_ADAM": "0", "CS_WORKER_THREADS": "0"},
                {"CS_EARLY_DRAIN": "0", "CS_SPEC_HOST_ADAM": "0", "CS_WORKER_THREADS": "16"}]
        if args.arms:
            arms = json.loads(args.arms)
        for rep in range(args.ab):
            for env in arms:
                tr, toks = make(args.batch, env, args.model, args.os)
                ms = timed_steps(tr, toks, 4)
                st = tr.executor.stats
                print(json.dumps({"env": env, "rep": rep, "ms_per_step": round(ms, 2),
                                  "host_adam_s": round(st.host_adam_seconds, 3),
                                  "spec": [st.spec_issued, st.spec_committed, st.spec_discarded,
                                           st.spec_cancelled], **timed_steps.last}), flush=True)
                tr.close()
                del tr, toks, st
                import gc
                gc.collect()
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
                torch._C._host_emptyCache()  # pinned blocks back to the OS between arms
    tr, toks = make(args.batch, {"CS_EARLY_DRAIN": "1", "CS_SPEC_HOST_ADAM": "1",
                                 "CS_WORKER_THREADS": "0"}, args.model, args.os)
    res = timeline(tr, toks)
    res["summary"] = summarize(res)
    st = tr.executor.stats
    res["summary"]["exec_stats"] = {k: getattr(st, k) for k in (
        "prefetch_issued", "prefetch_hits", "prefetch_discarded", "adam_prefetch_early",
        "adam_prefetch_oom", "preevict_issued", "preevict_hits", "preevict_discarded",
        "early_drains", "spec_issued", "spec_committed", "spec_cancelled")}
    res["summary"]["alloc_retries"] = torch.cuda.memory_stats().get("num_alloc_retries", 0)
    print(json.dumps(res["summary"]))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f)
    # compact view: GPU start of the FWD/BWD/ADAM phases of both steps
    for i, n, k, h, g in res["events"]:
        if n.startswith(("embedding", "adam", "l0.qkv", "l10.qkv", "l19.mlp_out")):
            print("%-28s %-6s host %8.2f  gpu %8.2f" % (n, k, h, g))
    print("copies:", len(res["copies"]), "host adam jobs:", len(res["host_adam"]))


if __name__ == "__main__":
    main()
