"""End-to-end parity of the REAL chunk-managed training step on a B200.

* Ledger parity: the trainer's transfer ledger (every H2D/D2H it really
  performed), collective ledger, placement plan and layout equal the
  REFERENCE's frozen ledgers (tests/golden/decisions.json.gz) for the tiny
  GPT C1 under an all-resident budget, a tight budget (evictions + optimizer
  state split between HBM and host) and forced host optimizer state.
* Adam parity inside the step: every K1 launch of a real step replayed by
  the C oracle, byte for byte.
* Placement invariance: the tight-budget run (evictions, host Adam) and the
  all-resident run produce bit-identical losses and parameters.
"""

import gzip
import json
import os

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec  # noqa: E402
from paper_2108_05818_b200.model import build_gpt_schema  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "decisions.json.gz")
with gzip.open(GOLDEN, "rt") as _f:
    CASES = json.load(_f)["cases"]


def _trainer(case, seed=0, **kw):
    """C1's plan computes the embedding on the CPU (`profiler.py:70-74`),
    which needs the untied LM head (explicit opt-in)."""
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES[case]
    schema = build_gpt_schema(**c["schema"])
    kw.setdefault("untied_head", True)
    return ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                        dtype=torch.float16, seed=seed, **kw), schema


def _tokens(schema, n, seed=123):
    g = torch.Generator().manual_seed(seed)
    return [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
            for _ in range(n)]


def _ledger(r):
    return {"transfers": [[t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason]
                          for t in r.transfers],
            "collectives": [[c.iteration, c.group_id, c.kind, c.bytes, c.includes_padding]
                            for c in r.collectives],
            "samples": [[s.moment, s.device, s.used_bytes, s.chunk_bytes, s.non_model_bytes]
                        for s in r.samples]}


@pytest.mark.parametrize("case", ["tiny_cap1Mi", "tiny_cap256Ki", "tiny_tight", "tiny_os_cpu",
                                  "tiny_ckpt_tight"])
def test_real_step_ledgers_match_reference(case):
    tr, schema = _trainer(case)
    ref = CASES[case]["ranks"]["0"]
    losses = [tr.step_host(t) for t in _tokens(schema, CASES[case]["iterations"])]
    tr.finish_host_work()  # the last step's host Adam / adam_copy H2D may still be in flight
    assert all(np.isfinite(losses))
    assert [list(r) for r in tr.sim.chunk_set.layout_rows()] == ref["layout"]
    plan = tr.sim.engine.plan
    assert list(plan.os_positions_on_gpu) == ref["plan"]["os_positions_on_gpu"]
    for mine, theirs in zip(tr.reports, ref["iterations"]):
        got = _ledger(mine)
        assert got["transfers"] == theirs["transfers"], (case, mine.iteration)
        assert got["collectives"] == theirs["collectives"]
        assert got["samples"] == theirs["samples"]
    # the executor moved exactly the bytes the ledger bills: chunk rows, and
    # (CPU-placed embedding, the plan for C1) the activation rows
    chunk_rows = [t for r in tr.reports for t in r.transfers if t.chunk_id != "embedding"]
    h2d = sum(t.bytes for t in chunk_rows if (t.src, t.dst) == ("cpu", "gpu"))
    d2h = sum(t.bytes for t in chunk_rows if (t.src, t.dst) == ("gpu", "cpu"))
    st = tr.executor.stats
    assert st.h2d_bytes - st.prefetch_discarded_bytes == h2d and st.d2h_bytes == d2h
    assert tr.sim.engine.embedding_device == tr.embedding_placement == "cpu"
    emb_rows = [t for r in tr.reports for t in r.transfers if t.chunk_id == "embedding"]
    he = tr.host_embedding
    assert he.h2d_bytes == sum(t.bytes for t in emb_rows if t.src == "cpu") > 0
    assert he.d2h_bytes == sum(t.bytes for t in emb_rows if t.src == "gpu") > 0


def test_adam_inside_real_step_matches_oracle():
    from oracle import step_check
    tr, schema = _trainer("tiny_cap256Ki")
    toks = _tokens(schema, 3)
    tr.step_host(toks[0])
    rec = step_check.arm(tr)
    tr.step_host(toks[1])
    tr.step_host(toks[2])
    step_check.disarm(tr)
    assert rec["checked"] >= 2 * (tr.sim.chunk_set.positions + len(tr.executor.embedding))
    assert rec["mismatch"] == []


def test_host_placement_and_eviction_do_not_change_numerics():
    from torch.nn.attention import SDPBackend, sdpa_kernel
    with sdpa_kernel(SDPBackend.MATH):  # deterministic attention backward
        runs = {}
        for case in ("tiny_cap256Ki", "tiny_tight"):
            tr, schema = _trainer(case)
            losses = [tr.step_host(t) for t in _tokens(schema, 4)]
            params = []
            for pos in range(tr.sim.chunk_set.positions):
                n = tr.sim.chunk_set.param_chunk(pos).used_elems
                params.append(tr.local_chunk_payload(pos).cpu()[:n].clone())
            runs[case] = (losses, params, tr.executor.stats)
        assert runs["tiny_tight"][2].host_adam_items > 0      # host Adam really ran
        assert runs["tiny_tight"][2].d2h_bytes > 0            # evictions really moved data
        assert runs["tiny_tight"][2].prefetch_hits > 0        # fetches ran ahead of need
        assert runs["tiny_cap256Ki"][0] == runs["tiny_tight"][0]
        for a, b in zip(runs["tiny_cap256Ki"][1], runs["tiny_tight"][1]):
            assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_loss_decreases_on_repeated_batch():
    tr, schema = _trainer("tiny_cap256Ki")
    batch = _tokens(schema, 1)[0]
    losses = [tr.step_host(batch) for _ in range(8)]
    assert losses[-1] < losses[0] - 0.05, losses


def test_cuda_graph_replay_matches_eager_steps():
    """Steady-state CUDA-graph replay is bit-identical to eager steps and the
    accounting still produces every iteration's (unchanged) ledger."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_cap256Ki"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 8)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for graph in (False, True):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, cuda_graph=graph,
                              embedding_placement="gpu")  # graphs need no host operator
            losses = [tr.step_host(t) for t in toks]
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            out[graph] = (losses, params, tr)
    assert out[True][2]._graph is not None and out[False][2]._graph is None
    assert out[True][0] == out[False][0]
    for a, b in zip(out[True][1], out[False][1]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    ref = CASES["tiny_cap256Ki"]["ranks"]["0"]["iterations"][-1]
    for r in out[True][2].reports[2:]:
        assert _ledger(r)["transfers"] == ref["transfers"]
        assert _ledger(r)["samples"] == ref["samples"]


@pytest.mark.parametrize("case,graph", [("tiny_cap256Ki", True), ("tiny_tight", False)])
def test_lagged_loss_reads_match_synchronous_steps(case, graph):
    """step_host_async with step k's loss read after step k+1 is enqueued (the
    bench's e2e loop) trains exactly like synchronous step_host: CUDA-graph
    replay, and eager steps with evictions, host Adam and the CPU embedding."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES[case]
    schema = build_gpt_schema(**c["schema"])
    toks = [t.pin_memory() for t in _tokens(schema, 7)]
    extra = dict(cuda_graph=True, embedding_placement="gpu") if graph else {}
    out = []
    with sdpa_kernel(SDPBackend.MATH):
        for lagged in (False, True):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, **extra)
            if not lagged:
                losses = [tr.step_host(t) for t in toks]
            else:
                pend = [tr.step_host_async(t) for t in toks[:1]]
                for t in toks[1:]:
                    pend.append(tr.step_host_async(t))
                    pend[-2].result()
                losses = [p.result() for p in pend]
            tr.finish_host_work()
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            out.append((losses, params, tr._graph is not None))
    assert out[0][2] == out[1][2] == graph
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1], out[1][1]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("case,init_scale", [("tiny_os_cpu", None), ("tiny_tight", None),
                                              ("tiny_os_cpu", 2.0 ** 40)])
def test_speculative_host_adam_is_bit_identical(case, init_scale):
    """Speculative host Adam (updates of host-placed positions started during
    the backward on the priority worker, settled at ADAM: adopted only if the
    real step scalars match, else recomputed) gives the same ledgers, losses
    and parameters as the normal walk; an overflowing start (scale 2^40)
    exercises the discard path."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES[case]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 6)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for spec in (False, True):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, speculative_host_adam=spec,
                              init_loss_scale=init_scale, untied_head=True)
            tr.executor.copy_delay_cycles = 500_000 if spec else 0  # moves land late too
            losses = [tr.step_host(t) for t in toks]
            tr.finish_host_work()
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            out[spec] = (losses, params, [_ledger(r) for r in tr.reports], tr.executor.stats)
    st = out[True][3]
    assert st.spec_issued > 0 and out[False][3].spec_issued == 0
    if init_scale is None:
        assert st.spec_committed > 0 and st.spec_discarded == 0
    else:  # overflow steps: speculation thrown away (or cancelled before it ran)
        assert st.spec_discarded + st.spec_cancelled > 0
    assert out[True][0] == out[False][0]
    assert out[True][2] == out[False][2]
    for a, b in zip(out[True][1], out[False][1]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_checkpointing_does_not_change_numerics():
    """Recomputed activations give bit-identical training (deterministic attention)."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_cap256Ki"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 3)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for ckpt in (False, True):
            pol = dict(c["policy"], checkpointing=ckpt)
            tr = ChunkTrainer(schema, PolicySpec(**pol), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0)
            out[ckpt] = [tr.step_host(t) for t in toks]
            if ckpt:
                names = [tr.sim.timeline.events[0].name]
                assert tr.sim.timeline.checkpointed and tr.model.checkpointing
    assert out[True] == out[False]


def test_real_run_ledger_files_equal_reference_files(tmp_path):
    """A real B200 run writes the same ledger bytes the reference simulator
    writes for the same config (tests/golden/ledgers/tiny_tight)."""
    tr, schema = _trainer("tiny_tight")
    for t in _tokens(schema, 3):
        tr.step_host(t)
    tr.write_ledgers(str(tmp_path))
    gold = os.path.join(os.path.dirname(__file__), "golden", "ledgers", "tiny_tight")
    for fname in ("layout.csv", "moments_chunk.csv", "transfers_chunk.csv",
                  "collectives_chunk.csv"):
        with open(os.path.join(gold, fname), "rb") as f, open(tmp_path / fname, "rb") as g:
            assert g.read() == f.read(), fname


def test_measured_warmup_tracer_drives_the_same_decisions():
    """non_model='measured': the warm-up's live R - C readings drive the plan
    and the frozen curve drives later iterations; replaying exactly those
    values through the accounting-only engine (pinned to the reference by
    tests/test_decisions_golden.py) reproduces every ledger row."""
    from paper_2108_05818_b200.scenario import Simulator
    from paper_2108_05818_b200.trainer import ChunkTrainer
    import gc
    gc.collect()  # earlier tests' trainers must not be freed mid-measurement
    torch.cuda.empty_cache()
    c = CASES["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    probe = ChunkTrainer(schema, PolicySpec(**c["policy"]),
                         HardwareSpec(gpu_count=1, gpu_bytes=8 << 30), dtype=torch.float16,
                         seed=0, non_model="measured")
    probe.step_host(_tokens(schema, 1)[0])
    budget = probe.tracer.peak + (24 << 20)  # measured footprint + a few chunks
    del probe
    import gc
    gc.collect()
    hw = HardwareSpec(gpu_count=1, gpu_bytes=budget)
    tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), hw, dtype=torch.float16, seed=0,
                      non_model="measured")
    for t in _tokens(schema, 3):
        tr.step_host(t)
    tracer = tr.tracer
    assert tracer.frozen and tracer.peak > 0
    n_moments = tr.sim.timeline.moment_count
    # the plan's peak = measured R - C plus the accounted BWD staging temp
    assert tr.sim.engine.plan.peak_non_model_bytes >= max(v for _, v in
                                                          tracer.history[:n_moments])
    assert any(t.reason in ("evict", "adam_copy") for r in tr.reports for t in r.transfers)
    values = list(tracer.history)

    def replay(m):
        mm, v = values.pop(0)
        assert mm == m
        return v

    sim = Simulator(schema, hw, PolicySpec(**c["policy"]), non_model_fn=replay)
    run = sim.run(3)
    assert not values
    for mine, ref in zip(tr.reports, run.reports):
        assert _ledger(mine) == _ledger(ref)


def test_cpu_placed_embedding_trains_like_gpu_placed():
    """Device-aware embedding placement (`profiler.py:70-74`): the CPU-placed
    operator (host lookup, activation H2D, gradient D2H, host scatter-add and
    host Adam; weights never in HBM) trains the same model as the GPU-placed
    one, bit for bit: the host and device operators sum gradients in the same
    order and the host Adam is K1's arithmetic (deterministic attention)."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_cap256Ki"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 5)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for place in ("cpu", "gpu"):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, embedding_placement=place,
                              untied_head=True)
            out[place] = ([tr.step_host(t) for t in toks], tr)
    cpu, gpu = out["cpu"][1], out["gpu"][1]
    assert cpu.host_embedding is not None and gpu.host_embedding is None
    assert cpu.model.wte.numel() == 0            # no embedding weights in HBM
    assert len(cpu.executor.embedding) == 1 and len(gpu.executor.embedding) == 3
    assert out["cpu"][0] == out["gpu"][0]
    he = cpu.host_embedding
    assert torch.equal(he.wte.view(torch.int16), gpu.model.wte.detach().cpu().view(torch.int16))
    assert torch.equal(he.wpe.view(torch.int16), gpu.model.wpe.detach().cpu().view(torch.int16))
    # every step moved B*S*H fp16 down and up, nothing else for the embedding
    u = schema.batch * schema.seq_len * schema.hidden_dim * 2
    assert he.h2d_bytes == he.d2h_bytes == u * len(toks)


def test_cpu_embedding_with_device_tokens():
    """step() with device-resident tokens (one small D2H of the token ids)
    equals step_host() with host tokens."""
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_cap1Mi"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 3)
    runs = []
    for dev in (False, True):
        tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                          dtype=torch.float16, seed=0, untied_head=True)
        assert tr.host_embedding is not None
        if dev:
            runs.append([float(tr.step(t.cuda()).item()) for t in toks])
        else:
            runs.append([tr.step_host(t) for t in toks])
    assert runs[0][0] == runs[1][0]
    np.testing.assert_allclose(runs[0], runs[1], rtol=1e-3)


def test_one_k1_launch_per_all_resident_step():
    """All GPU-placed positions (+ the non-chunked GPU parameters) are
    updated by ONE K1 launch per step — dropping stale host copies at ADAM
    (note_write) must not split the batch."""
    tr, schema = _trainer("tiny_cap1Mi")
    toks = _tokens(schema, 3)
    tr.step_host(toks[0])
    ex = tr.executor
    ex.record_k1 = True
    for t in toks[1:]:
        n0 = len(ex.k1_events)
        tr.step_host(t)
        assert len(ex.k1_events) == n0 + 1
    ex.record_k1 = False


@pytest.mark.parametrize("case", ["tiny_tight", "tiny_os_cpu"])
def test_async_host_adam_matches_synchronous(case):
    """Host Adam of CPU-placed positions on the worker thread (overlapping
    the rest of the step and the next forward, its adam_copy H2D issued by
    the worker) gives the synchronous run's bits, ledgers and moved bytes."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES[case]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 4)
    runs = {}
    with sdpa_kernel(SDPBackend.MATH):
        for async_adam in (False, True):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, async_host_adam=async_adam)
            losses = [tr.step_host(t) for t in toks]
            tr.finish_host_work()
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            st = tr.executor.stats
            runs[async_adam] = (losses, params, [_ledger(r)["transfers"] for r in tr.reports],
                                (st.h2d_bytes - st.prefetch_discarded_bytes, st.d2h_bytes),
                                st.host_adam_items)
    assert runs[True][4] > 0
    assert runs[True][0] == runs[False][0]
    for a, b in zip(runs[True][1], runs[False][1]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert runs[True][2] == runs[False][2] and runs[True][3] == runs[False][3]


def test_reference_criterion_06_volume_identity_on_the_real_step():
    """The reference's acceptance criterion 6 (`tests/test_acceptance.py:277-308`,
    chunk half) on the REAL step: with no GPU margin for optimizer state the
    chunk strategy moves exactly 4 bytes per parameter per measured iteration
    (fp16 grads down + updated fp16 params up) — and the executor physically
    moves exactly those chunk bytes; with a roomy GPU, ADAM moves nothing."""
    from paper_2108_05818_b200.trainer import ChunkTrainer
    schema = build_gpt_schema(layers=3, hidden_dim=64, heads=4, seq_len=32, vocab=100, batch=2,
                              context_bytes=500_000)
    toks = _tokens(schema, 4)
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=16384, os_placement="cpu"),
                      HardwareSpec(gpu_count=1, gpu_bytes=3_000_000, cpu_bytes=20_000_000),
                      dtype=torch.float16, seed=0)
    assert tr.sim.chunk_set.waste_elems == 0
    tr.step_host(toks[0])
    tr.finish_host_work()
    st, he = tr.executor.stats, tr.host_embedding
    moved0 = (st.h2d_bytes - st.prefetch_discarded_bytes + st.d2h_bytes
              + (he.h2d_bytes + he.d2h_bytes if he is not None else 0))
    for t in toks[1:]:
        tr.step_host(t)
    tr.finish_host_work()
    moved = (st.h2d_bytes - st.prefetch_discarded_bytes + st.d2h_bytes
             + (he.h2d_bytes + he.d2h_bytes if he is not None else 0)) - moved0
    assert tr.sim.engine.plan.os_positions_on_gpu == ()
    for r in tr.reports[1:]:
        assert r.feasible and r.pcie_bytes == 4 * schema.param_count
    # physically moved = billed, except the GPU-placed embedding's weight
    # round trip, which stays resident in HBM (accounting-only)
    emb = sum(t.bytes for r in tr.reports[1:] for t in r.transfers if t.chunk_id == "embedding")
    assert tr.embedding_placement == "gpu" and he is None
    assert moved == sum(r.pcie_bytes for r in tr.reports[1:]) - emb
    roomy = ChunkTrainer(schema, PolicySpec(capacity_elems=16384),
                         HardwareSpec(gpu_count=1, gpu_bytes=50_000_000, cpu_bytes=50_000_000),
                         dtype=torch.float16, seed=0)
    for t in toks[:3]:
        roomy.step_host(t)
    assert len(roomy.sim.engine.plan.os_positions_on_gpu) == roomy.sim.chunk_set.positions
    for r in roomy.reports[1:]:
        assert sum(t.bytes for t in r.transfers if t.reason == "adam_copy") == 0


@pytest.mark.parametrize("ckpt,dtype", [(True, torch.float16), (False, torch.bfloat16)])
def test_cuda_graph_replay_with_checkpointing_and_bf16(ckpt, dtype):
    """Graph replay of the steady state also covers the recomputing
    (activation-checkpointed) step and bf16 chunks: bit-identical to eager."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_cap256Ki"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 7)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for graph in (False, True):
            tr = ChunkTrainer(schema, PolicySpec(**dict(c["policy"], checkpointing=ckpt)),
                              HardwareSpec(**c["hardware"]), dtype=dtype, seed=0,
                              cuda_graph=graph, embedding_placement="gpu")
            losses = [tr.step_host(t) for t in toks]
            out[graph] = (losses, [tr.local_chunk_payload(p).cpu().clone()
                                   for p in range(tr.sim.chunk_set.positions)], tr)
    assert out[True][2]._graph is not None
    assert out[True][0] == out[False][0]
    for a, b in zip(out[True][1], out[False][1]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("case,graph", [("tiny_cap256Ki", False), ("tiny_tight", False),
                                        ("tiny_cap256Ki", True)])
def test_overflow_steps_are_skipped_without_touching_the_model(case, graph):
    """Dynamic loss scaling from an absurd scale: the first steps overflow and
    are skipped.  A skipped step must leave the model exactly as it was —
    the fp16 chunks, which hold the step's gradients under the grad
    overwrite, get their parameters back — so the same batch gives the same
    loss until the scale has backed off, and training then proceeds."""
    from paper_2108_05818_b200.chunks import ChunkKind
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES[case]
    schema = build_gpt_schema(**c["schema"])
    kw = dict(cuda_graph=True, embedding_placement="gpu") if graph else {}
    tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                      dtype=torch.float16, seed=0, init_loss_scale=2.0 ** 26,
                      dynamic_loss_scale=True, **kw)
    batch = _tokens(schema, 1)[0]
    losses = [tr.step_host(batch) for _ in range(16)]
    if graph:  # captured while still overflowing: the skip decision is on the device
        assert tr._graph is not None
    tr.finish_host_work()
    st = tr.step_state()
    skipped = 16 - int(st.step)
    assert 2 <= skipped < 16 and st.loss_scale < 2.0 ** 26, (skipped, st.loss_scale)
    assert all(np.isfinite(losses)), losses
    assert len(set(losses[:skipped])) == 1, losses[:skipped + 1]   # the model did not move
    assert losses[-1] < losses[0]
    for pos in range(tr.sim.chunk_set.positions):                  # p16 == round(p32)
        n = tr.sim.chunk_set.param_chunk(pos).used_elems
        p16 = tr.local_chunk_payload(pos)[:n].cpu()
        p32 = tr.local_chunk_payload(pos, ChunkKind.PARAM_FP32)[:n].cpu()
        assert torch.equal(p16, p32.half())


def test_gradient_clipping_in_the_real_step():
    """max_grad_norm > 0: the device step scalars carry the global norm and
    grad_scale = clip / loss_scale with clip = max_norm / norm (torch's
    clip_grad_norm_ coefficient, eps 1e-6), and every K1 launch of the step
    still matches the oracle bit for bit."""
    from oracle import step_check
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                      dtype=torch.float16, seed=0, max_grad_norm=1e-3)
    toks = _tokens(schema, 3)
    tr.step_host(toks[0])
    rec = step_check.arm(tr)
    for t in toks[1:]:
        assert np.isfinite(tr.step_host(t))
    step_check.disarm(tr)
    tr.finish_host_work()
    st = tr.step_state()
    assert st.grad_norm > 1e-3 and rec["checked"] > 0 and rec["mismatch"] == []
    clip = 1e-3 / (st.grad_norm + 1e-6)
    assert abs(st.grad_scale * st.loss_scale - clip) <= 1e-6 * clip


@pytest.mark.parametrize("place", ["cpu", "gpu"])
def test_unfused_model_trains_like_fused(place):
    """fused_ops=False (plain torch LayerNorm / GELU / embedding / loss, and
    autograd gradients packed over the non-chunked parameters by K3 at ADAM)
    through the same chunk-managed step: same ledgers as the fused model and
    losses within fp16 tolerance."""
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 4)
    out = {}
    for fused in (True, False):
        tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                          dtype=torch.float16, seed=0, fused_ops=fused,
                          embedding_placement=place, untied_head=True)
        out[fused] = ([tr.step_host(t) for t in toks], [_ledger(r)["transfers"] for r in tr.reports])
    assert out[True][1] == out[False][1]
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=2e-3)


def test_tied_model_under_a_cpu_embedding_plan_computes_it_on_the_gpu():
    """The untied LM head is an explicit opt-in (the batch size must not
    change the model): a tied model whose plan says CPU (C1) computes the
    embedding on the GPU, warns, still produces the reference's ledgers, and
    reports the embedding rows as billed but not realized."""
    import warnings
    case = "tiny_cap256Ki"
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        tr, schema = _trainer(case, untied_head=False)
    assert any("untied LM head" in str(x.message) for x in w)
    assert tr.sim.engine.embedding_device == "cpu" and tr.embedding_placement == "gpu"
    assert tr.host_embedding is None and not tr.untied_head
    ref = CASES[case]["ranks"]["0"]
    for t in _tokens(schema, 3):
        tr.step_host(t)
    for mine, theirs in zip(tr.reports, ref["iterations"]):
        assert _ledger(mine)["transfers"] == theirs["transfers"]
    emb = sum(t.bytes for t in tr.reports[-1].transfers if t.chunk_id == "embedding")
    assert emb > 0 and tr.ledger_rows_not_realized() == {"embedding": emb}
    assert tr.gpu_resident_bytes == 14 * (schema.vocab + schema.seq_len) * schema.hidden_dim
    import pytest as _pt
    with _pt.raises(ValueError, match="untied"):
        from paper_2108_05818_b200.trainer import ChunkTrainer
        c = CASES[case]
        ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                     embedding_placement="cpu")


@pytest.mark.parametrize("emb", ["gpu", "cpu"])
def test_clipped_training_is_placement_invariant(emb):
    """With max_grad_norm > 0 the clip coefficient comes from the global sum
    of squares, which K2 and its host twin evaluate in one canonical order
    whatever lives where: a tight-budget run (chunks evicted, optimizer state
    and gradients of some positions in host DRAM) and an all-resident run --
    and a CPU-placed embedding (host gradients) -- give bit-identical losses,
    norms and parameters."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 5)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for name, hw in (("tight", HardwareSpec(**c["hardware"])),
                         ("resident", HardwareSpec(gpu_count=1, gpu_bytes=180 * 10 ** 9))):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), hw, dtype=torch.float16,
                              seed=0, max_grad_norm=1e-3, embedding_placement=emb,
                              untied_head=True)
            losses, norms = [], []
            for t in toks:
                losses.append(tr.step_host(t))
                tr.finish_host_work()
                norms.append(tr.step_state().grad_norm)
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            out[name] = (losses, norms, params, tr)
    (l0, n0, p0, tight), (l1, n1, p1, _) = out["tight"], out["resident"]
    assert tight.executor.stats.copies > 0 and tight.executor.stats.host_adam_items > 0
    assert n0 == n1 and all(n > 1e-3 for n in n0)   # clipping engaged at every step
    assert l0 == l1
    for a, b in zip(p0, p1):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_clipped_training_cpu_and_gpu_embedding_agree():
    """Clipped training with the embedding on the CPU (host operator, host
    gradients summed by K2's host twin) and on the GPU (device operator,
    gradients summed by K2): bit-identical losses, norms and parameters."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 4)
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for place in ("cpu", "gpu"):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, max_grad_norm=1e-3,
                              embedding_placement=place, untied_head=True)
            losses, norms = [], []
            for t in toks:
                losses.append(tr.step_host(t))
                tr.finish_host_work()
                norms.append(tr.step_state().grad_norm)
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            out[place] = (losses, norms, params)
    assert out["cpu"][0] == out["gpu"][0] and out["cpu"][1] == out["gpu"][1]
    for a, b in zip(out["cpu"][2], out["gpu"][2]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_nvtx_ranges_do_not_change_the_step():
    """CS_NVTX=1 brackets every timeline event, chunk move and collective in
    an NVTX range (host-side markers): an evicting run with them gives the
    same losses and ledgers."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CASES["tiny_tight"]
    schema = build_gpt_schema(**c["schema"])
    toks = _tokens(schema, 3)
    out = []
    with sdpa_kernel(SDPBackend.MATH):
        for nvtx in (False, True):
            tr = ChunkTrainer(schema, PolicySpec(**c["policy"]), HardwareSpec(**c["hardware"]),
                              dtype=torch.float16, seed=0, untied_head=True)
            tr.nvtx = tr.executor.nvtx = nvtx
            losses = [tr.step_host(t) for t in toks]
            out.append((losses, [_ledger(r)["transfers"] for r in tr.reports]))
    assert out[0] == out[1]
