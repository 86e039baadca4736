"""The reference's GPU-computed embedding branch, realised
(`engine.py:214-219`: weights down at FWD, weight gradients up at BWD; the
weights live in host memory, `scenario.py:133`).

``ChunkTrainer(embedding_weights="host")``: the wte fp16 weights (the V x H
allocation the reference bills), its fp32 master and Adam moments in pinned
host DRAM; the GPU operator and the tied LM head read an HBM copy; each step
one D2H of the weight gradient and, after the host Adam, one H2D of the new
weights (the positional table is not billed and stays in HBM).  Checked
against the default
(state resident in HBM, updated by K1): the same ledgers, bit-identical
losses, chunk parameters and embedding weights, and physically moved bytes
equal to the ledger's embedding rows (which the default does not realise).
"""

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

from paper_2108_05818_b200.config import HardwareSpec, PolicySpec  # noqa: E402
from paper_2108_05818_b200.model import build_gpt_schema  # noqa: E402


def _rows(r):
    return ([(t.moment, t.chunk_id, t.src, t.dst, t.bytes, t.reason) for t in r.transfers],
            [(c.iteration, c.group_id, c.kind, c.bytes) for c in r.collectives],
            [(s.moment, s.device, s.used_bytes, s.chunk_bytes, s.non_model_bytes)
             for s in r.samples])


@pytest.mark.parametrize("dtype,budget,os_placement", [
    (torch.float16, 8 << 30, "auto"),
    (torch.bfloat16, 8 << 30, "cpu"),
    (torch.float16, None, "auto"),  # tight: evictions beside the embedding round trip
])
def test_host_weights_embedding_matches_resident(dtype, budget, os_placement):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from paper_2108_05818_b200.profiler import embedding_compute_device
    from paper_2108_05818_b200.scenario import Simulator
    from paper_2108_05818_b200.trainer import ChunkTrainer
    schema = build_gpt_schema(layers=3, hidden_dim=128, heads=4, seq_len=64, vocab=512,
                              batch=4, context_bytes=1 << 20)
    assert embedding_compute_device(schema) == "gpu"  # V <= 2*B*S: the GPU branch
    policy = PolicySpec(capacity_elems=1 << 16, os_placement=os_placement)
    if budget is None:  # just above the smallest feasible accounting budget
        lo, hi = 1 << 20, 1 << 32
        while hi - lo > (64 << 10):
            mid = (lo + hi) // 2
            ok = Simulator(schema, HardwareSpec(gpu_count=1, gpu_bytes=mid), policy).run(3)
            lo, hi = (lo, mid) if ok.feasible else (mid, hi)
        budget = int(hi * 1.1)
    g = torch.Generator().manual_seed(5)
    toks = [torch.randint(0, schema.vocab, (schema.batch, schema.seq_len + 1), generator=g)
            for _ in range(5)]
    out = {}
    with sdpa_kernel(SDPBackend.MATH):
        for weights in ("hbm", "host"):
            tr = ChunkTrainer(schema, policy, HardwareSpec(gpu_count=1, gpu_bytes=budget),
                              dtype=dtype, seed=0, embedding_weights=weights)
            losses = [tr.step_host(t) for t in toks]
            tr.finish_host_work()
            torch.cuda.synchronize()
            params = [tr.local_chunk_payload(p).cpu().clone()
                      for p in range(tr.sim.chunk_set.positions)]
            emb = [p.detach().cpu().clone() for p in tr.model.embedding_parameters()]
            out[weights] = (losses, params, emb, tr)
    (l0, p0, e0, hbm), (l1, p1, e1, host) = out["hbm"], out["host"]
    assert l0 == l1
    for a, b in zip(p0 + e0, p1 + e1):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    for a, b in zip(hbm.reports, host.reports):
        assert _rows(a) == _rows(b)
    he = host.host_embedding
    assert he is not None and he.device_compute and hbm.host_embedding is None
    # K1 updates only wpe in the realised mode; the host copy of wte is the
    # state: the last H2D carried exactly the host weights
    assert len(host.executor.embedding) == 1 and len(hbm.executor.embedding) == 2  # wpe stays
    assert torch.equal(he.wte.view(torch.int16), e1[0].view(torch.int16))
    rows = [t for r in host.reports for t in r.transfers if t.chunk_id == "embedding"]
    assert he.h2d_bytes == sum(t.bytes for t in rows if t.src == "cpu") > 0
    assert he.d2h_bytes == sum(t.bytes for t in rows if t.src == "gpu") > 0
    assert host.ledger_rows_not_realized() == {}
    assert hbm.ledger_rows_not_realized() == {"embedding": sum(
        t.bytes for t in hbm.reports[-1].transfers if t.chunk_id == "embedding")}
    # HBM charged for the weights only, not their optimizer state
    V, S, H = schema.vocab, schema.seq_len, schema.hidden_dim
    assert host.gpu_resident_bytes == V * H * 2 + S * H * 14
    assert hbm.gpu_resident_bytes == (V + S) * H * 14
