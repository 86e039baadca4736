import sys, torch
sys.path.insert(0, '.')
from torch.nn.attention import SDPBackend, sdpa_kernel
from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200.chunks import ChunkKind
from paper_2108_05818_b200.config import PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.trainer import ChunkTrainer
schema = build_gpt_schema(layers=4, hidden_dim=1024, heads=8, seq_len=512, vocab=50304, batch=16)
g = torch.Generator().manual_seed(5)
toks = [torch.randint(0, 50304, (16, 513), generator=g) for _ in range(3)]
res = {}
with sdpa_kernel(SDPBackend.MATH):
    for os_pl in ("auto", "cpu"):
        for asy in ((False, True) if os_pl == "cpu" else (False,)):
            tr = ChunkTrainer(schema, PolicySpec(capacity_elems=4 << 20, os_placement=os_pl), seed=0,
                              hyper=K.AdamHyper(lr=3e-4, betas=(0.9, 0.95)), async_host_adam=asy)
            out = []
            mode = sys.argv[1] if len(sys.argv) > 1 else "host"
            for t in toks:
                if mode == "host":
                    out.append(tr.step_host(t))
                    tr.finish_host_work()
                else:  # device tokens, no join between steps (the demo's loop)
                    out.append(float(tr.step(t.cuda()).item()))
            tr.finish_host_work()
            p32 = [tr.local_chunk_payload(p, ChunkKind.PARAM_FP32).cpu().clone() for p in range(tr.sim.chunk_set.positions)]
            p16 = [tr.local_chunk_payload(p).cpu().clone() for p in range(tr.sim.chunk_set.positions)]
            he = tr.host_embedding
            emb = he.wte.clone() if he is not None else None
            res[(os_pl, asy)] = (out, p32, p16, emb, tr.embedding_placement)
            print(os_pl, asy, out, tr.embedding_placement, tr.executor.stats.host_adam_items, flush=True)
            del tr
base = res[("auto", False)]
for k, v in res.items():
    d32 = [float((a - b).abs().max()) for a, b in zip(v[1], base[1])]
    d16 = [int((a.view(torch.int16) != b.view(torch.int16)).sum()) for a, b in zip(v[2], base[2])]
    de = None if v[3] is None else int((v[3].view(torch.int16) != base[3].view(torch.int16)).sum())
    print(k, 'loss eq', v[0] == base[0], 'p32 maxdiff per pos', d32, 'p16 ndiff', d16, 'emb ndiff', de)
