"""Cross-process determinism probe: print the first losses of a small run."""
import sys, torch
sys.path.insert(0, '.')
from torch.nn.attention import SDPBackend, sdpa_kernel
from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200.config import PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.trainer import ChunkTrainer
place = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "host"
schema = build_gpt_schema(layers=4, hidden_dim=1024, heads=8, seq_len=512, vocab=50304, batch=16)
g = torch.Generator().manual_seed(5)
toks = [torch.randint(0, 50304, (16, 513), generator=g) for _ in range(3)]
with sdpa_kernel(SDPBackend.MATH):
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=4 << 20), seed=0,
                      hyper=K.AdamHyper(lr=3e-4, betas=(0.9, 0.95)), embedding_placement=place,
                      untied_head=True)
    if mode == "host":
        print(place, mode, [repr(tr.step_host(t)) for t in toks])
    else:
        print(place, mode, [repr(float(tr.step(t.cuda()).item())) for t in toks])
