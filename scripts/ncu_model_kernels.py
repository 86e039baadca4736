"""One launch of each model-side kernel of this library at the bench shape
(1B GPT, B=32, S=1024, H=2048, V=50304), for `ncu --set full`
(profiles/r01/model_kernels_ncu.md).  Algorithmic bytes per launch are
printed so the summary can divide them by ncu's duration."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2108_05818_b200 import kernels as K  # noqa: E402

B, S, H, V = 32, 1024, 2048, 50304
rows = B * S
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(rows, H, device=dev, generator=g).half()
dy = torch.randn(rows, H, device=dev, generator=g).half()
dres = torch.randn(rows, H, device=dev, generator=g).half()
tok = torch.randint(0, V, (B, S), device=dev, generator=g)
wte = (torch.randn(V, H, device=dev, generator=g) * 0.02).half()
wpe = (torch.randn(S, H, device=dev, generator=g) * 0.02).half()
logits = torch.randn(rows, V, device=dev, generator=g).half()
tgt = torch.randint(0, V, (rows,), device=dev, generator=g)
torch.cuda.synchronize()

y, mean, rstd = K.layernorm_fwd(x)
dx = K.layernorm_bwd(dy, x, mean, rstd, dres)
loss, lse = K.xent_fwd(logits, tgt)
K.xent_bwd_(logits, tgt, lse, torch.ones((), device=dev), 1.0 / rows)
emb = K.embed_fwd(tok, wte, wpe)
K.embed_bwd_into(tok, emb, wte, wpe, accumulate=True)
torch.cuda.synchronize()

E = rows * H
hit = int(torch.unique(tok).numel())
print(json.dumps({
    "ln_fwd_kernel": {"bytes": E * 4 + rows * 8, "what": "x read + y write (2+2 B/elem) + mean/rstd"},
    "ln_bwd_row_kernel": {"bytes": E * 8 + rows * 8,
                          "what": "dy, x, residual grad read + dx write (8 B/elem) + mean/rstd"},
    "xent_fwd_kernel": {"bytes": rows * V * 2 + rows * 16, "what": "logits read once (2 B/elem)"},
    "xent_bwd_kernel": {"bytes": rows * V * 4 + rows * 16,
                        "what": "logits read + gradient written in place (4 B/elem)"},
    "embed_fwd_kernel": {"bytes": E * 6 + rows * 8,
                         "what": "wte row + wpe row read, output written (6 B/elem of B*S*H)"},
    "embed_bwd_kernel": {"bytes": E * 2 + hit * H * 4 + S * H * 2 + rows * 16,
                         "what": "dout read once + the %d hit gwte rows read-modify-written "
                                 "(accumulate) + gwpe written" % hit},
}))
