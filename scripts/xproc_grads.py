"""Cross-process determinism probe on the Markov stream: hash of every K1
input (gradients, masters, moments) of the first two steps, and of the host
embedding gradients.  Run twice; diff the outputs."""
import hashlib, os, sys, torch
sys.path.insert(0, '.')
from torch.nn.attention import SDPBackend, sdpa_kernel
from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200.config import PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.trainer import ChunkTrainer

def h(t):
    return hashlib.md5(t.detach().contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:10]

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1234)
V, A = 50304, 2048
vocab_ids = torch.randperm(V, device=dev, generator=g)[:A]
table = torch.randint(0, A, (A, 4), device=dev, generator=g)
def batch():
    st = torch.empty(16, 513, dtype=torch.int64, device=dev)
    st[:, 0] = torch.randint(0, A, (16,), device=dev, generator=g)
    for t in range(512):
        st[:, t + 1] = table[st[:, t], torch.randint(0, 4, (16,), device=dev, generator=g)]
    return vocab_ids[st]
schema = build_gpt_schema(layers=4, hidden_dim=1024, heads=8, seq_len=512, vocab=V, batch=16)
mode = sys.argv[1] if len(sys.argv) > 1 else "math"
ctx = sdpa_kernel(SDPBackend.MATH) if mode == "math" else sdpa_kernel(SDPBackend.CUDNN_ATTENTION)
with ctx:
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=4 << 20), seed=0,
                      hyper=K.AdamHyper(lr=3e-4, betas=(0.9, 0.95)))
    ex = tr.executor
    log = []
    def obs(phase, items):
        if phase == "pre":
            torch.cuda.synchronize()
            log.append(" ".join(h(p16[:n]) for p16, p32, m, v, n in items))
    ex.adam_observer = obs
    for i in range(2):
        b = batch()
        loss = float(tr.step(b).item())
        he = tr.host_embedding
        print("step", i, repr(loss), "tok", h(b), "wte_host", h(he.wte) if he else None, flush=True)
    for i, l in enumerate(log):
        print("K1 grads step", i, l)
