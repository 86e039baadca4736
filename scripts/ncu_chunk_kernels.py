"""One launch of each chunk kernel at 2^28 elements (K1..K6), for
`ncu --set full` (profiles/r01/chunk_kernels_ncu.md)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2108_05818_b200 import kernels as K

n = 1 << 28
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
p16 = (torch.randn(n, device=dev, generator=g) * 1e-3).half()
p32 = torch.randn(n, device=dev, generator=g) * 0.02
m = torch.zeros(n, device=dev)
v = torch.zeros(n, device=dev)
src16 = torch.randn(n, device=dev, generator=g).half()
src32 = torch.randn(n, device=dev, generator=g)
hyper = K.AdamHyper(lr=1e-4)
state = K.StepState(dev)
state.sumsq().fill_(1.0)
K.adam_prepare(state, hyper)
scratch = torch.empty(K.sumsq_scratch([(p16, n)]), device=dev)
item_sums = torch.empty(1, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
K.adam_chunks([(p16, p32, m, v, n)], hyper, state)                  # K1
K.grad_sumsq([(p16, n)], scratch, item_sums)                          # K2
K.pack([(p16, 0, src16, n)])                                         # K3
K.pack([(p16, 0, src16, n)], accumulate=True)                        # K4
K.cast_pack([(p16, 0, src32, n)])                                    # K5
K.master_init(p32, m, v, p16, n)                                     # K6
torch.cuda.synchronize()
print("ok")
