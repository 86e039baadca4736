"""Do the step's per-layer D2D memcpys come from cuDNN SDPA (q/k/v layout)?"""
import torch, torch.nn.functional as F
from torch.profiler import profile, ProfilerActivity
B, S, H, nh = 32, 1024, 2048, 16
D = H // nh
def run(layout):
    x = [torch.randn(B, S, H, device="cuda", dtype=torch.float16, requires_grad=True) for _ in range(3)]
    if layout == "bshd":
        q, k, v = (t.view(B, S, nh, D).transpose(1, 2) for t in x)
    else:
        q, k, v = (t.view(B, S, nh, D).transpose(1, 2).contiguous() for t in x)
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    out = o.transpose(1, 2).reshape(B, S, H)
    g = torch.randn_like(out)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        out = o.transpose(1, 2).reshape(B, S, H)
        out.backward(g)
        torch.cuda.synchronize()
    n = [e for e in prof.events() if "Memcpy DtoD" in e.name]
    k_ = [e.name[:50] for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name]
    print(layout, "memcpy DtoD:", len(n), "kernels:", k_)
run("bshd")
run("bhsd")
