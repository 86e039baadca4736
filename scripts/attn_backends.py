"""A/B of torch SDPA backends for the 1B step's attention (B=32, 16 heads,
S=1024, D=128, causal, fp16): forward + backward time per layer."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, Hh, S, D = 32, 16, 1024, 128
q, k, v = (torch.randn(B, Hh, S, D, device="cuda", dtype=torch.float16, requires_grad=True)
           for _ in range(3))
do = torch.randn(B, Hh, S, D, device="cuda", dtype=torch.float16)
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    try:
        with sdpa_kernel(be):
            for _ in range(3):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                o.backward(do)
            torch.cuda.synchronize()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            for _ in range(10):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            b.record()
            for _ in range(10):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                o.backward(do)
            c.record()
            torch.cuda.synchronize()
            f = a.elapsed_time(b) / 10
            fb = b.elapsed_time(c) / 10
            fl = 4 * B * Hh * S * S * D / 2
            print("%-22s fwd %.3f ms (%.0f TF/s)  fwd+bwd %.3f ms (%.0f TF/s)"
                  % (be.name, f, fl / f / 1e9, fb, 3.5 * fl / fb / 1e9))
    except Exception as e:
        print(be.name, "unavailable:", repr(e)[:150])
