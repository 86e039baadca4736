"""Which Python lines issue the step's device-to-device memcpys?"""
import sys
sys.path.insert(0, '.')
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200.config import PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.trainer import ChunkTrainer
schema = build_gpt_schema(layers=2, hidden_dim=2048, heads=16, seq_len=1024, vocab=50304, batch=32)
tr = ChunkTrainer(schema, PolicySpec(capacity_elems=64 << 20), seed=0, hyper=K.AdamHyper(lr=1e-4))
tok = torch.randint(0, 50304, (32, 1025)).cuda()
for _ in range(3):
    tr.step(tok)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True, record_shapes=True) as prof:
    tr.step(tok)
    torch.cuda.synchronize()
for ev in prof.key_averages(group_by_input_shape=True):
    if ev.key in ("aten::copy_", "aten::clone", "aten::contiguous", "aten::_to_copy") and ev.count:
        print(ev.key, ev.count, "dev_us", round(getattr(ev, "device_time_total", 0), 1), ev.input_shapes)
for e in prof.events():
    if "Memcpy" in e.name and e.device_type == torch.autograd.DeviceType.CUDA:
        print("DEV", e.name, round(e.time_range.elapsed_us(), 1))
