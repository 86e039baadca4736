import time, numpy as np, torch, os, subprocess
print(subprocess.run("lscpu | grep -E 'Model name|Flags|NUMA|Socket|Core|Thread'", shell=True, capture_output=True, text=True).stdout[:1500])
n = 1 << 28
a = torch.empty(n, dtype=torch.float32).normal_()
b = torch.empty_like(a)
torch.set_num_threads(16)
for _ in range(2): b.copy_(a)
t = time.perf_counter()
for _ in range(5): b.copy_(a)
dt = (time.perf_counter() - t) / 5
print("torch copy 1 GiB fp32: %.1f GB/s (read+write)" % (2 * n * 4 / dt / 1e9))
