"""Freeze torch.optim.Adam/AdamW (CPU, fp32) trajectories as golden vectors.

Pins the C oracle's Adam (oracle/cs_oracle.c) to the published algorithm:
the reference itself has no numerics.  Gradients are fp16
values (the chunk step reads fp16 grads and widens them), params fp32.
Run from the repo root:  python tests/golden/gen_adam_golden.py
"""

import os

import numpy as np
import torch

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "adam_torch.npz")
N, STEPS = 4099, 5  # odd size: exercises the non-multiple-of-8 tail
CASES = {
    "adam": dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0, adamw=False),
    "adam_l2": dict(lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1, adamw=False),
    "adamw": dict(lr=3e-4, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.01, adamw=True),
}


def main() -> None:
    g = torch.Generator().manual_seed(2108_05818)
    out = {}
    for name, hp in CASES.items():
        p0 = (torch.randn(N, generator=g) * 0.02).float()
        grads16 = [(torch.randn(N, generator=g) * 10 ** float(torch.empty(1).uniform_(-4, 0, generator=g)))
                   .half() for _ in range(STEPS)]
        p = torch.nn.Parameter(p0.clone())
        kw = dict(lr=hp["lr"], betas=hp["betas"], eps=hp["eps"], weight_decay=hp["weight_decay"],
                  foreach=False, fused=False)
        opt = (torch.optim.AdamW if hp["adamw"] else torch.optim.Adam)([p], **kw)
        traj_p, traj_m, traj_v = [], [], []
        for t in range(STEPS):
            p.grad = grads16[t].float()
            opt.step()
            st = opt.state[p]
            traj_p.append(p.detach().clone().numpy())
            traj_m.append(st["exp_avg"].clone().numpy())
            traj_v.append(st["exp_avg_sq"].clone().numpy())
        out[name + "/p0"] = p0.numpy()
        out[name + "/g16"] = np.stack([x.numpy().view(np.uint16) for x in grads16])
        out[name + "/p"] = np.stack(traj_p)
        out[name + "/m"] = np.stack(traj_m)
        out[name + "/v"] = np.stack(traj_v)
        out[name + "/hyper"] = np.array([hp["lr"], hp["betas"][0], hp["betas"][1], hp["eps"],
                                         hp["weight_decay"], float(hp["adamw"])], np.float64)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, "torch", torch.__version__)


if __name__ == "__main__":
    main()
