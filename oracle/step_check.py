"""Check the fused Adam inside a REAL chunk-managed step against the C oracle.
TEST INFRASTRUCTURE ONLY (tests/ and __graft_entry__.smoke()).

Installs an observer on the trainer's executor: before the K1 launch the
gradient (fp16 chunk), master, momentum and variance prefixes and the step
scalars are copied to the host; after it the outputs are copied back; the
oracle replays the update on the host copies and every byte must match.
"""

import numpy as np
import torch

from . import numerics as O


def arm(trainer):
    record = {"checked": 0, "elements": 0, "mismatch": []}
    ex = trainer.executor
    code = O.FP16 if trainer.dtype == torch.float16 else O.BF16
    snap = {}

    def observer(phase, items):
        torch.cuda.synchronize()
        if phase == "pre":
            snap["state"] = ex.state.read()
            snap["items"] = [(p16[:n].cpu().view(torch.int16).numpy().view(np.uint16).copy(),
                              p32[:n].cpu().numpy().copy(), m[:n].cpu().numpy().copy(),
                              v[:n].cpu().numpy().copy(), n) for p16, p32, m, v, n in items]
            return
        st = snap["state"]
        s = O.OrStepState()
        for f, _ in s._fields_:
            setattr(s, f, getattr(st, f))
        h = trainer.hyper
        for (g, p, m, v, n), (d16, d32, dm, dv, _) in zip(snap["items"], items):
            O.adam(g, p, m, v, n, code, h.lr, h.betas[0], h.betas[1], h.eps, h.weight_decay,
                   h.adamw, s, 8)
            ok = (np.array_equal(d32[:n].cpu().numpy().view(np.uint32), p.view(np.uint32)) and
                  np.array_equal(dm[:n].cpu().numpy().view(np.uint32), m.view(np.uint32)) and
                  np.array_equal(dv[:n].cpu().numpy().view(np.uint32), v.view(np.uint32)) and
                  np.array_equal(d16[:n].cpu().view(torch.int16).numpy().view(np.uint16), g))
            record["checked"] += 1
            record["elements"] += n
            if not ok:
                record["mismatch"].append(n)

    ex.adam_observer = observer
    return record


def disarm(trainer):
    trainer.executor.adam_observer = None
