"""Real warm-up memory tracer: measured non-model footprint R - C per moment.

PatrickStar §5 profiles the first iteration: at every moment it samples the
device memory in use R and the bytes held by chunks C; R - C is the
non-model footprint (activations, workspaces, the non-chunked embedding)
that decides how much HBM the chunk manager may use and the placement plan's
margin.  The reference models R - C analytically (`cs/model.py:332-345`) and
feeds it to the engine through ``non_model_fn`` (`cs/engine.py:68,77-83,
147-148`); its samples land in ``WarmupStats`` (`cs/profiler.py:28-57`).

Here ``non_model_fn`` is this object:

* during the warm-up it returns the LIVE measurement at the moment the
  engine asks: ``torch.cuda.memory_allocated`` (relative to the process's
  allocation when the run was built) minus the physical bytes of
  every chunk payload on the device (payloads, group slabs, prefetches,
  retained buffers).  The engine asks for moment 2i+1 when event i starts
  and for 2i+2 when it finishes, so the placement plan computed at the
  warm-up's ADAM sees the measured peak;
* :meth:`freeze` then fixes the curve for the measured iterations: the
  during-event moment takes the larger of the event's two readings (the
  operator's outputs exist by its end), boundary moments keep their reading.

The engine's BWD grad staging charge (``param_bytes``) is accounted
separately; physically the gradient is written straight into the chunk slot,
so R - C contains no grad temp and nothing is counted twice.
"""

from typing import Dict, List, Tuple

import torch

from .model import GPU


class MemoryTracer:
    def __init__(self, executor, device: torch.device):
        self.executor = executor
        self.device = torch.device(device)
        # bytes owned by anything else in the process when this run started
        self.base = torch.cuda.memory_allocated(self.device)
        self.live: Dict[int, int] = {}
        self.curve: Dict[int, int] = {}
        self.history: List[Tuple[int, int]] = []  # (moment, value) in call order
        self.frozen = False

    def chunk_bytes(self) -> int:
        ex = self.executor
        seen = {}
        tensors = list(ex.payload[GPU].values()) + list(ex._group_slab.values())
        tensors += [t for t, _ in ex._prefetched.values()]
        tensors += [t for (cid, dev), t in ex._retained.items() if dev == GPU]
        tensors += ex.slabs.free_tensors()  # recycled chunk slabs are chunk memory
        for t in tensors:
            st = t.untyped_storage()
            seen[st.data_ptr()] = st.nbytes()
        return sum(seen.values())

    def measure(self) -> int:
        used = torch.cuda.memory_allocated(self.device) - self.base
        return max(0, used - self.chunk_bytes())

    def __call__(self, moment: int) -> int:
        if self.frozen:
            value = self.curve.get(moment, max(self.curve.values(), default=0))
        else:
            value = self.measure()
            self.live[moment] = max(self.live.get(moment, 0), value)
        self.history.append((moment, value))
        return value

    def freeze(self) -> None:
        """Fix the curve measured during the warm-up for later iterations."""
        curve = dict(self.live)
        for m, v in self.live.items():
            if m % 2 == 1:
                curve[m] = max(v, self.live.get(m + 1, 0))
        self.curve = curve
        self.frozen = True

    @property
    def peak(self) -> int:
        return max((self.curve or self.live).values(), default=0)
