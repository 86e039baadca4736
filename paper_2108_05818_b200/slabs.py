"""HBM slab pool for chunk payloads (the physical side of ``DevicePool``).

The reference charges every resident chunk its full capacity
(`chunks.py:99-102`) and its ``DevicePool`` (`memory.py:62-93`) only counts
bytes.  Physically, every chunk payload of a list has the same size
(cap x 2 B for fp16/bf16, cap x 4 B for fp32), so a chunk manager recycles
them whole: this pool hands out chunk slabs and takes them back when the
accounting drops a copy (evict, release, ``note_write``), so the evict /
fetch churn of an offloading run is served without going through the
caching allocator (whose out-of-memory path frees every cached block with a
device sync and retries).

Reuse is stream-ordered without host syncs: ``give`` records an event on
the compute stream and takes the completion events of the slab's last copy
on each side stream (the executor tracks them per slab), and ``take`` makes
the taking stream wait on them.  Events at the side streams' *tails* would
also be safe but make a taker wait for every unrelated copy queued there
(at ADAM the H2D stream holds the whole walk's fetches, after it the D2H
stream the pre-evictions).  Inside a CUDA-graph capture
the pool is bypassed (events recorded outside a capture cannot be waited on
inside it).

Two rules keep HBM shared with the model's activations:

* every slab comes from the COMPUTE stream's pool of the caching allocator
  (a miss taken for another stream makes that stream wait for the compute
  stream once).  Blocks allocated on a side stream can only ever be
  recycled by that stream, so H2D destinations allocated on the copy stream
  used to strand HBM the activations then could not use;
* at most ``max_free`` free slabs of each kind are kept; beyond that a
  dropped slab goes back to the caching allocator, because the accounting
  only drops chunk bytes when something else (activations) needs them.
"""

import os
from typing import Dict, List, Optional, Sequence, Tuple

import torch


class SlabPool:
    def __init__(self, device: torch.device, streams: Sequence[torch.cuda.Stream],
                 max_free: int = 4):
        self.device = torch.device(device)
        self.streams = list(streams)      # streams[0] allocates (the compute stream)
        self.max_free = max_free
        self.disabled = os.environ.get("CS_SLABS") == "0"  # A/B switch: plain allocator
        self._free: Dict[Tuple[torch.dtype, int], List[Tuple[torch.Tensor, list]]] = {}
        self._owned: Dict[int, Tuple[torch.dtype, int]] = {}
        self.allocs = 0      # slabs created (the pool's high-water mark)
        self.reuses = 0      # takes served from the free list
        self.gives = 0

    def take(self, numel: int, dtype: torch.dtype, stream: torch.cuda.Stream) -> torch.Tensor:
        """A slab of ``numel`` elements, safe to use on ``stream``."""
        if torch.cuda.is_current_stream_capturing() or self.disabled:
            with torch.cuda.stream(stream):  # (capture: the graph's private pool)
                return torch.empty(numel, dtype=dtype, device=self.device)
        key = (dtype, int(numel))
        lst = self._free.get(key)
        if lst:
            t, events = lst.pop()
            for ev in events:
                stream.wait_event(ev)
            self.reuses += 1
            return t
        home = self.streams[0]
        with torch.cuda.stream(home):
            t = torch.empty(numel, dtype=dtype, device=self.device)
        if stream is not home:  # the block is free in the compute stream's order only
            ev = torch.cuda.Event()
            ev.record(home)
            stream.wait_event(ev)
            # no record_stream: the side stream's use is handed back with the
            # slab (``give(side_events=...)``), which orders its eventual free
        self._owned[t.data_ptr()] = key
        self.allocs += 1
        return t

    def owns(self, t: torch.Tensor) -> bool:
        key = self._owned.get(t.data_ptr())
        return key is not None and t.numel() == key[1] and t.dtype == key[0]

    def give(self, t: torch.Tensor, side_events: Optional[Sequence] = None) -> bool:
        """Return a slab obtained from :meth:`take` (any other tensor: False).
        Work already enqueued that uses it finishes before its next user:
        the compute stream's work as enqueued now, the side streams' work up
        to ``side_events`` (the completion of the slab's last copy on each;
        None: up to their tails)."""
        key = self._owned.get(t.data_ptr())
        if key is None or t.numel() != key[1] or t.dtype != key[0] \
                or torch.cuda.is_current_stream_capturing():
            return False
        lst = self._free.setdefault(key, [])
        home = self.streams[0]
        if len(lst) >= self.max_free:  # back to the caching allocator (compute pool)
            del self._owned[t.data_ptr()]
            if side_events is None:
                for s in self.streams[1:]:
                    t.record_stream(s)
            else:  # free in compute order once its own copies have landed
                for ev in side_events:
                    home.wait_event(ev)
            return True
        if side_events is None:
            events = []
            for s in self.streams:
                ev = torch.cuda.Event()
                ev.record(s)
                events.append(ev)
        else:
            ev = torch.cuda.Event()
            ev.record(home)
            events = [ev] + list(side_events)
        lst.append((t, events))
        self.gives += 1
        return True

    def free_tensors(self) -> List[torch.Tensor]:
        return [t for lst in self._free.values() for t, _ in lst]

    @property
    def slab_bytes(self) -> int:
        return sum(dt.itemsize * n for dt, n in self._owned.values())

    def trim(self) -> int:
        """Release every free slab to PyTorch (after a device sync); bytes freed."""
        torch.cuda.synchronize(self.device)
        freed = 0
        for (dt, n), lst in self._free.items():
            for t, _ in lst:
                self._owned.pop(t.data_ptr(), None)
                freed += dt.itemsize * n
        self._free.clear()
        return freed
