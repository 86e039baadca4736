"""Chunk-group collectives through the library's C ABI (``cs_comm_*``,
``cs_allgather``, ``cs_reduce_scatter_avg``, ``cs_allreduce``).

Same interface and semantics as :class:`.payload.ChunkComm` (the
reference's protocol, `parallel.py:196-264`), but the NCCL communicator is the
library's own, so a non-Python host (the cgo / JNI bindings in INTEGRATION.md)
drives exactly the calls the Python executor makes.  ``ChunkTrainer`` uses it
when ``CS_COMM=native``; the default is torch.distributed's NCCL.
torch.distributed is used only to broadcast the 128-byte unique id.

Async ops run on a dedicated comm stream that first waits for the caller's
stream; the returned work's ``wait()`` orders the caller's current stream
after the collective (no host wait), like torch's NCCL work objects.
"""

import ctypes
import sys
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

from . import _native as N

CODE = {torch.float16: N.CS_FP16, torch.bfloat16: N.CS_BF16, torch.float32: N.CS_FP32}


class NcclAsyncError(RuntimeError):
    """A collective failed after it was enqueued (ncclCommGetAsyncError);
    the communicator has been aborted."""


class _Work:
    __slots__ = ("_event", "_comm", "_start")

    def __init__(self, event: torch.cuda.Event, comm: "NativeChunkComm",
                 start: Optional[torch.cuda.Event] = None):
        self._event = event
        self._comm = comm
        self._start = start

    def get_duration(self) -> float:
        """Milliseconds the collective ran on the comm stream (after it)."""
        return self._start.elapsed_time(self._event)

    def wait(self) -> None:
        torch.cuda.current_stream().wait_event(self._event)

    def is_completed(self) -> bool:
        return self._event.query()

    def wait_host(self, timeout_s: float = 600.0) -> None:
        """Block the host until the collective completed, polling the
        communicator's asynchronous error; abort it on error or timeout."""
        self._comm.wait_event_host(self._event, timeout_s)


class NativeChunkComm:
    """One rank's library-owned NCCL communicator over a process group."""

    def __init__(self, group: Optional["dist.ProcessGroup"] = None,
                 device: Optional[torch.device] = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device(device or "cuda:%d" % torch.cuda.current_device())
        self.calls: List[Tuple[str, int]] = []
        lib = N.load()
        uid = b"\0" * 128
        if self.rank == 0:
            buf = ctypes.create_string_buffer(128)
            N.check(lib.cs_comm_unique_id(buf), "cs_comm_unique_id")
            uid = buf.raw
        box = [uid]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(box, src=src, group=group)
        self._comm = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.check(lib.cs_comm_init(box[0], self.world, self.rank, ctypes.byref(self._comm)),
                    "cs_comm_init")
        self.stream = torch.cuda.Stream(self.device)

    def check(self) -> None:
        """Raise (after aborting the communicator) if a collective failed
        asynchronously; SURVEY §5 failure detection."""
        if not self._comm:
            raise NcclAsyncError("the communicator was aborted")
        rc = N.load().cs_comm_check(self._comm)
        if rc not in (0, N.CS_EINPROGRESS):
            msg = N.load().cs_last_error().decode(errors="replace")
            self.abort()
            raise NcclAsyncError("NCCL asynchronous error (rc=%d): %s" % (rc, msg))

    def abort(self) -> None:
        """ncclCommAbort: unblocks kernels stuck on a dead peer; the
        communicator cannot be used afterwards."""
        if self._comm:
            N.load().cs_comm_abort(self._comm)
            self._comm = ctypes.c_void_p()

    def wait_event_host(self, event: torch.cuda.Event, timeout_s: float = 600.0) -> None:
        import time
        t0 = time.monotonic()
        delay = 1e-4
        while not event.query():
            self.check()
            if time.monotonic() - t0 > timeout_s:
                self.abort()
                raise NcclAsyncError("collective did not complete in %.0f s; communicator "
                                     "aborted" % timeout_s)
            time.sleep(delay)
            delay = min(delay * 2, 0.05)
        self.check()

    def close(self) -> None:
        if self._comm:
            N.check(N.load().cs_comm_destroy(self._comm), "cs_comm_destroy")
            self._comm = ctypes.c_void_p()

    def __del__(self):
        # at interpreter exit the CUDA context may already be gone: leave the
        # communicator to the process teardown rather than call into NCCL
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass

    def _run(self, call, async_op: bool, *tensors: torch.Tensor):
        self.check()  # a failed earlier collective surfaces at the next issue
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)
        for t in tensors:  # the caching allocator must not recycle them under the op
            t.record_stream(self.stream)
        start = torch.cuda.Event(enable_timing=True)
        start.record(self.stream)
        call(ctypes.c_void_p(self.stream.cuda_stream))
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        work = _Work(ev, self, start)
        if async_op:
            return work
        work.wait()
        return None

    @staticmethod
    def _code(t: torch.Tensor) -> int:
        if t.dtype not in CODE or not t.is_cuda or not t.is_contiguous():
            raise ValueError("native collectives take contiguous CUDA fp16/bf16/fp32 tensors")
        return CODE[t.dtype]

    def all_gather_slab(self, slab: torch.Tensor, async_op: bool = False,
                        src: Optional[torch.Tensor] = None):
        """This rank's contribution is ``src`` (out of place) or slot ``rank``
        of ``slab`` (in place)."""
        cap = slab.numel() // self.world
        code = self._code(slab)
        keep = (slab,)
        if src is None:
            mine = slab.data_ptr() + self.rank * cap * slab.element_size()
        else:
            if self._code(src) != code or src.numel() < cap:
                raise ValueError("all_gather_slab: src must hold one slot of the slab's dtype")
            mine, keep = src.data_ptr(), (slab, src)
        self.calls.append(("all_gather", slab.numel() * slab.element_size()))
        lib = N.load()
        return self._run(lambda s: N.check(lib.cs_allgather(slab.data_ptr(), mine, cap, code,
                                                            self._comm, s), "cs_allgather"),
                         async_op, *keep)

    def reduce_scatter_avg(self, out: torch.Tensor, slab: torch.Tensor, async_op: bool = False):
        code = self._code(slab)
        if out.numel() * self.world != slab.numel() or out.dtype != slab.dtype:
            raise ValueError("reduce_scatter_avg: out must be one slot of the group buffer")
        self.calls.append(("reduce_scatter", slab.numel() * slab.element_size()))
        lib = N.load()
        return self._run(lambda s: N.check(lib.cs_reduce_scatter_avg(
            out.data_ptr(), slab.data_ptr(), out.numel(), code, self._comm, s),
            "cs_reduce_scatter_avg"), async_op, out, slab)

    def _all_reduce(self, t: torch.Tensor, avg: int) -> None:
        code = self._code(t)
        lib = N.load()
        self._run(lambda s: N.check(lib.cs_allreduce(t.data_ptr(), t.numel(), code, avg,
                                                     self._comm, s), "cs_allreduce"), False, t)

    def all_reduce_sum(self, t: torch.Tensor) -> None:
        self._all_reduce(t, 0)

    def all_reduce_avg(self, t: torch.Tensor) -> None:
        self._all_reduce(t, 1)
