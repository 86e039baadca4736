"""The C-ABI chunk-group collectives (``cs_comm_*``, ``cs_allgather``,
``cs_reduce_scatter_avg``, ``cs_allreduce``) through
:class:`NativeChunkComm`, the ``CS_COMM=native`` communicator of the executor.

This sandbox has one GPU and NCCL refuses two ranks on one device, so the
library's communicator is exercised at world size 1 (NCCL really runs: the
all-gather and reduce-scatter are its single-rank copies); the multi-rank
protocol above it is the executor's, covered over gloo by
tests/test_dp_step_gpu.py and tests/test_dp_gloo.py.
"""

import os
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    res = {}
    try:
        from paper_2108_05818_b200 import _native as N
        from paper_2108_05818_b200.native_comm import NativeChunkComm
        lib = N.load()
        res["version"] = lib.cs_comm_version()
        comm = NativeChunkComm(None, torch.device("cuda:0"))
        g = torch.Generator(device="cuda").manual_seed(5)
        for dtype in (torch.float16, torch.bfloat16):
            slab = torch.randn(1 << 20, device="cuda", generator=g).to(dtype)
            ref = slab.clone()
            comm.all_gather_slab(slab)                     # in place, slot 0 = mine
            res["ag_%s" % dtype] = torch.equal(slab.view(torch.int16), ref.view(torch.int16))
            mine = torch.empty_like(slab)
            w = comm.reduce_scatter_avg(mine, slab, async_op=True)
            w.wait()                                       # current stream after the op
            res["rs_%s" % dtype] = torch.equal(mine.view(torch.int16), ref.view(torch.int16))
        s = torch.tensor([3.25], device="cuda")
        comm.all_reduce_sum(s)
        comm.all_reduce_avg(s)
        res["allreduce"] = float(s.item())
        res["calls"] = [k for k, _ in comm.calls]
        try:
            comm.all_gather_slab(torch.zeros(8, 2, device="cuda").t())
            res["noncontig"] = "accepted"
        except ValueError:
            res["noncontig"] = "rejected"
        rc = lib.cs_allgather(None, None, 4, N.CS_FP16, comm._comm, None)
        res["einval"] = rc
        w = comm.reduce_scatter_avg(mine, slab, async_op=True)
        w.wait_host(timeout_s=60)                         # polls the async error
        res["check"] = lib.cs_comm_check(comm._comm)
        torch.cuda.synchronize()
        from paper_2108_05818_b200.native_comm import NcclAsyncError
        comm2 = NativeChunkComm(None, torch.device("cuda:0"))
        comm2.abort()                                      # ncclCommAbort
        try:
            comm2.all_gather_slab(torch.zeros(16, device="cuda").half())
            res["after_abort"] = "accepted"
        except NcclAsyncError:
            res["after_abort"] = "raised"
        res["check_null"] = lib.cs_comm_check(None)
        comm.close()
    finally:
        dist.destroy_process_group()
    torch.save(res, out)


def test_native_communicator_single_rank_round_trip():
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.pt")
        mp.spawn(_worker, args=(29400 + os.getpid() % 500, out), nprocs=1, join=True)
        res = torch.load(out, weights_only=False)
    major, minor, patch = torch.cuda.nccl.version()
    # the library reuses the NCCL torch already loaded (RTLD_NOLOAD first)
    assert res["version"] == major * 10000 + minor * 100 + patch
    for dtype in (torch.float16, torch.bfloat16):
        assert res["ag_%s" % dtype] and res["rs_%s" % dtype]
    assert res["allreduce"] == 3.25
    assert res["calls"] == ["all_gather", "reduce_scatter"] * 2
    assert res["noncontig"] == "rejected"
    assert res["einval"] == -1
    assert res["check"] == 0 and res["check_null"] == -1
    assert res["after_abort"] == "raised"
