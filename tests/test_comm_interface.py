"""The communicators the executor accepts share one interface (no GPU needed):
torch.distributed's ``ChunkComm``, the C-ABI ``NativeChunkComm`` and any
caller-supplied object passed as ``ChunkTrainer(comm=...)``."""

import inspect

from paper_2108_05818_b200.native_comm import NativeChunkComm
from paper_2108_05818_b200.payload import ChunkComm
from paper_2108_05818_b200.trainer import ChunkTrainer

METHODS = ("all_gather_slab", "reduce_scatter_avg", "all_reduce_sum", "all_reduce_avg",
           "check")


def test_native_comm_mirrors_chunk_comm():
    for name in METHODS:
        a = inspect.signature(getattr(ChunkComm, name))
        b = inspect.signature(getattr(NativeChunkComm, name))
        assert list(a.parameters) == list(b.parameters), name
        for p in a.parameters:
            assert a.parameters[p].default == b.parameters[p].default, (name, p)


def test_trainer_accepts_a_communicator():
    assert "comm" in inspect.signature(ChunkTrainer.__init__).parameters
    assert hasattr(ChunkTrainer, "step_host_async") and hasattr(ChunkTrainer, "step_host")
