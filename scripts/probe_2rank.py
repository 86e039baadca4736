import os, torch, torch.distributed as dist, torch.multiprocessing as mp
def run(rank, ws, backend, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    try:
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", 0))
        else:
            dist.init_process_group(backend, rank=rank, world_size=ws)
        slab = torch.zeros(8, dtype=torch.float16, device="cuda")
        slab[rank*4:(rank+1)*4] = rank + 1
        dist.all_gather_into_tensor(slab, slab[rank*4:(rank+1)*4])
        out = torch.empty(4, dtype=torch.float16, device="cuda")
        dist.reduce_scatter_tensor(out, torch.arange(8, dtype=torch.float16, device="cuda") * (rank + 1), op=dist.ReduceOp.AVG)
        t = torch.tensor([rank + 1.0], device="cuda"); dist.all_reduce(t)
        torch.cuda.synchronize()
        print(backend, rank, "ok", slab.tolist(), out.tolist(), t.item(), flush=True)
    except Exception as e:
        print(backend, rank, "FAIL", repr(e)[:300], flush=True)
    finally:
        try: dist.destroy_process_group()
        except Exception: pass
if __name__ == "__main__":
    for i, b in enumerate(["gloo", "nccl"]):
        mp.spawn(run, args=(2, b, 29700 + i), nprocs=2, join=True)
