"""Which allocation makes the caching allocator free its cache and retry?
Runs a sweep configuration, records the allocator history for a few steps
and prints the Python frames of allocations around every segment free.

    python scripts/alloc_trace.py 12b_mixed [steps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    import torch
    from configs_sweep import CONFIGS
    from paper_2108_05818_b200 import kernels as K
    from paper_2108_05818_b200.config import PolicySpec
    from paper_2108_05818_b200.model import build_gpt_schema
    from paper_2108_05818_b200.trainer import ChunkTrainer
    c = CONFIGS[sys.argv[1]]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    schema = build_gpt_schema(layers=c["layers"], hidden_dim=c["hidden"], heads=c["heads"],
                              seq_len=1024, vocab=50304, batch=c["batch"])
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=c["cap"], os_placement=c["os"],
                                         checkpointing=c.get("ckpt", False)),
                      seed=0, hyper=K.AdamHyper(lr=1e-4))
    tok = torch.randint(0, 50304, (c["batch"], 1025)).cuda()
    for _ in range(3):
        tr.step(tok)
    tr.finish_host_work()
    torch.cuda.synchronize()
    r0 = torch.cuda.memory_stats().get("num_alloc_retries", 0)
    torch.cuda.memory._record_memory_history(max_entries=200000, stacks="python")
    for _ in range(steps):
        tr.step(tok)
    tr.finish_host_work()
    torch.cuda.synchronize()
    snap = torch.cuda.memory._snapshot()
    torch.cuda.memory._record_memory_history(enabled=None)
    print("retries during trace:", torch.cuda.memory_stats().get("num_alloc_retries", 0) - r0)
    for dev_trace in snap["device_traces"]:
        for i, ev in enumerate(dev_trace):
            if ev["action"] in ("segment_free", "segment_unmap", "oom"):
                # the allocation that forced it is the next 'alloc' event
                nxt = next((e for e in dev_trace[i:i + 4000] if e["action"] == "alloc"), None)
                print("==", ev["action"], ev.get("size"), "-> next alloc", nxt and nxt["size"])
                if nxt:
                    for fr in nxt.get("frames", [])[:12]:
                        if "site-packages" not in fr["filename"]:
                            print("   ", fr["filename"].split("/")[-1], fr["line"], fr["name"])
                break


if __name__ == "__main__":
    main()
