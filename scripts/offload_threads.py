"""Host-Adam thread count vs the all-host-optimizer 1B step (bench's offload
probe): the host Adam and the chunk DMAs share host DRAM bandwidth.

    python scripts/offload_threads.py [threads ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2108_05818_b200 import trainer as T
    threads = [int(x) for x in sys.argv[1:]] or [4, 8, 12, 16]
    schema_kw = dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, vocab=50304, batch=32)
    orig = T.ChunkTrainer.__init__
    for n in threads:
        def init(self, *a, _n=n, **kw):
            kw["host_threads"] = _n
            orig(self, *a, **kw)
        T.ChunkTrainer.__init__ = init
        out = bench.offload_probe(schema_kw, torch.device("cuda:0"))
        T.ChunkTrainer.__init__ = orig
        print(json.dumps({"host_threads": n, "ms_per_step": out["ms_per_step"],
                          "h2d_gbs": out["chunk_moves"]["h2d"]["achieved_gbs"],
                          "d2h_gbs": out["chunk_moves"]["d2h"]["achieved_gbs"],
                          "host_adam_s": out["host_adam_s_per_step"],
                          "host_adam_gelem_per_s": out["host_adam_gelem_per_s"]}), flush=True)


if __name__ == "__main__":
    main()
