"""Loss trajectories of the 1B step: eager/graph x fused/unfused, same data."""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2108_05818_b200 import kernels as K
from paper_2108_05818_b200.config import PolicySpec
from paper_2108_05818_b200.model import build_gpt_schema
from paper_2108_05818_b200.trainer import ChunkTrainer

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 20
schema = build_gpt_schema(layers=layers, hidden_dim=2048, heads=16, seq_len=1024, vocab=50304, batch=16)
gen = torch.Generator().manual_seed(1000)
pool = [torch.randint(0, 50304, (16, 1025), generator=gen).cuda() for _ in range(4)]
for graph, fused in ((False, False), (False, True), (True, True)):
    tr = ChunkTrainer(schema, PolicySpec(capacity_elems=64 << 20), seed=0,
                      hyper=K.AdamHyper(lr=1e-4), cuda_graph=graph, fused_ops=fused)
    losses = [round(float(tr.step(pool[i % 4]).item()), 4) for i in range(24)]
    st = tr.step_state()
    print(json.dumps({"graph": graph, "fused": fused, "losses": losses, "scale": st.loss_scale,
                      "steps": st.step, "norm": st.grad_norm}), flush=True)
    del tr
    torch.cuda.empty_cache()
