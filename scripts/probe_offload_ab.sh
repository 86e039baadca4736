for a in 0 1 0 1; do CS_ASYNC_HOST_ADAM=$a timeout 600 python -c "
import sys, json, torch; sys.path.insert(0,'.')
import bench
r = bench.offload_probe(dict(layers=20, hidden_dim=2048, heads=16, seq_len=1024, vocab=50304, batch=32), torch.device('cuda',0), steps=4)
print(json.dumps({k: r[k] for k in ('ms_per_step','host_adam_s_per_step','prefetch_issued','prefetch_discarded','async_host_adam')}), json.dumps(r['chunk_moves']))
" 2>&1 | tail -1; done
