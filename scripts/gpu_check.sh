mkdir -p gpurun_out
timeout 2400 python scripts/configs_sweep.py 2>&1 | tee gpurun_out/configs_sweep_r1.jsonl
free -g | head -2
