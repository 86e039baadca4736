for f in 0.93 0.92 0.91 0.89; do CS_GPU_FRAC=$f python scripts/configs_sweep.py 12b_mixed >> gpurun_out/g_frac.jsonl 2>&1; done
