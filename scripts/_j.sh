for r in 1 2 3; do
for v in 16 32 48; do CS_SWEEP_STEPS=5 CS_SPEC_HOST_GB=$v python scripts/configs_sweep.py 12b_mixed >> gpurun_out/j_ab.jsonl 2>&1; done
done
