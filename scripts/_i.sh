for r in 1 2 3; do
for v in 1 0; do CS_HOST_READ_EVENTS=$v python scripts/configs_sweep.py 1b_os_cpu >> gpurun_out/i_ab.jsonl 2>&1; done
done
for r in 1 2; do
for v in 1 0; do CS_HOST_READ_EVENTS=$v python scripts/configs_sweep.py 12b_mixed >> gpurun_out/i_ab.jsonl 2>&1; done
done
