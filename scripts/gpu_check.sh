set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python -m paper_2108_05818_b200.microbench --sizes 20,24,26,28,30 --iters 10 2>&1 | tee gpurun_out/microbench_r1a.jsonl
ncu --set full --clock-control none --import-source on -k regex:adam_chunks -s 3 -c 1 -o gpurun_out/k1_adam_2p28 python -m paper_2108_05818_b200.microbench --sizes 28 --iters 2 > gpurun_out/ncu_k1.log 2>&1
tail -3 gpurun_out/ncu_k1.log
lscpu | head -20
