mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_r1_final.json
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r1b.csv python bench.py --profile-step --warmup 2 --no-cpu-baseline --no-offload-probe > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:adam_tma -c 1 -o gpurun_out/k1_tma_insitu python bench.py --profile-step --warmup 2 --no-cpu-baseline --no-offload-probe > gpurun_out/ncu_k1_tma.log 2>&1
tail -1 gpurun_out/ncu_k1_tma.log
