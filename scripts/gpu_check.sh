set -x
python -m pytest tests -m gpu -q 2>&1 | tail -5
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r1.csv python bench.py --profile-step --warmup 2 --no-cpu-baseline > gpurun_out/launches_r1.log 2>&1
tail -2 gpurun_out/launches_r1.log
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:adam_chunks -c 1 -o gpurun_out/k1_insitu_r1 python bench.py --profile-step --warmup 2 --no-cpu-baseline > gpurun_out/ncu_k1_insitu.log 2>&1
tail -2 gpurun_out/ncu_k1_insitu.log
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_r1.json
