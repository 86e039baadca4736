python -m pytest tests/test_step_gpu.py tests/test_kernels_gpu.py -q -x 2>&1 | tail -4
for v in 0 1 2 3 4; do
  echo "variant $v"
  CS_ADAM_VARIANT=$v python -m paper_2108_05818_b200.microbench --sizes 30 --iters 10 2>&1 | grep adam
  CS_ADAM_VARIANT=$v timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks'], d['final_loss'], d['cuda_graph'])"
done
