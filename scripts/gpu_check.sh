for b in 8 16 32; do
  timeout 600 python bench.py --steps 6 --warmup 3 --batch $b --no-cpu-baseline --no-offload-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('B=$b', d['ms_per_step'], d['value'], d['tflops_per_gpu'], r['frac'], d['e2e']['value'])"
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
