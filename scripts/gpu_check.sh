python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-offload-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', d['ms_per_step'], d['value'], d['tflops_per_gpu'], r['frac'], d['e2e']['value'])"
