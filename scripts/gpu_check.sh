set -x
free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -20
