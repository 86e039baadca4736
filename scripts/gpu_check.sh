python -m pytest tests/test_step_gpu.py -q -x 2>&1 | tail -8
