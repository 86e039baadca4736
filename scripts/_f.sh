python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 1200 python -m pytest tests/test_embedding_host_weights_gpu.py tests/test_step_gpu.py tests/test_fuzz_step_gpu.py tests/test_offload_overlap_gpu.py -x -q -m gpu > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
python scripts/configs_sweep.py 1b_emb_host > gpurun_out/f_sweep.jsonl 2>&1

