python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1
timeout 900 python -m pytest tests/test_offload_overlap_gpu.py tests/test_fuzz_step_gpu.py -x -q -m gpu > gpurun_out/h_tests.log 2>&1; echo rc=$? >> gpurun_out/h_tests.log
timeout 800 python scripts/offload_timeline.py --model 12b --batch 8 --os auto --out gpurun_out/tl_12b_i.json > gpurun_out/tl_12b_i.log 2>&1
python scripts/configs_sweep.py 12b_mixed 12b_mixed 1b_os_cpu > gpurun_out/h_sweep.jsonl 2>&1
