python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/l_gputest.log 2>&1; echo rc=$? >> gpurun_out/l_gputest.log
timeout 800 python scripts/offload_timeline.py --model 12b --batch 8 --os auto --out gpurun_out/tl_12b_l.json > gpurun_out/tl_12b_l.log 2>&1
for r in 1 2 3; do CS_SWEEP_STEPS=5 python scripts/configs_sweep.py 12b_mixed >> gpurun_out/l_sweep.jsonl 2>&1; done
python scripts/configs_sweep.py 1b_os_cpu 12b_ckpt >> gpurun_out/l_sweep.jsonl 2>&1
