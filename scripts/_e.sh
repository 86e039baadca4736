python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/e_gputest.log 2>&1; echo rc=$? >> gpurun_out/e_gputest.log
python bench.py > gpurun_out/e_bench.log 2>&1; echo rc=$? >> gpurun_out/e_bench.log
timeout 600 python scripts/host_link_contention.py > gpurun_out/e_contention.jsonl 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo rc=$? >> gpurun_out/e_smoke.log
