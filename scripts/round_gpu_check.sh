#!/bin/bash
# Full GPU evidence pass for one round (run under gpurun from the repo root):
# GPU test suite, the default bench line, the ncu launch list of one
# post-warm-up step, an ncu --set full capture of the in-step K1 launch, the
# C5 microbench with CPU arms, the single-GPU configuration sweep, smoke, the
# 12B offload timeline and the host-link / host-DRAM ceilings.
# Everything lands in gpurun_out/<tag>_*.
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/${tag}_build.log 2>&1
python -m pytest tests -m gpu -x -q > $out/${tag}_gputest.log 2>&1; echo rc=$? >> $out/${tag}_gputest.log
python bench.py > $out/${tag}_bench.log 2>&1; echo rc=$? >> $out/${tag}_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $out/${tag}_step_launches.csv \
    python bench.py --profile-step --warmup 3 --no-cpu-baseline --no-offload-probe --no-c5 \
    > $out/${tag}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:adam_tma -c 1 -f -o $out/${tag}_k1_insitu \
    python bench.py --profile-step --warmup 3 --no-cpu-baseline --no-offload-probe --no-c5 \
    > $out/${tag}_ncu_k1.log 2>&1
ncu -i $out/${tag}_k1_insitu.ncu-rep --page raw --csv > $out/${tag}_k1_insitu_raw.csv 2>/dev/null
python -m paper_2108_05818_b200.microbench --cpu > $out/${tag}_microbench_c5.jsonl 2>&1
python scripts/configs_sweep.py ${SWEEP:-12b_mixed 12b_ckpt 1b_os_cpu 4b_gpu 4b_os_cpu 1b_emb_host} \
    > $out/${tag}_configs_sweep.jsonl 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo rc=$? >> $out/${tag}_smoke.log
timeout 900 python scripts/offload_timeline.py --model 12b --batch 8 --os auto \
    --out $out/${tag}_timeline_12b.json > $out/${tag}_timeline_12b.log 2>&1
timeout 600 python scripts/host_link_contention.py > $out/${tag}_host_link_contention.jsonl 2>&1
timeout 600 python scripts/host_bw.py > $out/${tag}_host_bw.jsonl 2>&1
echo done
