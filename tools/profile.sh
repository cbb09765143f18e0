#!/bin/bash
# ncu evidence for profiles/: launch list (cold, serialised) + one --set full capture per hot kernel.
set -x
mkdir -p gpurun_out
CFG=${CFG:-llama8b_128k}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 2 --warmup 1 --cpu-budget 1 \
  > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_paged_attn -s 1 -c 1 \
  -o gpurun_out/prof_attn_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 1 --cpu-budget 1 \
  > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block_scores -s 1 -c 1 \
  -o gpurun_out/prof_scores_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 1 --cpu-budget 1 \
  > gpurun_out/ncu_scores.log 2>&1
ls -la gpurun_out
