#!/bin/bash
# per-kernel durations (ncu launch list) of the stream-K path vs the per-unit grid on shard shapes
mkdir -p gpurun_out
for cfg in "llama8b_32k 2" "llama8b_128k 1"; do set -- $cfg
  CFG=$1 KVH=$2 FLAGSETS=0,1024 ROUNDS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/sk_prof_$1_$2.csv python tools/attn_bench.py paper_2605_16839_b200/libcpa.so > /dev/null 2>&1
done
