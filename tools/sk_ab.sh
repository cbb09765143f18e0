#!/bin/bash
# stream-K vs per-unit grid (CPA_F_NO_PERSIST = 1024) on per-GPU shards of the 128K chunk
mkdir -p gpurun_out
for kvh in 1 2 4 8; do
  KVH=$kvh FLAGSETS=0,1024,2048 ROUNDS=6 timeout 300 python tools/attn_bench.py paper_2605_16839_b200/libcpa.so > gpurun_out/sk_ab_kvh$kvh.log 2>&1
done
CFG=llama8b_32k KVH=2 FLAGSETS=0,1024,2048 ROUNDS=6 timeout 300 python tools/attn_bench.py paper_2605_16839_b200/libcpa.so > gpurun_out/sk_ab_32k.log 2>&1
