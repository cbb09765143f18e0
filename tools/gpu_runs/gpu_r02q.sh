#!/bin/bash
OUT=gpurun_out/r02q; mkdir -p $OUT
B=build_variants
ROUNDS=8 timeout 900 python tools/attn_bench.py $B/old.so $B/kv.so $B/kv_ns.so > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab rc=$?"; cat $OUT/ab.jsonl
CFG=llama8b_128k timeout 300 python tools/attn_trace2.py $B/kv_trace.so > $OUT/trace.txt 2>&1
