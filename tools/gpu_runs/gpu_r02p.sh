#!/bin/bash
OUT=gpurun_out/r02p; mkdir -p $OUT
B=build_variants
ROUNDS=6 timeout 900 python tools/attn_bench.py $B/old.so $B/w2_base.so $B/w2_spec.so $B/w2_base_ns.so > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab rc=$?"; cat $OUT/ab.jsonl
CFG=llama8b_128k timeout 300 python tools/attn_trace2.py $B/w2_base_trace.so > $OUT/trace.txt 2>&1
