#!/bin/bash
# r02n: polling (test_wait) vs suspending (try_wait) mbarrier waits in the softmax loop
OUT=gpurun_out/r02n; mkdir -p $OUT
B=build_variants
ROUNDS=6 timeout 900 python tools/attn_bench.py $B/base.so $B/base_smspin.so $B/base_allspin.so $B/spec_smspin.so > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab rc=$?"; cat $OUT/ab.jsonl
CFG=llama8b_128k timeout 300 python tools/attn_trace2.py $B/base_smspin_trace.so > $OUT/trace_base_smspin.txt 2>&1
