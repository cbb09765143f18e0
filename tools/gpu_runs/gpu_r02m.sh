#!/bin/bash
# r02m: speculative-exponential softmax A/B (base = max-then-exp, spec, spec without stagger), trace, parity
OUT=gpurun_out/r02m; mkdir -p $OUT
B=build_variants
ROUNDS=6 timeout 900 python tools/attn_bench.py $B/base.so $B/spec.so $B/specns.so > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab rc=$?"; cat $OUT/ab.jsonl
CFG=llama8b_128k timeout 300 python tools/attn_trace2.py $B/spec_trace.so > $OUT/trace_spec.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "attention or causal or full_tables or chunk_step or full_size or persistent or v_f16" > $OUT/parity.log 2>&1; echo "parity rc=$? $(tail -1 $OUT/parity.log)"
