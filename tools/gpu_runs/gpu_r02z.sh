#!/bin/bash
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "four_slice" > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
grep -E "Error|error|assert" $OUT/tests.log | head -5
FLAGSETS=0,65536 ROUNDS=6 timeout 600 python tools/attn_bench.py paper_2605_16839_b200/libcpa.so > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab rc=$?"; cat $OUT/ab.jsonl; tail -3 $OUT/ab.err
