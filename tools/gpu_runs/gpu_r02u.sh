#!/bin/bash
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fused_tables.py -m gpu -x -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
for kvh in 8 1; do CFG=llama8b_128k KVH=$kvh FLAGSETS=0,32768 ROUNDS=8 REPS=20 timeout 600 python tools/prep_ab.py build_variants/fused2.so >> $OUT/prep_ab.jsonl 2>> $OUT/prep_ab.err; done
cat $OUT/prep_ab.jsonl
