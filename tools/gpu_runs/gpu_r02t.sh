#!/bin/bash
# r02t: fused a3-a5 in the estimator epilogue: parity + prepare A/B (fused vs separate kernels)
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fused_tables.py tests/test_gpu_parity.py tests/test_gpu_abi.py -m gpu -x -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
for kvh in 8 1; do CFG=llama8b_128k KVH=$kvh FLAGSETS=0,32768 ROUNDS=8 REPS=20 timeout 600 python tools/prep_ab.py build_variants/fused.so >> $OUT/prep_ab.jsonl 2>> $OUT/prep_ab.err; done
CFG=llama8b_32k FLAGSETS=0,32768 ROUNDS=8 REPS=20 timeout 600 python tools/prep_ab.py build_variants/fused.so >> $OUT/prep_ab.jsonl 2>> $OUT/prep_ab.err
cat $OUT/prep_ab.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['stage_ms'], d['roofline']['frac'], d['clocks'])"
