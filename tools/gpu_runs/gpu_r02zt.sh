#!/bin/bash
# r02zt: pool_q with 128-element slabs (4x the CTAs) -- parity + prepare A/B + shard sweep
OUT=gpurun_out/r02zt; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_abi.py -m gpu -x -q -p no:cacheprovider -k "estimator or full_size or chunk_step or shard or tables or abi" > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
for kvh in 8 1; do CFG=llama8b_128k KVH=$kvh ROUNDS=8 REPS=20 timeout 600 python tools/prep_ab.py build_variants/base.so build_variants/poolq.so >> $OUT/prep_ab.jsonl 2>> $OUT/prep_ab.err; done
CFG=llama8b_32k ROUNDS=8 REPS=20 timeout 600 python tools/prep_ab.py build_variants/base.so build_variants/poolq.so >> $OUT/prep_ab.jsonl 2>> $OUT/prep_ab.err
cat $OUT/prep_ab.jsonl
timeout 900 python tools/shard_sweep.py --reps 20 > $OUT/shard.jsonl 2> $OUT/shard.err; cat $OUT/shard.jsonl
