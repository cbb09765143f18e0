#!/bin/bash
# r02zu: CSR built by the last union CTA for small tables -- parity + prepare A/B + shard sweep
OUT=gpurun_out/r02zu; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_abi.py tests/test_gpu_block_sparse.py tests/test_c_abi.py -m gpu -x -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
for kvh in 1 2; do CFG=llama8b_128k KVH=$kvh ROUNDS=8 REPS=20 timeout 600 python tools/prep_ab.py build_variants/base.so build_variants/csrf.so >> $OUT/prep_ab.jsonl 2>> $OUT/prep_ab.err; done
cat $OUT/prep_ab.jsonl
timeout 900 python tools/shard_sweep.py --reps 20 > $OUT/shard.jsonl 2> $OUT/shard.err; cat $OUT/shard.jsonl
