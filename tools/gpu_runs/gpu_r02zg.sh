#!/bin/bash
OUT=gpurun_out/r02zg; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_abi.py tests/test_gpu_block_sparse.py -m gpu -x -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
for c in llama8b_32k llama8b_128k; do
CFG=$c ROUNDS=6 timeout 600 python tools/attn_bench.py build_variants/before_prologue.so build_variants/prologue.so > $OUT/ab_$c.jsonl 2>&1; grep sparse_ms $OUT/ab_$c.jsonl
done
