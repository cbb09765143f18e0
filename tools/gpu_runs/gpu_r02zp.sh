#!/bin/bash
# r02zp: WG1's P in shared memory (triple-buffered) -- parity + A/B
OUT=gpurun_out/r02zp; mkdir -p $OUT
CPA_LIB_PATH=build_variants/p1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "attention or causal or full_tables or chunk_step or full_size or v_f16 or edge" > $OUT/tests.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/tests.log)"
ROUNDS=6 timeout 800 python tools/attn_bench.py build_variants/cur.so build_variants/p1.so build_variants/p1ns.so > $OUT/ab.jsonl 2>&1; grep -E "sparse_ms|maxdiff" $OUT/ab.jsonl
