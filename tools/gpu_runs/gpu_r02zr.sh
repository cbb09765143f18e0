#!/bin/bash
# r02zr: asymmetric key split between the softmax warpgroups (CPA_SPLIT0 = keys of WG0) -- parity + A/B
OUT=gpurun_out/r02zr; mkdir -p $OUT
for v in s80 s96; do
CPA_LIB_PATH=build_variants/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "attention or causal or full_tables or chunk_step or v_f16 or edge" > $OUT/tests_$v.log 2>&1; echo "tests $v rc=$? $(tail -1 $OUT/tests_$v.log)"
done
ROUNDS=6 timeout 900 python tools/attn_bench.py build_variants/base.so build_variants/s64.so build_variants/s80.so build_variants/s96.so > $OUT/ab.jsonl 2>&1; grep -E "sparse_ms|maxdiff" $OUT/ab.jsonl
