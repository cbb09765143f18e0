#!/bin/bash
# Attention-kernel A/B on the 128K chunk (tools/attn_bench.py) + one ncu --set full capture.
#   tools/gpu_ab.sh TAG "libs..." FLAGSETS [ncu_lib ncu_flags]
TAG=$1; LIBS=$2; FLAGSETS=${3:-0}; NLIB=$4; NFLAGS=${5:-0}
OUT=gpurun_out/$TAG; mkdir -p $OUT
FLAGSETS=$FLAGSETS ROUNDS=${ROUNDS:-5} timeout 900 python tools/attn_bench.py $LIBS > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab rc=$?"; cat $OUT/ab.jsonl
if [ -n "$NLIB" ]; then
  CPA_LIB_PATH=$NLIB FLAGSETS=$NFLAGS ROUNDS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_paged_attn -c 1 -o $OUT/attn python tools/attn_bench.py $NLIB > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
fi
