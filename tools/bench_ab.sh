#!/bin/bash
# Interleaved bench.py A/B over libcpa builds: ROUNDS x libs, one JSON summary line per run.
#   tools/bench_ab.sh TAG "lib1 lib2 ..." [config] [extra bench args]
TAG=$1; LIBS=$2; CFG=${3:-llama8b_128k}; EXTRA=$4
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in $(seq 1 ${ROUNDS:-3}); do
  for lib in $LIBS; do
    CPA_LIB_PATH=$lib timeout 600 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu $EXTRA > $OUT/b.json 2> $OUT/b.err
    python -c "import json; d=json.load(open('$OUT/b.json')); print(json.dumps({'lib': '$lib', 'round': $r, 'value': d['value'], 'attention': d['stage_ms']['attention'], 'frac': d['roofline']['frac'], 'dense': d['dense_ms_per_chunk'], 'sm_mhz': d['clocks']['sm_mhz']}))" | tee -a $OUT/ab.jsonl
  done
done
