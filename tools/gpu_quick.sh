#!/bin/bash
# Quick GPU iteration: build, a parity subset, bench lines (no cpu leg), optional extra command.
#   tools/gpu_quick.sh TAG "configs" ["extra command"]
TAG=$1; CONFIGS=${2:-llama8b_128k}; EXTRA=$3
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import sys; sys.path.insert(0,'.'); from paper_2605_16839_b200.build import build; build()" > $OUT/build.log 2>&1 || { echo "build failed"; tail -20 $OUT/build.log; exit 1; }
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $OUT/extra.log 2>&1; echo "extra rc=$?"; tail -5 $OUT/extra.log; fi
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_shard.py tests/test_gpu_host_stream.py tests/test_gpu_block_sparse.py -m gpu -x -q -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/gputest.log)"
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$? $(python -c "import json; d=json.load(open('$OUT/bench_$c.json')); print(d['value'], d['speedup_vs_dense'], d['stage_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
