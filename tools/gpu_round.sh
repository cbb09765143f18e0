#!/bin/bash
# One GPU session: tests (optional), bench lines, ncu of the step's kernels. Usage:
#   tools/gpu_round.sh TAG [tests|notests] [configs...]
# Writes gpurun_out/TAG/*. Every step under its own timeout; never fails the whole call.
TAG=${1:-rxx}; MODE=${2:-tests}; shift 2; CONFIGS=${@:-llama8b_128k}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import sys; sys.path.insert(0,'.'); from paper_2605_16839_b200.build import build; build()" > $OUT/build.log 2>&1
if [ "$MODE" = "tests" ]; then
  CPA_PARITY_OUT=$OUT timeout 1800 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > $OUT/gputest.log 2>&1
  echo "tests rc=$? $(tail -1 $OUT/gputest.log)"
fi
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$? $(python -c "import json,sys; d=json.load(open('$OUT/bench_$c.json')); print(d['value'], d['speedup_vs_dense'], d['stage_ms'], d['roofline']['frac'])" 2>&1)"
done
