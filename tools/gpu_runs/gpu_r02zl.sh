#!/bin/bash
# r02zl: driver-like final run: build, smoke, every GPU test, reference arm, bench (N=1)
OUT=gpurun_out/r02zl; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/gputest.log)"
S=$(date +%s); timeout 900 python bench.py --impl reference > $OUT/reference.json 2> $OUT/reference.err; echo "reference rc=$? wall=$(( $(date +%s) - S )) s"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['speedup_vs_dense'], d['stage_ms'], d['roofline']['frac'], d['step_ms_stats'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
python -c "import json; d=json.load(open('$OUT/reference.json')); print(d['value'], d['steps'], d['cpu_baseline']['sample'][:200])"
