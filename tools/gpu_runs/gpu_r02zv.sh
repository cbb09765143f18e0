#!/bin/bash
# r02zv: final driver-like run on the round's last code: build, smoke, every GPU test, bench (N=1), 32K line,
# ncu launch list of the bench step
OUT=gpurun_out/r02zv; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/gputest.log)"
timeout 900 python bench.py > $OUT/bench_llama8b_128k.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config llama8b_32k --steps 20 --warmup 5 --no-cpu > $OUT/bench_llama8b_32k.json 2> $OUT/bench32.err; echo "bench32 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_llama8b_128k.csv python bench.py --steps 2 --warmup 1 --no-cpu > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?"
for c in 128k 32k; do python -c "import json; d=json.load(open('$OUT/bench_llama8b_$c.json')); print('$c', d['value'], d['speedup_vs_dense'], d['stage_ms'], d['roofline']['frac'], d.get('step_ms_stats'), d['e2e']['value'])"; done
