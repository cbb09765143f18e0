#!/bin/bash
# r02y: driver-like run on the round's kernels: build, smoke, every GPU test, bench lines (128K with the
# cpu leg, 32K), ncu launch list + --set full of the attention and the scores kernel, racecheck/synccheck
OUT=gpurun_out/r02y; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/gputest.log)"
timeout 900 python bench.py > $OUT/bench_llama8b_128k.json 2> $OUT/bench_128k.err; echo "bench rc=$?"
timeout 600 python bench.py --config llama8b_32k --steps 20 --warmup 5 --no-cpu > $OUT/bench_llama8b_32k.json 2> $OUT/bench_32k.err; echo "bench32 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_llama8b_128k.csv python bench.py --steps 2 --warmup 1 --no-cpu > $OUT/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_paged_attn -s 1 -c 1 -o $OUT/prof_attn_llama8b_128k -f python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_attn.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block_scores -s 1 -c 1 -o $OUT/prof_scores_llama8b_128k -f python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_scores.log 2>&1; echo "ncu3 rc=$?"
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_case.py > $OUT/sanitize_$tool.log 2>&1; echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases' $OUT/sanitize_$tool.log | tr '\n' ' ')"
done
