OUT=gpurun_out/r02b; mkdir -p $OUT
python -c "import sys; sys.path.insert(0,'.'); from paper_2605_16839_b200.build import build; build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_shard.py tests/test_gpu_host_stream.py tests/test_gpu_block_sparse.py -m gpu -x -q -p no:cacheprovider > $OUT/gputest.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/gputest.log)"
for c in llama8b_128k llama8b_32k; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$? $(python -c "import json; d=json.load(open('$OUT/bench_$c.json')); print(d['value'], d['speedup_vs_dense'], d['stage_ms'], d['roofline']['frac'], d['clocks'])" 2>&1 | tail -1)"
done
CPA_BENCH_NO_PDL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_nopdl.json 2> $OUT/bench_nopdl.err; echo "nopdl $(python -c "import json; d=json.load(open('$OUT/bench_nopdl.json')); print(d['value'], d['stage_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
timeout 600 ncu --set full --clock-control none -k regex:"k_append|k_pool_q|k_block_scores|k_mask_union" -c 4 -o $OUT/small python bench.py --steps 1 --warmup 0 --no-cpu > $OUT/ncu_small.log 2>&1; echo "ncu small rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_case.py > $OUT/sanitize_$tool.log 2>&1; echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases' $OUT/sanitize_$tool.log | tr '\n' ' ')"
done
