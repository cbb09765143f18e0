#!/bin/bash
# r02zc: bench lines of every BASELINE config on the final kernels + the four-slice ablation tests
OUT=gpurun_out/r02zc; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "four_slice" > $OUT/ks4_tests.log 2>&1; echo "ks4 tests rc=$? $(tail -1 $OUT/ks4_tests.log)"
for c in llama8b_64k_b4 qwen3_30b_128k; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --config qwen3_30b_128k --exec-group 4 --steps 20 --warmup 5 --no-cpu > $OUT/bench_qwen_e4.json 2> $OUT/bench_qwen_e4.err; echo "bench qwen e4 rc=$?"
for f in $OUT/bench_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['speedup_vs_dense'], d['stage_ms'], d['roofline']['frac'])"; done
