#!/bin/bash
# r02k: state-of-the-art comparators (FA4 CuTe, trtllm-gen) + bench + ncu of the final kernels
OUT=gpurun_out/r02k; mkdir -p $OUT
python -c "import sys; sys.path.insert(0,'.'); from paper_2605_16839_b200.build import build; build()" > $OUT/build.log 2>&1
timeout 900 python tools/sota_compare.py > $OUT/sota.jsonl 2> $OUT/sota.err; echo "sota rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > $OUT/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_paged_attn -s 1 -c 1 \
  -o $OUT/prof_attn -f python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_attn.log 2>&1; echo "ncu2 rc=$?"
ls -la $OUT
