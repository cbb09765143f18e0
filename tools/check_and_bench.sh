#!/bin/bash
# one gpurun call: GPU parity suite + bench (+ optional extra configs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 400 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
for c in ${EXTRA_CFGS}; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget 2 > gpurun_out/bench_$c.log 2>&1; done
