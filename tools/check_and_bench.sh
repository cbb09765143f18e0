#!/bin/bash
# one gpurun call: GPU parity suite + bench (+ optional extra configs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 400 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
for c in ${EXTRA_CFGS}; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget 2 > gpurun_out/bench_$c.log 2>&1; done
# sharded bench path smoke on one GPU (gloo, all ranks on cuda:0)
if [ -n "${SHARD_SMOKE}" ]; then
  CPA_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config llama8b_32k > gpurun_out/bench_shard2.log 2>&1
fi
