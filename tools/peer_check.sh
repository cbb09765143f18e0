#!/bin/bash
# one gpurun call: GPU tests (incl. simulated-peer fused all-gather), bench, and the fused peer path
# through real torch symmetric memory on a 1-rank NCCL group.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
CPA_BENCH_PEER_W1=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29513 bench.py --steps 5 --warmup 3 --config llama8b_32k --cpu-budget 1 > gpurun_out/bench_peer_w1.log 2>&1
CPA_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config llama8b_32k > gpurun_out/bench_shard2.log 2>&1
