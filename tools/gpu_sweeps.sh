#!/bin/bash
# NEXT-3 / NEXT-4 measurements on the final kernels (profiles/r02_*.jsonl):
#   chunk-size sweep at 128K (whole prefills, base + qdiverse workloads), context sweep, rho sweep
#   (bench.py --rho, final chunk), execution ablation at 128K / chunk 512 / B = 1..16.
TAG=${1:-r02s}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import sys; sys.path.insert(0,'.'); from paper_2605_16839_b200.build import build; build()" > $OUT/build.log 2>&1
timeout 1500 python tools/prefill_sweep.py --contexts 131072 --chunks 512,1024,2048,4096 > $OUT/chunk_sweep_base.jsonl 2> $OUT/chunk_sweep_base.err; echo "chunk base rc=$?"; cat $OUT/chunk_sweep_base.jsonl
timeout 1500 python tools/prefill_sweep.py --contexts 131072 --chunks 512,1024,2048,4096 --variant qdiverse --rho 0.47 > $OUT/chunk_sweep_qdiverse.jsonl 2> $OUT/chunk_sweep_qdiverse.err; echo "chunk qdiverse rc=$?"; cat $OUT/chunk_sweep_qdiverse.jsonl
timeout 1200 python tools/prefill_sweep.py --contexts 8192,16384,32768,65536,131072 --chunks 4096 > $OUT/context_sweep.jsonl 2> $OUT/context_sweep.err; echo "context rc=$?"; cat $OUT/context_sweep.jsonl
for rho in 0.1 0.2 0.3 0.5 1.0; do
  timeout 600 python bench.py --rho $rho --steps 10 --warmup 3 --no-cpu >> $OUT/rho_sweep.jsonl 2>> $OUT/rho_sweep.err; echo "rho $rho rc=$?"
done
timeout 2400 python tools/ablation_exec.py --context 131072 --chunk 512 --batches 1,2,4,8,16 > $OUT/exec_ablation.jsonl 2> $OUT/exec_ablation.err; echo "ablation rc=$?"; cat $OUT/exec_ablation.jsonl
