mkdir -p gpurun_out
for s in ${STEPS:-maskin scores scores128 attn attn128}; do
  echo "=== $s" >> gpurun_out/dbg.log
  timeout 60 python tools/gpu_debug.py $s >> gpurun_out/dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dbg.log
done
