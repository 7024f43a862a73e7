bash tools/gpu_evidence.sh r02g
for row in "context: 50 models x 754-node scene, W=stride" C1; do
  HGM_LANES=1 HGM_TRACE_W=1 timeout 300 python tools/bench_configs.py --only "$row" --steps 1 --warmup 0 2>&1 | grep -v "^{" | head -40
done > gpurun_out/r02g_wtrace.txt
head -80 gpurun_out/r02g_wtrace.txt
