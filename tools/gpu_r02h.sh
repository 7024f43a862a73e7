bash tools/gpu_quick.sh r02h "window or c1_all or stream or bit or c0_T10 or single_instance_754" "C1|context|f2 single instance 754 nodes, T=10"
for row in "context: 50 models x 754-node scene, W=stride" C1; do
  HGM_LANES=1 HGM_TRACE_W=1 timeout 300 python tools/bench_configs.py --only "$row" --steps 1 --warmup 0 2>&1 | grep -v "^{" | head -14
done
