#!/bin/bash
# Pinned uploads + compute-warp PDL wait: probe, rows, C3/C4 short, K-DP tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ab_build.log 2>&1 || { tail gpurun_out/r02ab_build.log; exit 1; }
timeout 300 python tools/ctx_probe.py 2>&1 | tail -5
for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "context: 50 models x 754-node scene, W=723" "f2 single instance 754 nodes, T=10" "C4 T=10 rho=4"; do
  timeout 300 python tools/bench_configs.py --only "$row" --steps 5 --warmup 2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:34].ljust(34), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
done
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']
print('C3 ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'xu', round(r.get('xu_frac',0),4))"
timeout 1200 python -m pytest tests -m gpu -q -x -k "tiled_kernel or model_batched or c4_shaped or dense_fallbacks or tile_sizes or c1_all or window_kernel or single_instance or stream or determinism" > gpurun_out/r02ab_tests.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02ab_tests.log
