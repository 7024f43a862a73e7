#!/bin/bash
# Copy-warp-only PDL wait, K-U in-place model descriptors; bounds-checked build test; host
# enqueue probe; rows.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aa_build.log 2>&1 || { tail gpurun_out/r02aa_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -k "debug_checks or tiled_kernel or model_batched or c4_shaped or dense_fallbacks or tile_sizes or c1_all or window_kernel or single_instance_754 or determinism or classify or chains" > gpurun_out/r02aa_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02aa_tests.log
timeout 300 python tools/ctx_probe.py 2>&1 | tail -5
for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "context: 50 models x 754-node scene, W=723" "f2 single instance 754 nodes, T=10"; do
  timeout 300 python tools/bench_configs.py --only "$row" --steps 5 --warmup 2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:34].ljust(34), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
done
