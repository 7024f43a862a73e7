#!/bin/bash
# A/B: round-start library (libhgm_base.so) vs the current one; small-problem rows; K-DP tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02y_build.log 2>&1 || { tail gpurun_out/r02y_build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "tiled_kernel or model_batched or c4_shaped or dense_fallbacks or tile_sizes or c3_sampled or c2_sampled or determinism" > gpurun_out/r02y_tests.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02y_tests.log
for rep in 1 2; do bash tools/ab_run.sh r02y base default > /dev/null 2>&1; done
cat gpurun_out/r02y_ab.txt
for v in base default; do
  if [ $v = default ]; then unset HGM_LIB; else export HGM_LIB=$PWD/paper_1505_00581_b200/lib/libhgm_$v.so; fi
  for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "context: 50 models x 754-node scene, W=723" "f2 single instance 754 nodes, T=10" "f2 single instance 754 nodes, T=inf"; do
    timeout 300 python tools/bench_configs.py --only "$row" --steps 5 --warmup 2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'][:34].ljust(34), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
  done
done
