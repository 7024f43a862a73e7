#!/bin/bash
# K-DPW v2 (merged dummy forms, 3 barriers per step), K-BT fewer dependent loads, unary
# unroll, trace-pointer hoist: config rows, full GPU tests, C3 bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02w_build.log 2>&1 || { tail gpurun_out/r02w_build.log; exit 1; }
for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "context: 50 models x 754-node scene, W=723" "f2 single instance 754 nodes, T=10" "C2"; do
  timeout 300 python tools/bench_configs.py --only "$row" --steps 3 --warmup 2 2>/dev/null | cut -c1-420
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02w_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r02w_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02w_bench.json 2>gpurun_out/r02w_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02w_bench.json')); r=d['roofline']
print('C3', round(d['value']), 'pairs/s ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'kernel_ms', {k: round(v,3) for k,v in r['kernel_ms'].items()})"
