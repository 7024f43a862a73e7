#!/bin/bash
# Verification of the final commit: GPU tests, smoke, bench line, large-T rows.
mkdir -p gpurun_out
bash tools/gpu_verify.sh r02af
for row in "C4 T=80 rho=4" "C4 T=40 rho=4" "C4 T=20 rho=8"; do
  timeout 600 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(json.dumps(d))" >> gpurun_out/r02af_largeT.jsonl
done
cut -c1-260 gpurun_out/r02af_largeT.jsonl
