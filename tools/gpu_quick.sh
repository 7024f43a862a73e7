#!/bin/bash
# Quick GPU iteration (run under gpurun): build, selected GPU tests, selected config rows.
# usage: tools/gpu_quick.sh <tag> "<pytest -k expr or ''>" "<row1>|<row2>|..." [extra env for rows]
tag=$1; kexpr=$2; rows=$3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo build failed; tail gpurun_out/${tag}_build.log; exit 1; }
if [ -n "$kexpr" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$kexpr" > gpurun_out/${tag}_tests.log 2>&1
  echo "pytest rc=$?"; tail -4 gpurun_out/${tag}_tests.log
fi
IFS='|' read -ra R <<< "$rows"
for row in "${R[@]}"; do
  [ -z "$row" ] && continue
  timeout 600 python tools/bench_configs.py --only "$row" --steps 3 --warmup 2 2>>gpurun_out/${tag}_rows.err | tee -a gpurun_out/${tag}_rows.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:44].ljust(44), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
done
