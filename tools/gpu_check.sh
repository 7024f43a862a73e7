#!/bin/bash
# One GPU session (run under gpurun): build, GPU tests, smoke, bench, config sweep.
# usage: tools/gpu_check.sh <tag> [pytest -k expr]
tag=${1:-chk}; kexpr=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo build failed; tail gpurun_out/${tag}_build.log; exit 1; }
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_gpu_tests.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1
fi
echo "pytest rc=$?"; tail -15 gpurun_out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/${tag}_bench.json
timeout 900 python tools/bench_configs.py > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err; echo "configs rc=$?"
timeout 900 python tools/bench_configs.py --dp fused > gpurun_out/${tag}_configs_fused.jsonl 2>> gpurun_out/${tag}_configs.err; echo "configs(fused) rc=$?"
python - <<PY
import json
for f in ("gpurun_out/${tag}_configs.jsonl", "gpurun_out/${tag}_configs_fused.jsonl"):
    for ln in open(f):
        d = json.loads(ln)
        print(d["dp_path"], d["config"][:48].ljust(48), "ms", d["ms_per_call"], "frac", d["frac"], "wall", d["frac_wall"])
PY
