#!/bin/bash
# Final bench line + configuration sweep after the device-memory fix.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/r02ai_bench.json 2> gpurun_out/r02ai_bench.err; echo "bench rc=$?"
timeout 1500 python tools/bench_configs.py > gpurun_out/r02ai_configs.jsonl 2> gpurun_out/r02ai_configs.err; echo "configs rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/r02ai_bench.json")); r=d["roofline"]
print("C3", round(d["value"]), round(d["ms_per_step"],2), round(r["frac"],4), round(r["xu_frac"],4), "e2e", round(d["e2e"]["value"]), d["clocks"])
for ln in open("gpurun_out/r02ai_configs.jsonl"):
    d = json.loads(ln)
    print(d["config"][:40].ljust(40), d["pairs_per_s"], d["ms_per_call"], d["frac"], d["frac_wall"], d["kernel_ms"])
PY
