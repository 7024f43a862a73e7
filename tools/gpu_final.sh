#!/bin/bash
# Round-end evidence (run under gpurun): all GPU tests, smoke, bench line, §8(d) config sweep,
# launch list, ncu --set full of the benchmarked K-DP launch, of K-DPW (C1) and of K-U.
tag=${1:-fin}
mkdir -p gpurun_out
bash tools/gpu_verify.sh $tag
timeout 1500 python tools/bench_configs.py > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err; echo "configs rc=$?"
python - <<PY
import json
for ln in open("gpurun_out/${tag}_configs.jsonl"):
    d = json.loads(ln)
    print(d["config"][:50].ljust(50), "ms", d["ms_per_call"], "frac", d["frac"], "wall", d["frac_wall"])
PY
bash tools/gpu_evidence.sh $tag
timeout 600 bash tools/prof_cfg.sh ${tag}_win_c1 k_dp_window C1 1 > /dev/null 2>&1; echo "win ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_win_c1_raw.csv > gpurun_out/${tag}_win_c1_summary.txt 2>&1; head -25 gpurun_out/${tag}_win_c1_summary.txt
rm -f gpurun_out/${tag}_win_c1_src.csv
