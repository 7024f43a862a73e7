#!/bin/bash
# Evidence pass (run under gpurun): launch list of the bench command, ncu --set full of the
# benchmarked K-DP launch and of K-U, roofline traffic regenerated from it.  usage: tools/gpu_evidence.sh <tag>
tag=${1:-ev}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_launches_bench.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py gpurun_out/${tag}_launches.csv 14 | tee gpurun_out/${tag}_launches_summary.txt
timeout 900 bash tools/prof_dp.sh ${tag}_dp k_dp_fused 100 25000 > /dev/null 2>&1; echo "dp ncu rc=$?"
python tools/make_traffic.py gpurun_out/${tag}_dp_raw.csv "ncu --set full, launch 100 of bench.py --steps 1 --warmup 0 --frames-per-gpu 25000, tools/prof_dp.sh" gpurun_out/${tag}_dp_traffic.json
timeout 600 bash tools/prof_dp.sh ${tag}_unary k_unary 0 25000 > /dev/null 2>&1; echo "unary ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_dp_raw.csv > gpurun_out/${tag}_dp_summary.txt 2>&1; head -40 gpurun_out/${tag}_dp_summary.txt
python tools/ncu_summary.py gpurun_out/${tag}_unary_raw.csv > gpurun_out/${tag}_unary_summary.txt 2>&1; head -30 gpurun_out/${tag}_unary_summary.txt
python tools/ncu_lines.py gpurun_out/${tag}_dp.ncu-rep 40 > gpurun_out/${tag}_dp_lines.txt 2>&1
rm -f gpurun_out/${tag}_dp_src.csv gpurun_out/${tag}_dp_cuda.csv gpurun_out/${tag}_unary_src.csv gpurun_out/${tag}_unary_cuda.csv
