#!/bin/bash
# ncu --set full capture of one mid-run K-DP launch of a short C3 bench (run under gpurun).
# usage: tools/prof_dp.sh <tag> [kernel-regex] [launch-skip]
tag=${1:-dp}; pat=${2:-k_dp_fused}; skip=${3:-10}; frames=${4:-6000}
mkdir -p gpurun_out
python -c "from paper_1505_00581_b200 import build as B; B.build()"
ncu --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 1 \
    -o gpurun_out/$tag -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --frames-per-gpu $frames \
    > gpurun_out/$tag.ncu.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=cuda > gpurun_out/${tag}_cuda.csv 2>/dev/null
ls -la gpurun_out/$tag*
