#!/bin/bash
# ncu --set full capture of one launch of a kernel while tools/bench_configs.py runs one
# configuration row (run under gpurun).  usage: tools/prof_cfg.sh <tag> <kernel-regex> <row-substring> [skip]
tag=${1:-cfg}; pat=${2:-k_dp_window}; row=${3:-C1}; skip=${4:-2}
mkdir -p gpurun_out
python -c "from paper_1505_00581_b200 import build as B; B.build()"
ncu --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 1 \
    -o gpurun_out/$tag -f python tools/bench_configs.py --only "$row" --steps 1 --warmup 1 \
    > gpurun_out/$tag.ncu.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out/$tag*
