#!/bin/bash
# Final build: all GPU tests, smoke, bench line, launch list of the bench command.
mkdir -p gpurun_out
bash tools/gpu_verify.sh r02ak
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02ak_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02ak_launches_bench.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py gpurun_out/r02ak_launches.csv 14 | tee gpurun_out/r02ak_launches_summary.txt
