#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_cases.py (run under gpurun)
# usage: tools/gpu_sanitize.sh <tag> [cases...]
tag=${1:-san}; shift
cases="$@"
mkdir -p gpurun_out
python -c "from paper_1505_00581_b200 import build as B; B.build()"
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 700 $S --tool $tool $extra --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py $cases \
     > gpurun_out/${tag}_$tool.log 2>&1
  echo "$tool exit=$?" | tee -a gpurun_out/${tag}_summary.txt
  tail -3 gpurun_out/${tag}_$tool.log >> gpurun_out/${tag}_summary.txt
done
