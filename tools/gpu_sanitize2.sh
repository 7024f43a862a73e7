#!/bin/bash
# Targeted compute-sanitizer runs per K-DP path (run under gpurun): racecheck and initcheck on
# small cases with the per-window kernel (HGM_DP=window) and the per-step kernel (HGM_DP=fused).
# usage: tools/gpu_sanitize2.sh <tag>
tag=${1:-san2}
mkdir -p gpurun_out
python -c "from paper_1505_00581_b200 import build as B; B.build()"
S=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool path cases...
  tool=$1; dp=$2; shift 2
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  log=gpurun_out/${tag}_${tool}_${dp}.log
  HGM_DP=$dp timeout 1500 $S --tool $tool $extra --print-limit 20 python tools/sanitize_cases.py "$@" > $log 2>&1
  rc=$?
  echo "$tool HGM_DP=$dp cases [$*] exit=$rc: $(grep -c 'Error\|Uninitialized' $log) reports; $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tail -1)" | tee -a gpurun_out/${tag}_summary.txt
  grep -h "^=========     \(Write\|Read\|at \)" $log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -6 | tee -a gpurun_out/${tag}_summary.txt
}
run racecheck window c0 c1 lanes
run racecheck fused c0 c1
run initcheck fused c0 c1 c2
run initcheck window c0 c1
