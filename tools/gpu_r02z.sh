#!/bin/bash
# Verification of e4d52c1: all GPU tests (incl. the compute-sanitizer test), racecheck of the
# per-window (K-DPW) and per-step (K-DP) paths on C0, smoke, bench line.
mkdir -p gpurun_out
bash tools/gpu_verify.sh r02z
S=/usr/local/cuda/bin/compute-sanitizer
for dp in window fused; do
  HGM_DP=$dp timeout 1200 $S --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py c0 > gpurun_out/r02z_racecheck_$dp.log 2>&1
  echo "racecheck HGM_DP=$dp c0 exit=$?: $(grep 'RACECHECK SUMMARY\|ERROR SUMMARY' gpurun_out/r02z_racecheck_$dp.log | tail -1) $(grep -c 'case c0 ok' gpurun_out/r02z_racecheck_$dp.log)"
done
