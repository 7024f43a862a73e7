#!/bin/bash
# A/B of the K-DPW trip-sorted task list + K-DP programmatic dependent launch; GPU tests of
# the touched paths; source-level ncu of K-DPW on C1.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02v_build.log 2>&1 || { tail gpurun_out/r02v_build.log; exit 1; }
for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "f2 single instance 754 nodes, T=10" "C4 T=10 rho=4"; do
  timeout 300 python tools/bench_configs.py --only "$row" --steps 3 --warmup 2 2>/dev/null | cut -c1-330
done
echo "--- HGM_PDL=0"
for row in "f2 single instance 754 nodes, T=10" "C4 T=10 rho=4"; do
  HGM_PDL=0 timeout 300 python tools/bench_configs.py --only "$row" --steps 3 --warmup 2 2>/dev/null | cut -c1-330
done
timeout 900 python -m pytest tests -m gpu -q -x -k "window_kernel_paths or c1_all or single_instance_754 or tiled_kernel or c0_T10 or model_batched or c4_shaped or dense_fallbacks" > gpurun_out/r02v_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02v_tests.log
timeout 600 bash tools/prof_cfg.sh r02v_win_c1 k_dp_window C1 1 > /dev/null 2>&1; echo "c1 prof rc=$?"
python tools/ncu_lines.py gpurun_out/r02v_win_c1.ncu-rep 80 > gpurun_out/r02v_win_c1_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/r02v_win_c1_raw.csv > gpurun_out/r02v_win_c1_summary.txt 2>&1
head -22 gpurun_out/r02v_win_c1_summary.txt
rm -f gpurun_out/r02v_win_c1_src.csv
