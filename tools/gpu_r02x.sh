#!/bin/bash
# K-DPW (eps, x) per-thread variant for NM >= 3; rows; window-path tests; C3 K-DP source profile.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02x_build.log 2>&1 || { tail gpurun_out/r02x_build.log; exit 1; }
for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "context: 50 models x 754-node scene, W=723" "f2 single instance 754 nodes, T=10"; do
  timeout 300 python tools/bench_configs.py --only "$row" --steps 5 --warmup 2 2>/dev/null | cut -c1-330
done
timeout 900 python -m pytest tests -m gpu -q -x -k "window_kernel_paths or c1_all or classify or stream or chains or edge or single_instance_754" > gpurun_out/r02x_tests.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02x_tests.log
timeout 900 bash tools/prof_dp.sh r02x_dp k_dp_fused 10 6000 > /dev/null 2>&1; echo "dp prof rc=$?"
python tools/ncu_summary.py gpurun_out/r02x_dp_raw.csv > gpurun_out/r02x_dp_summary.txt 2>&1; head -22 gpurun_out/r02x_dp_summary.txt
rm -f gpurun_out/r02x_dp_src.csv gpurun_out/r02x_dp_cuda.csv
