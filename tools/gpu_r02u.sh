#!/bin/bash
# Small-problem diagnosis (run under gpurun): source-level ncu of K-DPW on C1 and on the
# context row, launch list (per-kernel durations) of the f2 T=10 and context rows.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for row in "C1" "context: 50 models x 754-node scene, W=stride=60" "f2 single instance 754 nodes, T=10"; do
  timeout 300 python tools/bench_configs.py --only "$row" --steps 3 --warmup 2 2>/dev/null | cut -c1-400
done
timeout 600 bash tools/prof_cfg.sh r02u_win_c1 k_dp_window C1 2 > /dev/null 2>&1; echo "c1 prof rc=$?"
python tools/ncu_lines.py gpurun_out/r02u_win_c1.ncu-rep 70 > gpurun_out/r02u_win_c1_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/r02u_win_c1_raw.csv > gpurun_out/r02u_win_c1_summary.txt 2>&1
head -25 gpurun_out/r02u_win_c1_summary.txt
for row in "f2 single instance 754 nodes, T=10" "context: 50 models x 754-node scene, W=stride=60"; do
  tag=$(echo "$row" | cut -c1-7 | tr ' :' '__')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r02u_launch_$tag.csv python tools/bench_configs.py --only "$row" --steps 1 --warmup 1 \
      > /dev/null 2>&1; echo "launch list $tag rc=$?"
done
rm -f gpurun_out/r02u_win_c1_src.csv
