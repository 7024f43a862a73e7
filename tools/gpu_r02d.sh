set -x
python -c "from paper_1505_00581_b200 import build as B; B.build()" > /dev/null
bash tools/ab_build.sh base "-DHGM_SQRT_SPLIT=0 -DHGM_TRIP_SORT=0" sort "-DHGM_SQRT_SPLIT=0 -DHGM_TRIP_SORT=1" split "-DHGM_SQRT_SPLIT=1 -DHGM_TRIP_SORT=0" > /dev/null
bash tools/ab_run.sh r02d base sort split default
for L in 1 8; do HGM_LANES=$L timeout 300 python tools/bench_configs.py --only context --steps 3 --warmup 2 > gpurun_out/r02d_ctx_lanes$L.jsonl 2>&1; done
cut -c1-400 gpurun_out/r02d_ctx_lanes*.jsonl
timeout 600 bash tools/prof_cfg.sh r02d_win_c1 k_dp_window C1 1
