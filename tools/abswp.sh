# A/B sweep of K-DP block-size builds x tile frames (device-input bench)
for lib in lib_t256_b4 lib_t128_b6 lib_t128_b8; do
  for ft in 3 4 6; do
    echo "$lib FT $ft"
    HGM_LIB=paper_1505_00581_b200/$lib/libhgm.so HGM_TILE_FRAMES=$ft timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['frac'],3), 'dp', round(d['roofline']['kernel_ms']['dp'],1), 'bt', round(d['roofline']['kernel_ms']['backtrack'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
