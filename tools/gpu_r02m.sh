python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HGM_DEBUG_TILING=1 HGM_TRACE=1 timeout 300 python tools/bench_configs.py --only "f2 single instance 754 nodes, T=inf" --steps 1 --warmup 0 2>&1 | grep -v "^{" | head -60
HGM_DEBUG_TILING=1 HGM_TRACE=1 timeout 300 python tools/bench_configs.py --only "C4 T=80 rho=4" --steps 1 --warmup 0 2>&1 | grep -v "^{" | head -50
