python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1 || { tail gpurun_out/r02l_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "tile_sizes or row_tails or c4_shaped or single_instance or dense_fallbacks" > gpurun_out/r02l_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r02l_tests.log
for RT in 0 1; do
  for row in "C4 T=40 rho=4" "C4 T=80 rho=4" "f2 single instance 754 nodes, T=inf" "C4 T=20 rho=8"; do
    HGM_RT=$RT timeout 900 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>>gpurun_out/r02l_rows.err | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('RT=$RT', d['config'][:40].ljust(40), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
  done
done | tee gpurun_out/r02l_rows.txt
HGM_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --frames-per-gpu 6000 2>&1 >/dev/null | grep -A70 HGM_TRACE | head -75 > gpurun_out/r02l_kdp_trace.txt
head -40 gpurun_out/r02l_kdp_trace.txt
