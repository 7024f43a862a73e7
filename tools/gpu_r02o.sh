python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1 || { tail gpurun_out/r02o_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "tile_sizes or c4_shaped or single_instance or dense_fallbacks or model_batched or c4_sampled" > gpurun_out/r02o_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r02o_tests.log
for row in "C4 T=40 rho=4" "C4 T=80 rho=4" "f2 single instance 754 nodes, T=inf" "C4 T=20 rho=8" "C4 T=10" "C2"; do
  timeout 900 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>>gpurun_out/r02o_rows.err | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:40].ljust(40), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
done | tee gpurun_out/r02o_rows.txt
