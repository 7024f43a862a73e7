python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "single_instance or c4_shaped" > gpurun_out/r02p_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02p_tests.log
for row in "f2 single instance 754 nodes, T=inf" "C4 T=80 rho=4" "C4 T=20 rho=8" "C4 T=40 rho=4"; do
  timeout 900 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:40].ljust(40), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
done
