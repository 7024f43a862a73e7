#!/bin/bash
# PDL only for a stream running alone: C4 T=80/40 (two chunk lanes), context W=723 (7 lanes), f2, C3.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for row in "C4 T=80 rho=4" "C4 T=40 rho=4" "context: 50 models x 754-node scene, W=723" "f2 single instance 754 nodes, T=10" "C4 T=10 rho=4"; do
  timeout 600 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:34].ljust(34), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
done
timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']
print('C3 ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'xu', round(r.get('xu_frac',0),4))"
