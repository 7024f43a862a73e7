#!/bin/bash
# A/B of the alpha-history chunk budget (HGM_HIST_GB): C3 bench, C2, C4 T=20.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for gb in 6 24 12; do
  HGM_HIST_GB=$gb timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']
print('hist $gb GB C3 ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), {k: round(v,2) for k,v in r['kernel_ms'].items() if v})"
  for row in "C2" "C4 T=20 rho=4"; do
    HGM_HIST_GB=$gb timeout 600 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('hist $gb GB', d['config'][:20], 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'])"
  done
done
done
