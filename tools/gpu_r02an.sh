#!/bin/bash
# C4 large T: default tiling vs one 110 KB stage per CTA (2 CTAs/SM).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 900 python tools/bench_configs.py --only "$ROW" --steps 1 --warmup 1 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$ROW', '$*'.ljust(30), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'])"; }
for ROW in "C4 T=80 rho=4" "C4 T=40 rho=4" "C4 T=20 rho=8"; do
  run HGM_X=default; run HGM_SMEM_KB=110 HGM_STAGES=1
done
