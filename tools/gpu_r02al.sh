#!/bin/bash
# f2 T=+inf tiling knobs under PDL (A/B): default (one 220 KB stage per SM) vs smaller / double stages.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/bench_configs.py --only "f2 single instance 754 nodes, T=inf" --steps 5 --warmup 2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$*'.ljust(34), 'ms', d['ms_per_call'], 'frac', d['frac'], d['kernel_ms'])"; }
for rep in 1 2; do
run HGM_X=default
run HGM_SMEM_KB=110
run HGM_SMEM_KB=110 HGM_STAGES=1
run HGM_SMEM_KB=220 HGM_STAGES=2
run HGM_SMEM_KB=150 HGM_STAGES=1
done
