#!/bin/bash
# A/B K-DPW static task dealing; descriptor scratch; rows + lane tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for v in default kstatic; do
  if [ $v = default ]; then unset HGM_LIB; else export HGM_LIB=$PWD/paper_1505_00581_b200/lib/libhgm_$v.so; fi
  for row in "C1" "context: 50 models x 754-node scene, W=stride=60"; do
    timeout 300 python tools/bench_configs.py --only "$row" --steps 5 --warmup 2 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'][:34].ljust(34), 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])"
  done
done
done
unset HGM_LIB
for r in "context W=60" "f2" "context W=723"; do timeout 300 python tools/ctx_probe.py "$r" 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "window_kernel or stream or detect or c4_shaped or dense_fallbacks or single_instance_754 or c1_all" 2>&1 | tail -2
