#!/bin/bash
# A/B timing of prebuilt variants (tools/ab_build.sh): C3 bench (short), C2, C4 T=20 / T=40.
# usage: tools/ab_run.sh <tag> variant...   ("default" = lib/libhgm.so)
tag=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then unset HGM_LIB; else export HGM_LIB=$PWD/paper_1505_00581_b200/lib/libhgm_$v.so; fi
  echo "== $v" >> gpurun_out/${tag}_ab.txt
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']
print('C3 ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'xu', round(r.get('xu_frac',0),4))" >> gpurun_out/${tag}_ab.txt
  for row in "C2" "C4 T=20 rho=4" "C4 T=40 rho=4"; do
    timeout 600 python tools/bench_configs.py --only "$row" --steps 2 --warmup 1 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:30], 'ms', d['ms_per_call'], 'frac', d['frac'], 'wall', d['frac_wall'], d['kernel_ms'])" >> gpurun_out/${tag}_ab.txt
  done
done
cat gpurun_out/${tag}_ab.txt
