#!/bin/bash
# Large-T tiling rule A/B: new default (110 KB single stage, 2 CTAs/SM) vs the previous rule
# (HGM_SMEM_KB=220 HGM_STAGES=1 = one 220 KB stage per SM); single-instance T sweep; tests.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  echo "== new"; PYTHONPATH=. timeout 600 python tools/bench_single.py --T 160 320 724 --steps 10 2>/dev/null | cut -c1-200
  echo "== old"; HGM_SMEM_KB=220 HGM_STAGES=1 PYTHONPATH=. timeout 600 python tools/bench_single.py --T 160 320 724 --steps 10 2>/dev/null | cut -c1-200
done
timeout 900 python -m pytest tests -m gpu -q -x -k "single_instance or tile_sizes or dense_fallbacks" 2>&1 | tail -2
