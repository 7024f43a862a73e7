python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for G in 0 5; do for row in "context: 50 models x 754-node scene, W=stride" C1; do
  echo "== HGM_WIN_GSH=$G $row"
  HGM_WIN_GSH=$G HGM_LANES=1 HGM_TRACE_W=1 timeout 300 python tools/bench_configs.py --only "$row" --steps 1 --warmup 0 2>&1 | grep -v "^{" | sed -n '1p;6,9p'
done; done
