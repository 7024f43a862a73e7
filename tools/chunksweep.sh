# tuning sweep: windows per chunk (device-input bench, no e2e / oracle)
for c in 4096 2048 1024 512; do
  echo "chunk $c"
  HGM_CHUNK=$c timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['frac'],3), {k: round(v,1) for k,v in d['roofline']['kernel_ms'].items()})"
done
