# tuning sweep: windows per chunk x streams (device-input bench, no e2e / oracle)
for cfg in "891 1" "256 1" "128 1" "256 2" "128 2" "64 2"; do
  set -- $cfg
  echo "chunk $1 streams $2"
  HGM_CHUNK=$1 HGM_STREAMS=$2 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['frac'],3), {k: round(v,1) for k,v in d['roofline']['kernel_ms'].items() if v > 0.5})"
done
