python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/ab_build.sh minb3 "-DHGM_KDP_MINB=3" nolpt "-DHGM_NO_LPT" > /dev/null 2>&1
run() {  # variant smem_kb
  if [ $1 = default ]; then unset HGM_LIB; else export HGM_LIB=$PWD/paper_1505_00581_b200/lib/libhgm_$1.so; fi
  HGM_SMEM_KB=$2 timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$1 smem $2 C3 ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'dp ms', round(r['dp_ms_per_step'],1), 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2; do run default 110; run nolpt 110; run minb3 110; run minb3 72; done
