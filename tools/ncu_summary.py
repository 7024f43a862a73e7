"""Key counters of an ncu --set full raw CSV page (one kernel launch) and the
per-source-line stall breakdown of the --page source CSV (SASS view).
usage: python tools/ncu_summary.py gpurun_out/<tag>_raw.csv [gpurun_out/<tag>_src.csv]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__cycles_elapsed.avg.per_second", "launch__shared_mem_per_block_dynamic"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
for k in KEYS:
    if k in d:
        print(f"{k:75s} {d[k][0]:>16s} {d[k][1]}")
st = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v]
tot = sum(float(v) for _, v in st) or 1
print("stall samples:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100 * float(v) / tot:.1f}%" for h, v in sorted(st, key=lambda x: -float(x[1]))[:8]))
if len(sys.argv) > 2:
    src = list(csv.reader(open(sys.argv[2])))
    if src[0] and src[0][0] == "Kernel Name":
        src = src[1:]
    h = src[0]
    idx = {n: i for i, n in enumerate(h)}
    # columns: Address, Source, Warp Stall Sampling (All Samples), Instructions Executed ...
    samp = next(n for n in h if n.startswith("Warp Stall Sampling (All"))
    ex = next(n for n in h if n.startswith("Instructions Executed"))
    tot_s = sum(float(r[idx[samp]] or 0) for r in src[1:] if len(r) == len(h))
    tot_e = sum(float(r[idx[ex]] or 0) for r in src[1:] if len(r) == len(h))
    print(f"total samples {tot_s:.0f}, warp instructions executed {tot_e:.0f}")
    base = int(src[1][idx["Address"]], 16)
    # cumulative share by code region (offsets relative to the kernel start; compare with tools/sass_loops.py)
    regions = []
    cur = None
    for r in src[1:]:
        if len(r) != len(h):
            continue
        off = int(r[idx["Address"]], 16) - base
        regions.append((off, float(r[idx[samp]] or 0), float(r[idx[ex]] or 0), r[idx["Source"]].strip()))
    if len(sys.argv) > 3:
        cuts = [int(x, 16) for x in sys.argv[3].split(",")]
        bounds = [0] + cuts + [1 << 40]
        for lo, hi in zip(bounds, bounds[1:]):
            ss = sum(x[1] for x in regions if lo <= x[0] < hi)
            ee = sum(x[2] for x in regions if lo <= x[0] < hi)
            print(f"region [{lo:#x},{hi:#x}): samples {100 * ss / tot_s:5.1f}%  warp-inst {100 * ee / tot_e:5.1f}%")
    top = sorted((r for r in src[1:] if len(r) == len(h)), key=lambda r: -float(r[idx[samp]] or 0))[:25]
    for r in top:
        print(f"{int(r[idx['Address']], 16) - base:#8x} {100 * float(r[idx[samp]] or 0) / tot_s:5.1f}% ex={r[idx[ex]]:>10s}  {r[idx['Source']][:90]}")
