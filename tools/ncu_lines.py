"""Per-CUDA-line totals (warp instructions executed, stall samples) of an ncu report's
source page, from `ncu -i R --page source --csv --print-source=cuda,sass`.
usage: python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
acc = defaultdict(lambda: [0.0, 0.0])
src = {}
hdr = None
line = None
fname = "?"
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        idx = {n: i for i, n in enumerate(r)}
        ex = idx["Instructions Executed"]
        sm = next(i for i, n in enumerate(r) if n.startswith("Warp Stall Sampling (All"))
        continue
    if not hdr or len(r) < len(hdr):
        continue
    if r[0]:
        line = (fname, int(r[0]))
        src[line] = r[1]
    if line is not None and r[2]:
        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        acc[line][0] += f(r[ex])
        acc[line][1] += f(r[sm])
te = sum(v[0] for v in acc.values()) or 1
ts = sum(v[1] for v in acc.values()) or 1
for ln, (e, s) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln[0][:16]:16s}{ln[1]:5d} {100 * e / te:5.1f}% inst {100 * s / ts:5.1f}% samp | {src.get(ln, '').strip()[:90]}")
