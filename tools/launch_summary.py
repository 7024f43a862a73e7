"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_summary.py <launches.csv> [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
idx = {n: i for i, n in enumerate(h)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    k = r[idx["Kernel Name"]].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(r[idx["Metric Value"]].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':62s} {'launches':>8s} {'avg us':>9s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[:62]:62s} {n:8d} {t / n / 1e3:9.1f} {100 * t / tot:5.1f}%")
