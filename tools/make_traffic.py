"""Regenerate profiles/dp_traffic.json (bench.py's roofline.traffic) from the raw page of
an `ncu --set full` capture of one K-DP launch of the benchmarked build.
usage: python tools/make_traffic.py <raw.csv> <description of the capture> [out.json]"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def nbytes(key):
    v = float(d[key].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u[key], 1)
    return int(round(v * scale))


rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
kern = d.get("Kernel Name", "k_dp_fused")
out = dict(kernel=kern, dram_bytes_per_launch=rd + wr, dram_read=rd, dram_write=wr,
           duration=d.get("gpu__time_duration.sum"), duration_unit=u.get("gpu__time_duration.sum"),
           source=f"{sys.argv[1]} ({sys.argv[2]})")
path = sys.argv[3] if len(sys.argv) > 3 else "profiles/dp_traffic.json"
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
