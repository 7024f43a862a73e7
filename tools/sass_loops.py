"""Instruction mix of the hot loops of a kernel in libhgm.so (cuobjdump -sass):
every backward branch whose body holds >= MIN_MUFU MUFU.SQRT is reported with its
opcode histogram.  Usage: python tools/sass_loops.py <kernel-substring> [min_mufu]"""
import re
import subprocess
import sys
from collections import Counter

lib = "paper_1505_00581_b200/lib/libhgm.so"
pat = sys.argv[1] if len(sys.argv) > 1 else "k_dp_fused"
min_mufu = int(sys.argv[2]) if len(sys.argv) > 2 else 6
s = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", s):
    name = f.split("\n", 1)[0]
    if pat not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    for a, t in ins:
        m = re.match(r"(@!?U?P\w+\s+)?BRA (0x[0-9a-f]+)", t)
        if m and int(m.group(2), 16) < a:
            tgt = int(m.group(2), 16)
            body = [x for x in ins if tgt <= x[0] <= a]
            nm = sum("MUFU.SQRT" in x[1] for x in body)
            if nm >= min_mufu and len(body) < 300:
                ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0] for x in body)
                print(name[:70], hex(tgt), hex(a), "instructions", len(body), "MUFU.SQRT", nm)
                print("   ", dict(ops.most_common()))
