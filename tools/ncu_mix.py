"""dev tool: instruction mix + stall samples by opcode from an ncu report's SASS source page.
    python tools/ncu_mix.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
r = csv.reader(out)
next(r)
h = next(r)
rows = list(r)
ie, src, smp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[ie] or 0) for x in rows)
c, cs = Counter(), Counter()
for x in rows:
    t = x[src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    c[op] += int(x[ie] or 0)
    cs[op] += int(x[smp] or 0)
print("warp instructions", tot, "samples", sum(cs.values()))
for k, v in c.most_common(top):
    print(f"{k:8s} {v:12d} {100 * v / tot:5.1f}%  stall-samples {cs[k]}")
