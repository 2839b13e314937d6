"""Per-CUDA-source-line stall samples and instructions of a kernel in an ncu report (cuda,sass
view; SASS rows are attributed to the preceding source line); dev tool.
usage: ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
fname = ""
cur_line = "-1"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    if r[0].strip().isdigit():
        cur_line = r[0].strip()
    line = cur_line if r[0].strip() == "" else r[0]
    num = lambda x: int(x) if x and x.strip().isdigit() else 0
    st = num(d.get("Warp Stall Sampling (All Samples)"))
    ins = num(d.get("Instructions Executed"))
    key = (fname, int(line) if line.isdigit() else -1)
    agg[key][0] += st
    agg[key][1] += ins
    if r[1].strip():
        agg[key][2] = r[1].strip()[:100]
S = sum(v[0] for v in agg.values()) or 1
I = sum(v[1] for v in agg.values()) or 1
print(f"samples {S} instructions {I}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:<5} {100*v[0]/S:5.1f}%s {100*v[1]/I:5.1f}%i  {v[2]}")
