"""Per-SASS-instruction profile (largest launch of a kernel) from an ncu report; dev tool.
usage: ncu_sass.py report.ncu-rep kernel_regex [min_pct]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
minp = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
best = None
for k, s in enumerate(hi):
    e = hi[k + 1] if k + 1 < len(hi) else len(rows)
    h = rows[s]
    sec = [dict(zip(h, r)) for r in rows[s + 1:e] if r and r[0].startswith("0x")]
    tot = sum(int(d.get("Instructions Executed") or 0) for d in sec)
    if best is None or tot > best[0]:
        best = (tot, sec)
tot, sec = best
S = sum(int(d.get("Warp Stall Sampling (All Samples)") or 0) for d in sec) or 1
print(f"instructions {tot}  samples {S}  sass lines {len(sec)}")
for d in sec:
    ins = int(d.get("Instructions Executed") or 0)
    st = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    if 100 * st / S >= minp or 100 * ins / max(tot, 1) >= minp:
        print(f"{d['Address'][-5:]} {100*ins/max(tot,1):5.2f}%i {100*st/S:5.2f}%s thr={d.get('Avg. Threads Executed'):>5} {d['Source'][:90]}")
