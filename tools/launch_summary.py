"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel; dev tool."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki]).split("::")[-1].split("<")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
mine = sum(v for k, v in tot.items() if k.startswith("k_"))
print(f"# {sys.argv[1]}: {sum(cnt.values())} launches, {T:.1f} ms total (cold-cache, serialised)")
print(f"# own kernels (k_*): {mine:.1f} ms = {100 * mine / T:.1f}%")
print(f"{'kernel':34s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k:34s} {cnt[k]:8d} {v:10.2f} {100 * v / T:6.1f}%")
