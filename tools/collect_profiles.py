"""dev tool: assemble profiles/r02_* from the outputs of tools/profile_round3.sh (gpurun_out/p3).
   python tools/collect_profiles.py [gpurun_out/p3]"""
import csv
import glob
import json
import os
import shutil
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/p3"
dst = "profiles"
tag = "r02"


def last_json_line(path):
    lines = [l for l in open(path).read().splitlines() if l.strip().startswith("{")]
    return json.loads(lines[-1])


for name in ("bench", "bench_reference"):
    json.dump(last_json_line(f"{src}/{name}.json"), open(f"{dst}/{tag}_{name}.json", "w"), indent=1)
shutil.copy(f"{src}/configs.jsonl", f"{dst}/{tag}_configs.jsonl")
shutil.copy(f"{src}/launches_summary.txt", f"{dst}/{tag}_launches_summary.txt")
keep = [l for l in open(f"{src}/match_traffic.csv") if not l.startswith("==PROF==")]
open(f"{dst}/{tag}_match_traffic.csv", "w").writelines(keep)

with open(f"{dst}/{tag}_ncu_full_summary.txt", "w") as out:
    for p in sorted(glob.glob(f"{src}/*.summary.txt")):
        name = os.path.basename(p)[: -len(".summary.txt")]
        out.write(f"# {name} (tools/profile_round3.sh: --set full of one launch; k_*_6 = level 1 of a cfg2 compress, "
                  f"*_0 = first inflate of its full retrieval)\n")
        out.write(open(p).read().rstrip() + "\n\n")

# DRAM traffic per family: tools/compress_once.py runs two compresses, the second is counted
rows = list(csv.reader(l for l in keep if l.startswith('"')))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = {}  # launch id -> (kernel, {metric: value})
for r in rows[1:]:
    kid = int(r[0])
    per.setdefault(kid, [r[ki], {}])[1][r[mi]] = float(r[vi].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}[r[ui]]
traffic = {}
for fam, kern, what in (("deflate.match", "k_match", "k_match launches (one per level)"),
                        ("deflate.walk", "k_od_walk", "k_od_walk launches (the levels whose streams take the on-demand parse)")):
    ls = [v for k, v in sorted(per.items()) if kern + "<" in v[0] or kern + "(" in v[0]]
    ls = ls[len(ls) // 2:]  # the second compress
    rd = sum(v[1].get("dram__bytes_read.sum", 0) for v in ls)
    wr = sum(v[1].get("dram__bytes_write.sum", 0) for v in ls)
    ns = sum(v[1].get("gpu__time_duration.sum", 0) for v in ls)
    traffic[fam] = {"dram_bytes": int(rd + wr), "read": int(rd), "write": int(wr), "ms_cold": round(ns / 1e6, 3),
                    "launches": len(ls),
                    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the {len(ls)} {what} of one cfg2 "
                              f"compress (profiles/{tag}_match_traffic.csv; tools/compress_once.py runs two, the second counted)"}
json.dump(traffic, open(f"{dst}/{tag}_traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
