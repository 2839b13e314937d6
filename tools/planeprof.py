"""Dev tool: per-plane deflate family timings of cfg2's level-1 planes (one stream per call)."""
import json, sys, zlib
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
level = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg, seed=0, dims=c["dims"], device="cuda:0")
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
arch = r.to_bytes()
rec = r.record(level)
ib = r.index_bytes()
planes = []
for p in range(32):
    off = ib + rec.plane_offset[p]
    be = arch[off]
    ln = int.from_bytes(arch[off + 9:off + 17], 'little')
    pay = arch[off + 21:off + 21 + ln]
    raw = zlib.decompress(pay) if be == 1 else pay
    planes.append(np.frombuffer(raw, np.uint8))
n = len(planes[0])
print("plane bytes", n)
tot = {}
for p, pl in enumerate(planes):
    nz = int(np.count_nonzero(pl))
    if nz == 0:
        continue
    ipc.backend_encode(pl, ctx=ctx)  # warm
    ctx.profile(True)
    res = ipc.backend_encode(pl, ctx=ctx)
    prof = ctx.profile_read()
    ctx.profile(False)
    ms = {k: round(v["ms"], 3) for k, v in prof.items()}
    for k, v in ms.items():
        tot[k] = tot.get(k, 0) + v
    print(p, f"nz {nz/n:.3f} be {res[0][0]} ratio {len(res[0][1])/n:.3f}", json.dumps(ms), flush=True)
print("total", json.dumps({k: round(v, 2) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}))
if len(sys.argv) > 3 and sys.argv[3] != "-":  # save the named planes for CPU-side analysis
    for p in sys.argv[3].split(','):
        np.save(f"gpurun_out/plane_l{level}_{p}.npy", planes[int(p)])
if len(sys.argv) > 4 and sys.argv[4] == "inflate":  # per-plane inflate family timings
    tot = {}
    for p in range(32):
        off = ib + rec.plane_offset[p]
        be = arch[off]
        ln = int.from_bytes(arch[off + 9:off + 17], 'little')
        crc = int.from_bytes(arch[off + 17:off + 21], 'little')
        pay = arch[off + 21:off + 21 + ln]
        if be != 1 or not np.count_nonzero(planes[p]):
            continue
        blk = [(be, pay, crc, len(planes[p]))]
        ipc.backend_decode(blk, ctx=ctx)
        ctx.profile(True)
        res = ipc.backend_decode(blk, ctx=ctx)
        prof = ctx.profile_read()
        ctx.profile(False)
        assert res[0] == planes[p].tobytes()
        ms = {k: round(v["ms"], 3) for k, v in prof.items()}
        for k, v in ms.items():
            tot[k] = tot.get(k, 0) + v
        print("inflate", p, f"comp {ln} syms?", json.dumps(ms), flush=True)
    print("inflate total", json.dumps({k: round(v, 2) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}))
