"""Dev tool: decode one level-1 plane of cfg2 (its deflate block) a few times, for launch lists."""
import sys, zlib
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

cfg, level = 2, 1
planes_wanted = [int(p) for p in sys.argv[1].split(',')] if len(sys.argv) > 1 else [21]
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg, seed=0, dims=c["dims"], device="cuda:0")
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
r = ipc.compress_field(torch.from_numpy(f).cuda(), c["dims"], eb, c["interp"], ctx=ctx)
arch = r.to_bytes()
rec = r.record(level)
ib = r.index_bytes()
blks = []
for p in planes_wanted:
    off = ib + rec.plane_offset[p]
    be = arch[off]
    ln = int.from_bytes(arch[off + 9:off + 17], 'little')
    crc = int.from_bytes(arch[off + 17:off + 21], 'little')
    pay = arch[off + 21:off + 21 + ln]
    n = len(zlib.decompress(pay)) if be == 1 else ln
    blks.append((be, pay, crc, n))
for _ in range(3):
    ipc.backend_decode(blks, ctx=ctx)
torch.cuda.synchronize()
print("ok", [len(b[1]) for b in blks])
