"""TEST PROGRAM for tests/test_sanitizer.py: one small pass over every device path (compress with
outliers and non-finite values, partial and full reconstruction, refinement, session file
round trip, metrics, backend encode/decode incl. a corrupt block, bitplane ops), run under
compute-sanitizer.  Prints OK on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

ctx = ipc.Context(0)
for dims, interp, dt in (((20, 24, 18), 1, np.float32), ((33, 21), 0, np.float64), ((257,), 1, np.float32)):
    f = synth.smooth_field(dims, 3).astype(dt)
    f.reshape(-1)[::97] += 50.0  # spikes -> outliers
    f.reshape(-1)[5] = np.nan
    eb = 1e-3 * float(np.nanmax(f) - np.nanmin(f))
    r = ipc.compress_field(f, dims, eb, interp, ctx=ctx)
    arch = r.to_bytes()
    rd = ipc.ArchiveReader(arch, ctx=ctx)
    p1 = [0 if l + 1 <= rd.header().progressive_levels else 32 for l in range(rd.levels)]
    a = ipc.reconstruct_field(rd, p1)
    b = ipc.refine_field(rd, a.session, a.values, ipc.full_plan(rd))
    c = ipc.reconstruct_field(rd, ipc.full_plan(rd))
    assert b.values.tobytes() == c.values.tobytes()
    s = ipc.write_session(a.session)
    ipc.read_session(s, rd)
    ipc.compute_metrics(np.nan_to_num(f), np.nan_to_num(c.values), ctx=ctx)
rng = np.random.default_rng(1)
planes = (rng.random((3, 5000)) < 0.05).astype(np.uint8)
enc = ipc.backend_encode(planes, ctx=ctx)
blocks = [(be, pl, crc, 5000) for be, pl, crc in enc]
bad = bytearray(blocks[0][1])
bad[len(bad) // 2] ^= 0x5A
blocks.append((blocks[0][0], bytes(bad), blocks[0][2], 5000))
out = ipc.backend_decode(blocks, ctx=ctx)
assert out[0] == planes[0].tobytes() and isinstance(out[-1], Exception)
print("OK")
