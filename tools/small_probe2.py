"""dev tool: host phases (IPCG_DEBUG_TIMING) and device span of a small-field compress/retrieve."""
import os, sys, time
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg)
eb = synth.abs_eb(f, c["rel_eb"])
ft = torch.from_numpy(f).cuda()
ctx = ipc.Context(0)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    o = ipc.reconstruct_field(r, ipc.full_plan(r), device=True, keep_session=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"compress {1e3*(t1-t0):.2f} ms  retrieve {1e3*(t2-t1):.2f} ms  launches {ctx.kernel_launches()}", flush=True)
