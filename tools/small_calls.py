"""dev tool: wall time, GPU busy time and launch count of one compress and one full retrieval of a
small BASELINE config (cfg1 64^3, cfg3 1800x3600), with the host phase marks (IPCG_DEBUG_TIMING)."""
import os, sys, time
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg)
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
for it in range(4):
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches()
    t0 = time.time()
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
    torch.cuda.synchronize()
    t1 = time.time()
    l1 = ctx.kernel_launches()
    plan = ipc.full_plan(r)
    o = ipc.reconstruct_field(r, plan, device=True, keep_session=False)
    torch.cuda.synchronize()
    t2 = time.time()
    l2 = ctx.kernel_launches()
    if it >= 2:
        print(f"cfg{cfg} compress {1e3*(t1-t0):.3f} ms ({l1-l0} launches)  full retrieval {1e3*(t2-t1):.3f} ms ({l2-l1} launches)", flush=True)
