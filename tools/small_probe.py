import sys, time
sys.path.insert(0, '.')
import torch, paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
cfg = int(sys.argv[1])
c = synth.CONFIGS[cfg]; f = synth.make_field(cfg); eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
plan = ipc.full_plan(r)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    o = ipc.reconstruct_field(r, plan, device=True, keep_session=False)
    torch.cuda.synchronize(); t1 = time.time()
    print("wall", (t1 - t0) * 1e3, flush=True)
ctx.profile(True)
o = ipc.reconstruct_field(r, plan, device=True, keep_session=False)
import json; print(json.dumps({k: round(v["ms"], 3) for k, v in ctx.profile_read().items()}))
