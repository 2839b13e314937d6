import sys, time, torch
sys.path.insert(0, '.')
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
c = synth.CONFIGS[2]
f = synth.make_field(2, dims=c["dims"]); eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context.default(); ft = torch.from_numpy(f).cuda()
for i in range(6):
    torch.cuda.synchronize(); t0 = time.time()
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
    torch.cuda.synchronize(); t1 = time.time()
    if i >= 2: print(f"compress {1e3*(t1-t0):.2f} ms")
