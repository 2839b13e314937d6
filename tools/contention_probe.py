"""dev tool: does a concurrent bulk D2H (the host-async copy-outs) slow compress?  Times
compress of the cfg2 field (device input, then pinned host input) alone and while a torch
D2H of 2 GB runs on another stream."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

c = synth.CONFIGS[2]
f = synth.make_field(2)
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
hf = torch.from_numpy(f).pin_memory()
big_d = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
big_h = torch.empty(2 << 30, dtype=torch.uint8).pin_memory()
side = torch.cuda.Stream()
for src, name in ((ft, "device"), (hf, "host")):
    for conc in (False, True, False, True):
        torch.cuda.synchronize()
        if conc:
            with torch.cuda.stream(side):
                big_h.copy_(big_d, non_blocking=True)
        t0 = time.time()
        r = ipc.compress_field(src, c["dims"], eb, c["interp"], ctx=ctx)
        t1 = time.time()
        torch.cuda.synchronize()
        t2 = time.time()
        print(f"{name:6s} concurrent D2H {conc!s:5s}: compress {1e3*(t1-t0):.2f} ms (D2H drained at {1e3*(t2-t0):.1f} ms)")
