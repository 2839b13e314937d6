"""Dev/profiling driver: one warm-up + one compress (+ optional full retrieval) of a BASELINE config."""
import sys
sys.path.insert(0, '.')
import torch, paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "compress"
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg)
eb = synth.abs_eb(f, c["rel_eb"])
ft = torch.from_numpy(f).cuda()
r = ipc.compress_field(ft, c["dims"], eb, c["interp"])
if mode == "compress":
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"])
else:
    out = ipc.reconstruct_field(r, ipc.full_plan(r), device=True)
torch.cuda.synchronize()
print("ok", r.size())
