"""Dev probe: one full-fidelity retrieval of cfg2 with per-stream inflate stats (stderr)."""
import os, sys, time
sys.path.insert(0, '.')
os.environ["IPCG_DEBUG_INFLATE"] = "1"
import torch, paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
c = synth.CONFIGS[2]
f = synth.make_field(2)
eb = synth.abs_eb(f, c["rel_eb"])
ft = torch.from_numpy(f).cuda()
r = ipc.compress_field(ft, c["dims"], eb, 1)
out = ipc.reconstruct_field(r, ipc.full_plan(r), device=True)
