"""dev tool: IPCG_DEBUG_TIMELINE marks of one cfg2 compress (q<l> quant done, m<l> match search
enqueued/done, d<l> deflate done, L<l> loss table done), ms from the start."""
import os, sys
os.environ["IPCG_DEBUG_TIMELINE"] = "1"
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
c = synth.CONFIGS[2]
f = synth.make_field(2)
eb = synth.abs_eb(f, c["rel_eb"])
ft = torch.from_numpy(f).cuda()
ctx = ipc.Context(0)
for _ in range(3):
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
torch.cuda.synchronize()
