import sys; sys.path.insert(0,'.')
import torch, paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
cfg=int(sys.argv[1]); c=synth.CONFIGS[cfg]; f=synth.make_field(cfg); eb=synth.abs_eb(f,c["rel_eb"])
ctx=ipc.Context(0); ft=torch.from_numpy(f).cuda()
r=ipc.compress_field(ft,c["dims"],eb,c["interp"],ctx=ctx)
o=ipc.reconstruct_field(r, ipc.full_plan(r), device=True, keep_session=False)
torch.cuda.synchronize()
