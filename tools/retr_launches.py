"""dev tool: one compress (untimed) then ONE fresh full retrieval of a config, for an ncu launch list of
the retrieval kernels only (profile with --nvtx-free range: cudaProfilerStart/Stop around the call).
   ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file X python tools/retr_launches.py CFG"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg, seed=0)
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
ipc.reconstruct_field(r, ipc.full_plan(r), device=True, keep_session=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ipc.reconstruct_field(r, ipc.full_plan(r), device=True, keep_session=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
