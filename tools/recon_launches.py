"""dev tool: the cfg2 bench chain (fresh rel 1e-1 + refines) between cudaProfilerStart/Stop, for
ncu --profile-from-start off launch lists of the retrieval kernels."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

c = synth.CONFIGS[2]
f = synth.make_field(2)
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
rng = r.header().range
rels = [0.1, 0.01, 0.001, 0.0001]
o = ipc.reconstruct_field(r, ipc.plan_for_error(r, rels[0] * rng), device=True)  # warm
torch.cuda.synchronize()
torch.cuda.profiler.start()
o = ipc.reconstruct_field(r, ipc.plan_for_error(r, rels[0] * rng), device=True)
for rel in rels[1:]:
    o = ipc.refine_field(r, o.session, o.values, ipc.plan_for_error(r, rel * rng))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
