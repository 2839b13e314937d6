"""Dev tool: per-family device timings of bench.py's retrieval chain (reconstruct + refines)."""
import json, sys
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
c = synth.CONFIGS[2]
f = synth.make_field(2, seed=0, dims=c["dims"], device="cuda:0")
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ft = torch.from_numpy(f).cuda()
rels = c["retrieve"]["rel"]
r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
rng = r.header().range
for it in range(2):
    o = None
    for i, rel in enumerate(rels):
        plan = ipc.plan_for_error(r, rel * rng)
        ctx.profile(True)
        o = ipc.reconstruct_field(r, plan, device=True) if i == 0 else ipc.refine_field(r, o.session, o.values, plan)
        prof = ctx.profile_read()
        ctx.profile(False)
        if it == 1:
            print(rel, plan.k, json.dumps({k: round(v["ms"], 3) for k, v in prof.items()}))
