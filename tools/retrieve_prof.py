"""dev tool: per-family CUDA-event times of ONE compress and of each retrieval of the bench chain
(fresh rel 1e-1, refines), on the cfg2 field.   python tools/retrieve_prof.py [cfg]"""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = synth.CONFIGS[cfg]
f = synth.make_field(cfg, seed=0)
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
ft = torch.from_numpy(f).cuda()
rels = c["retrieve"].get("rel", [1e-2])
for it in range(2):
    ctx.profile(it == 1)
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx)
    if it:
        print("compress", json.dumps({k: round(v["ms"], 3) for k, v in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1]["ms"])}))
    rng = r.header().range
    o = ipc.reconstruct_field(r, ipc.plan_for_error(r, rels[0] * rng), device=True)
    if it:
        print("fresh", rels[0], json.dumps({k: round(v["ms"], 3) for k, v in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1]["ms"])}))
    for rel in rels[1:]:
        o = ipc.refine_field(r, o.session, o.values, ipc.plan_for_error(r, rel * rng))
        if it:
            print("refine", rel, json.dumps({k: round(v["ms"], 3) for k, v in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1]["ms"])}))
    full = ipc.reconstruct_field(r, ipc.full_plan(r), device=True, keep_session=False)
    if it:
        print("fresh full", json.dumps({k: round(v["ms"], 3) for k, v in sorted(ctx.profile_read().items(), key=lambda kv: -kv[1]["ms"])}))
torch.cuda.synchronize()
