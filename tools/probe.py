"""Quick per-family timing probe of compress + retrieval on a BASELINE config (dev tool)."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dims = tuple(int(x) for x in sys.argv[2].split('x')) if len(sys.argv) > 2 else synth.CONFIGS[cfg]["dims"]
c = synth.CONFIGS[cfg]
t0 = time.time()
f = synth.make_field(cfg, dims=dims)
print("gen", time.time() - t0, flush=True)
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context.default()
ft = torch.from_numpy(f).cuda()
torch.cuda.synchronize()
reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)  # warm
for it in range(2):
    ctx.profile(True)
    t0 = time.time()
    reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)
    t1 = time.time()
    prof = ctx.profile_read()
    ctx.profile(False)
    print(f"compress wall {t1-t0:.4f}s  {f.nbytes/(t1-t0)/1e9:.3f} GB/s archive {reader.size()} CR {f.nbytes/reader.size():.2f}")
    print(json.dumps({k: round(v["ms"], 3) for k, v in prof.items()}))
rng = float(reader.header().range)
for rel in c["retrieve"].get("rel", [1e-2]):
    plan = ipc.plan_for_error(reader, rel * rng)
    out = ipc.reconstruct_field(reader, plan, device=True)
    ctx.profile(True)
    t0 = time.time()
    out = ipc.reconstruct_field(reader, plan, device=True)
    torch.cuda.synchronize()
    t1 = time.time()
    prof = ctx.profile_read(); ctx.profile(False)
    err = float((out.values.double() - ft.double()).abs().max())
    print(f"retrieve rel {rel}: k={plan.k} wall {t1-t0:.4f}s {f.nbytes/(t1-t0)/1e9:.3f} GB/s loaded {out.stats.payload_bytes_loaded} maxerr/target {err/(rel*rng):.3f}")
    print(json.dumps({k: round(v["ms"], 3) for k, v in prof.items()}))
