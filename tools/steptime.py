"""Dev tool: host wall time of each API call in bench.py's device step (compress + 4 retrievals)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth
c = synth.CONFIGS[2]
f = synth.make_field(2, seed=0, dims=c["dims"], device="cuda:0")
eb = synth.abs_eb(f, c["rel_eb"])
ctx = ipc.Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
ft = torch.from_numpy(f).cuda()
rels = c["retrieve"]["rel"]
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    r = ipc.compress_field(ft, c["dims"], eb, c["interp"], ctx=ctx); t.append(time.perf_counter())
    rng = r.header().range
    o = ipc.reconstruct_field(r, ipc.plan_for_error(r, rels[0] * rng), device=True); t.append(time.perf_counter())
    for rel in rels[1:]:
        o = ipc.refine_field(r, o.session, o.values, ipc.plan_for_error(r, rel * rng)); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print(" ".join(f"{1e3*(b-a):7.2f}" for a, b in zip(t, t[1:])), f"total {1e3*(t[-1]-t[0]):.1f} ms", flush=True)
