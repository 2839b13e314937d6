"""dev tool: per-call wall times of bench.py's e2e step in steady state (host-async copy-outs,
no drain between steps, as in the timed loop)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

c = synth.CONFIGS[2]
dims = c["dims"]
f = synth.make_field(2, dims=dims)
eb = synth.abs_eb(f, c["rel_eb"])
rels = [0.1, 0.01, 0.001, 0.0001]
ctx = ipc.Context.default()
host_f = torch.from_numpy(f).pin_memory()
host_out = torch.empty(f.size, dtype=torch.float32).pin_memory()
host_arch = torch.empty(150 << 20, dtype=torch.uint8).pin_memory()
ctx.set_host_async(True)
for it in range(6):
    T = [time.time()]
    r = ipc.compress_field(host_f, dims, eb, c["interp"], ctx=ctx); T.append(time.time())
    if len(sys.argv) > 1 and "stage" in sys.argv[1] and it < 5:
        ctx.stage_field(host_f)
    size = r.size()
    r.write_to(host_arch[:size]); T.append(time.time())
    del r
    rh = ipc.ArchiveReader(host_arch[:size], ctx=ctx)
    rng_ = rh.header().range
    if len(sys.argv) > 1 and "nod2h" in sys.argv[1]:  # experiment: results stay on the device
        o = ipc.reconstruct_field(rh, ipc.plan_for_error(rh, rels[0] * rng_), device=True); T.append(time.time())
        for rel in rels[1:]:
            o = ipc.refine_field(rh, o.session, o.values, ipc.plan_for_error(rh, rel * rng_)); T.append(time.time())
    else:
        o = ipc.reconstruct_field(rh, ipc.plan_for_error(rh, rels[0] * rng_), out=host_out); T.append(time.time())
        for rel in rels[1:]:
            o = ipc.refine_field(rh, o.session, host_out, ipc.plan_for_error(rh, rel * rng_), out=host_out); T.append(time.time())
    if it >= 3:
        d = [1e3 * (b - a) for a, b in zip(T, T[1:])]
        print(f"step {1e3*(T[-1]-T[0]):.1f} ms: compress {d[0]:.1f} write {d[1]:.1f} fresh {d[2]:.1f} refines " +
              " ".join(f"{x:.1f}" for x in d[3:]))
ctx.synchronize()
