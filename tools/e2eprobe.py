"""Wall-clock breakdown of bench.py's e2e step (host field in, archive to host, host-archive
retrieval into a pinned host output) per public call; dev tool."""
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
n = f.size
host_out = torch.empty(n, dtype=torch.float32).pin_memory()
host_arch = None


ASYNC = len(sys.argv) > 1 and sys.argv[1] == "async"
if ASYNC:
    ctx.set_host_async(True)


def step(report):
    global host_arch
    T = [time.time()]
    names = []
    def mark(s):
        if not ASYNC:
            torch.cuda.synchronize()
        T.append(time.time()); names.append(s)
    r = ipc.compress_field(host_f, dims, eb, c["interp"], ctx=ctx); mark("compress(host)")
    size = r.size()
    if host_arch is None:
        host_arch = torch.empty(size + (1 << 20), dtype=torch.uint8).pin_memory()
    r.write_to(host_arch[:size]); mark("write_to")
    del r
    rh = ipc.ArchiveReader(host_arch[:size], ctx=ctx); mark("reader")
    rng_ = rh.header().range
    o = ipc.reconstruct_field(rh, ipc.plan_for_error(rh, rels[0] * rng_), out=host_out); mark(f"reconstruct {rels[0]}")
    for rel in rels[1:]:
        o = ipc.refine_field(rh, o.session, host_out, ipc.plan_for_error(rh, rel * rng_), out=host_out); mark(f"refine {rel}")
    if ASYNC:
        ctx.synchronize(); mark("synchronize")
    if report:
        tot = T[-1] - T[0]
        print(f"step {tot*1e3:.1f} ms  e2e {f.nbytes/tot/1e9:.3f} GB/s")
        for a, b, s in zip(T, T[1:], names):
            print(f"  {s:18s} {1e3*(b-a):7.2f} ms")


step(False)
step(True)
step(True)
