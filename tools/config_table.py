"""Per-config throughput on one B200 for all five BASELINE configs (full sizes, device-resident,
CUDA events, median of 3 after a warm-up); writes one JSON object per config.  Dev tool for
the DESIGN.md table (profiles/r01_configs.jsonl)."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2502_04093_b200 as ipc  # noqa: E402
from paper_2502_04093_b200 import synth  # noqa: E402


def timed(fn, reps=3):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


ctx = ipc.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg in (int(x) for x in (sys.argv[1:] or "1 2 3 4 5".split())):
    c = synth.CONFIGS[cfg]
    dims = c["dims"]
    f = synth.make_field(cfg)
    eb = synth.abs_eb(f, c["rel_eb"])
    ft = torch.from_numpy(f).cuda()
    nbytes = f.nbytes
    ms_c = timed(lambda: ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx))
    reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)
    rng = reader.header().range
    plans = [(f"rel {r}", ipc.plan_for_error(reader, r * rng)) for r in c["retrieve"].get("rel", [])]
    for b in c["retrieve"].get("bitrate", []):
        plans.append((f"{b} bit/value", ipc.plan_for_size(reader, int(b * f.size / 8))))
    ret = {}
    for name, plan in plans:
        ms = timed(lambda: ipc.reconstruct_field(reader, plan, device=True, keep_session=False))
        ret[name] = {"ms": round(ms, 3), "GBps": round(nbytes / ms / 1e6, 2), "loaded": ipc.plan_payload_bytes(reader, plan)}

    def chain():
        out = ipc.reconstruct_field(reader, plans[0][1], device=True)
        for _, p in plans[1:]:
            out = ipc.refine_field(reader, out.session, out.values, p)

    ms_chain = timed(chain)
    print(json.dumps({"cfg": cfg, "dims": list(dims), "dtype": str(f.dtype), "MiB": nbytes >> 20,
                      "archive_bytes": reader.size(), "ratio": round(nbytes / reader.size(), 2),
                      "compress_ms": round(ms_c, 3), "compress_GBps": round(nbytes / ms_c / 1e6, 2),
                      "retrieve_fresh": ret, "progressive_chain_ms": round(ms_chain, 3),
                      "cycle_GBps": round(nbytes / (ms_c + ms_chain) / 1e6, 2)}), flush=True)
