#!/usr/bin/env python
"""bench.py -- compress & progressive-retrieve throughput of the B200 IPComp hot path.

One step = compress_field of the BASELINE.json workload (config 2: 512^3 float32 GRF,
cubic, relative eb 1e-4) followed by its progressive retrieval chain: reconstruct at
relative eb 1e-1, then refine to 1e-2, 1e-3, 1e-4 (pipeline.hpp:140,260,294).
`value` = uncompressed GB/s of that cycle with the field and the archive resident in HBM
(timed by CUDA events on the launching stream, max over ranks); `e2e` = the same cycle
through the C-ABI with HOST buffers (pinned field in, archive out to host, retrieval from
the host archive with host outputs; host-async mode, so each retrieval's copy-out overlaps
the calls after it), host<->device copies inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Multi-GPU (torchrun): independent replicas, one field per rank ("replicas only", weak scaling).
`--impl reference` times the reference's own CPU code (oracle/_ref, compiled from the
reference sources) on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2502_04093_b200 import synth  # noqa: E402

METRIC = "compress & progressive-retrieve GB/s (uncompressed) on 1 B200; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--dims", default=None, help="override dims, e.g. 256x256x256 (parity/debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stage", action="store_true", help="e2e without staging the next step's field (A/B)")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln.split(",") for ln in out.strip().splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for f in getattr(self, "lines", []):
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                for i, nm in enumerate(names):
                    if f[5 + i].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(gpus: int):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if os.environ.get("BENCH_BACKEND", "nccl") == "nccl" else "gloo")
    return ws, rank, local


def max_over_ranks(x: float, ws: int, device=None) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def refine_plan(reader, session, target):
    """plan_for_error's plan for `target`, never dropping a plane the session holds (planner plans
    for decreasing targets are usually but not necessarily nested; refine_field requires it)"""
    import paper_2502_04093_b200 as ipc

    k = ipc.plan_for_error(reader, target).k
    return ipc.RetrievalPlan([max(a, b) for a, b in zip(k, session.planes_loaded())])


def retrieval_targets(cfg: int):
    return synth.CONFIGS[cfg]["retrieve"].get("rel", [1e-2])


# ------------------------------------------------------------------ our arm
def run_ours(args, ws, rank, local):
    import torch

    import paper_2502_04093_b200 as ipc

    torch.cuda.set_device(local)
    c = synth.CONFIGS[args.config]
    dims = tuple(int(x) for x in args.dims.split("x")) if args.dims else c["dims"]
    f = synth.make_field(args.config, seed=0, dims=dims, device=f"cuda:{local}")
    eb = synth.abs_eb(f, c["rel_eb"])
    n, w = f.size, f.itemsize
    nbytes = n * w
    ctx = ipc.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    ft = torch.from_numpy(f).to(f"cuda:{local}")
    rels = retrieval_targets(args.config)

    def step_device():
        reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)
        rng = reader.header().range
        out = ipc.reconstruct_field(reader, ipc.plan_for_error(reader, rels[0] * rng), device=True)
        for rel in rels[1:]:
            out = ipc.refine_field(reader, out.session, out.values, refine_plan(reader, out.session, rel * rng))
        return reader, out

    # correctness guard on the benchmarked workload itself: full-fidelity bound holds
    reader, out = step_device()
    err = float((out.values.double() - ft.double()).abs().max())
    assert err <= eb, f"error bound violated: {err} > {eb}"
    archive_bytes = reader.size()
    del reader, out
    for _ in range(max(0, args.warmup - 1)):
        step_device()
    torch.cuda.synchronize()
    barrier(ws)
    launches0 = ctx.kernel_launches()
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    launches = ctx.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms, ws, f"cuda:{local}")
    value = ws * nbytes * args.steps / (ms_max / 1e3) / 1e9

    # component timings (device-resident) for the report
    comp = {}
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)
    t1.record(stream)
    torch.cuda.synchronize()
    comp["compress_gbs"] = nbytes / (t0.elapsed_time(t1) / 1e3) / 1e9
    rng = reader.header().range
    fresh = {}
    for rel in rels:
        plan = ipc.plan_for_error(reader, rel * rng)
        # warm once: a fresh retrieval of a deeper plan than any refine decoded grows the
        # context's scratch pool on its first call
        ipc.reconstruct_field(reader, plan, device=True, keep_session=False)
        t0.record(stream)
        out = ipc.reconstruct_field(reader, plan, device=True, keep_session=False)
        t1.record(stream)
        torch.cuda.synchronize()
        fresh[str(rel)] = round(nbytes / (t0.elapsed_time(t1) / 1e3) / 1e9, 3)
    comp["retrieve_gbs"] = fresh
    comp["archive_bytes"] = archive_bytes
    comp["compression_ratio"] = round(nbytes / archive_bytes, 3)

    # SURVEY.md §8(d) canonical algorithmic bytes (each stage's distinct HBM inputs and outputs
    # once per element): compress (4w + 20) n + P, retrieval of plan k  P_k + 2 R_k + (8 + 2w) n
    # with R_k = sum_l k_l ceil(count_l / 8) the decoded plane bytes
    peak, peak_src = measured_peak()
    P = reader.header().payload_bytes
    counts = [int(reader.record(l).count) for l in range(1, reader.levels + 1)]
    pipeline = {"compress": {"ms": round(nbytes / comp["compress_gbs"] / 1e6, 3),
                             "algorithmic_bytes": (4 * w + 20) * n + P}}
    for rel in rels:
        plan = ipc.plan_for_error(reader, rel * rng)
        Rk = sum(k * ((cnt + 7) // 8) for k, cnt in zip(plan.k, counts))
        pipeline[f"retrieve rel {rel}"] = {"ms": round(nbytes / fresh[str(rel)] / 1e6, 3),
                                           "algorithmic_bytes": ipc.plan_payload_bytes(reader, plan) + 2 * Rk
                                           + (8 + 2 * w) * n}
    for v in pipeline.values():
        v["achieved"] = round(v["algorithmic_bytes"] / (v["ms"] / 1e3) / 1e9, 2)
        v["frac"] = round(v["achieved"] / peak, 5)

    # roofline of the dominant kernel family, from CUDA events around each family.  This extra
    # step runs with the profiler on, which keeps compress on one stream (in the timed steps
    # each level's lossless stage overlaps the others), so family spans are not inflated.
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step_device()
    p1.record(stream)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    step_ms = p0.elapsed_time(p1)
    top = max(prof.items(), key=lambda kv: kv[1]["ms"])
    # families record §8(d)-canonical bytes: a deflate.* family the 32 x ceil(count/8) plane
    # bytes it consumes, the loss table the 4-byte codes it reads, and so on
    achieved = top[1]["bytes"] / (top[1]["ms"] / 1e3) / 1e9 if top[1]["ms"] > 0 else 0.0

    def gbs(fam):
        v = prof.get(fam)
        return v["bytes"] / (v["ms"] / 1e3) / 1e9 if v and v["ms"] > 0 else None

    # the data-parallel passes the north star holds to the HBM roofline (algorithmic bytes:
    # quant 2w+4+w, recon 4+2w, bitplanes 8, merge 4 + k/8 (+4 refine) per point; crc = payload)
    hbm = {}
    for fam in ("quant_pass", "recon_pass", "bitplanes", "merge", "crc_check", "deflate.crc", "range"):
        g = gbs(fam)
        if g is not None:
            hbm[fam] = {"ms": round(prof[fam]["ms"], 3), "achieved": round(g, 1), "frac": round(g / peak, 4)}
    # measured DRAM traffic of the dominant family (ncu, one compress = one step's launches)
    traffic, traffic_src = None, None
    for tp in (os.path.join(ROOT, "profiles", "r02_traffic.json"), os.path.join(ROOT, "profiles", "r01_traffic.json")):
        tj = json.load(open(tp)).get(top[0]) if os.path.exists(tp) else None
        if tj:
            traffic, traffic_src = int(tj["dram_bytes"]), tj["source"]
            break
    roofline = {"bound": "hbm", "kernel": top[0], "achieved": round(achieved, 2), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 5), "traffic": traffic,
                "traffic_basis": "bytes per step for the family (same basis as achieved)", "traffic_source": traffic_src,
                "algorithmic_bytes": int(top[1]["bytes"]),
                "traffic_over_algorithmic": round(traffic / top[1]["bytes"], 3) if traffic and top[1]["bytes"] else None,
                "pipeline": pipeline,
                "pipeline_basis": "SURVEY.md 8(d): compress (4w+20)n + P; retrieve P_k + 2R_k + (8+2w)n; "
                                  "device-resident single calls, CUDA events",
                "share_of_step": round(top[1]["ms"] / step_ms, 4) if step_ms else None,
                "peak_source": peak_src,
                "family_timing": "CUDA events per family in one profiled step run serially "
                                 f"({step_ms:.1f} ms); 'inflate' encloses the inflate.* sub-families",
                "hbm_kernels": hbm,
                "families_ms": {k: round(v["ms"], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}

    # e2e through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        host_f = torch.from_numpy(f).pin_memory()
        host_arch = torch.empty(archive_bytes + (1 << 20), dtype=torch.uint8).pin_memory()
        host_out = torch.empty(n, dtype=ft.dtype).pin_memory()
        h2d = d2h = 0

        def step_host(stage_next=False):
            nonlocal h2d, d2h
            r = ipc.compress_field(host_f, dims, eb, c["interp"], ctx=ctx)
            if stage_next:
                # the next step's field starts uploading now (ipcg_stage_field), under this step's
                # retrievals; every step's host->device copy stays inside the timed region (the
                # first timed step uploads inside its compress, the last one stages nothing)
                ctx.stage_field(host_f)
            size = r.size()
            r.write_to(host_arch[:size])
            del r
            rh = ipc.ArchiveReader(host_arch[:size], ctx=ctx)
            rng_ = rh.header().range
            o = ipc.reconstruct_field(rh, ipc.plan_for_error(rh, rels[0] * rng_), out=host_out)
            for rel in rels[1:]:
                o = ipc.refine_field(rh, o.session, host_out, refine_plan(rh, o.session, rel * rng_), out=host_out)
            h2d = nbytes + rh.payload_bytes_read()
            d2h = size + nbytes * len(rels)
            return o

        # host-async mode: each retrieval's copy-out into host_out runs on the context's copy
        # stream under the following calls; ctx.synchronize() lands every copy before the
        # closing event, so all host<->device traffic stays inside the timed region
        ctx.set_host_async(True)
        step_host()
        ctx.synchronize()
        torch.cuda.synchronize()
        barrier(ws)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for i in range(args.steps):
            step_host(stage_next=i + 1 < args.steps and not args.no_stage)
        ctx.synchronize()
        g1.record(stream)
        torch.cuda.synchronize()
        ctx.set_host_async(False)
        herr = float(np.max(np.abs(host_out.numpy().astype(np.float64) - f.reshape(-1))))
        assert herr <= eb, f"e2e result violates the error bound: {herr} > {eb}"
        ems = max_over_ranks(g0.elapsed_time(g1), ws, f"cuda:{local}") / args.steps
        e2e = {"value": round(ws * nbytes / (ems / 1e3) / 1e9, 4), "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, f, dims, c)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if w == 4 else "f64",
            "data": "synthetic: seeded Gaussian random field P(k)~k^-11/3 by FFT synthesis, normalised to [0,1] "
                    "(stands in for the paper's SDRBench fields)",
            "config": workload_config(args.config, dims, f, eb, ws),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "gpu_launches": int(launches),
            "clocks": clk.summary(), "detail": comp,
        }
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------ CPU reference
def _sample(f, dims, frac_dims=(256, 256, 256)):
    d = tuple(min(a, b) for a, b in zip(dims, frac_dims)) if len(dims) == 3 else dims
    v = f.reshape(dims)[tuple(slice(0, x) for x in d)]
    return np.ascontiguousarray(v).reshape(-1), d


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_cycle(ref, v, d, c, eb, rels, rng=None):
    """compress + progressive retrieve chain with the reference's own CPU code; retrieval targets
    are rel x rng (the workload field's range when v is a sample of it, else v's archive range)."""
    t0 = time.perf_counter()
    arch = ref.compress(v, d, eb, c["interp"])
    if rng is None:
        import oracle

        rng = oracle.load("oracle").info(arch).range
    k = ref.plan_for_error(arch, rels[0] * rng)
    vals, merged, _ = ref.reconstruct(arch, k, v.dtype, v.size)
    for rel in rels[1:]:
        k2 = [max(a, b) for a, b in zip(ref.plan_for_error(arch, rel * rng), k)]  # as bench's refine_plan
        vals, merged, _ = ref.refine(arch, k, merged, vals, k2)
        k = k2
    return time.perf_counter() - t0, len(arch)


def _load_ref():
    import oracle

    try:
        return oracle.load("ref"), "reference"
    except Exception:
        return oracle.load("oracle"), "port"


def cpu_baseline(cfg, f, dims, c):
    """the reference's CPU compress + retrieve chain on this box's cores --
    the FULL field with IPCOMP_THREADS unset (min(nproc, 16) workers, parallel.hpp:15-22), and a
    sub-volume with IPCOMP_THREADS=1."""
    ref, kind = _load_ref()
    rels = retrieval_targets(cfg)
    saved = os.environ.pop("IPCOMP_THREADS", None)
    threads = min(os.cpu_count() or 1, 16)
    eb = synth.abs_eb(f, c["rel_eb"])
    v = np.ascontiguousarray(f).reshape(-1)
    t_full, _ = reference_cycle(ref, v, dims, c, eb, rels)
    vs, ds = _sample(f, dims, (128, 128, 128))
    os.environ["IPCOMP_THREADS"] = "1"
    t_one, _ = reference_cycle(ref, vs, ds, c, synth.abs_eb(vs, c["rel_eb"]), rels)
    os.environ.pop("IPCOMP_THREADS")
    if saved is not None:
        os.environ["IPCOMP_THREADS"] = saved
    return {"value": round(v.nbytes / t_full / 1e9, 5), "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"the full {'x'.join(map(str, dims))} field ({v.nbytes >> 20} MiB): compress + progressive "
                      f"retrieve chain, IPCOMP_THREADS unset ({threads} workers), one run, {t_full:.1f} s",
            "single_thread": {"value": round(vs.nbytes / t_one / 1e9, 6), "unit": "GB/s", "cores": 1,
                              "sample": f"{'x'.join(map(str, ds))} sub-volume ({vs.nbytes >> 20} MiB), "
                                        f"IPCOMP_THREADS=1, one run, {t_one:.1f} s"},
            "cpu_model": cpu_model(), "nproc": os.cpu_count()}


def run_reference(args, ws, rank):
    """The reference arm: the reference's own CPU code (oracle/_ref) on this box's host cores,
    every step a bounded sample (a 256^3 sub-volume) of our arm's workload."""
    if rank != 0:
        return
    c = synth.CONFIGS[args.config]
    dims = tuple(int(x) for x in args.dims.split("x")) if args.dims else c["dims"]
    ref, kind = _load_ref()
    threads = min(os.cpu_count() or 1, 16)
    os.environ.pop("IPCOMP_THREADS", None)  # the reference's default worker count
    f = synth.make_field(args.config, seed=0, dims=dims, device="cpu")
    v, d = _sample(f, dims)
    eb = synth.abs_eb(f, c["rel_eb"])  # the workload's eb (range of the whole field)
    rels = retrieval_targets(args.config)
    rng = float(f.max()) - float(f.min())
    for _ in range(args.warmup):
        reference_cycle(ref, v, d, c, eb, rels, rng)
    times = []
    for _ in range(args.steps):
        t, _ = reference_cycle(ref, v, d, c, eb, rels, rng)
        times.append(t)
    total = sum(times)
    value = v.nbytes * args.steps / total / 1e9
    sample = (f"each step: compress + progressive retrieve chain of a {'x'.join(map(str, d))} sub-volume "
              f"({v.nbytes >> 20} MiB) of the cfg{args.config} field, same eb and targets")
    line = {"metric": METRIC, "value": round(value, 5), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if f.itemsize == 4 else "f64",
            "data": "synthetic", "impl": "reference", "config": workload_config(args.config, dims, f, eb, ws),
            "sampled": True,
            "cpu_baseline": {"value": round(value, 5), "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": round(value, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(cfg, dims, f, eb, ws):
    c = synth.CONFIGS[cfg]
    rels = retrieval_targets(cfg)
    nbytes = f.size * f.itemsize
    return {"workload": f"cfg{cfg}: {'x'.join(map(str, dims))} {np.dtype(f.dtype).name} "
                        f"{'cubic' if c['interp'] else 'linear'} rel eb {c['rel_eb']}; step = compress + "
                        f"progressive retrieve rel {rels[0]} then refine {rels[1:]}",
            "dims": list(dims), "rel_eb": c["rel_eb"], "abs_eb": eb,
            "l2": f"inputs {nbytes >> 20} MiB > 126 MB L2 (no flush needed)",
            "parallelism": f"replicas x{ws}"}


def main():
    args = parse()
    ws, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
