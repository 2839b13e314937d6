"""GPU at BASELINE.json's full sizes, all five configs (512^3 f32, 1800x3600, 100x500x500,
256x384x384 f64, 64^3), on the seeded synthetic fields bench.py uses.

Exact: the whole archive is byte-identical to the compiled reference (oracle/_ref, the
unmodified reference's own multi-threaded CPU code); for EVERY retrieval target of every config
(cfg2's four, cfg5's six, cfg3's bitrates incl. the non-fill partial plans) the reconstruction
and the session's merged codewords equal the reference's bit for bit, and every refine step
equals the reference's refine_field from the same session.  Size-independent
properties on top (the reference's acceptance criteria, acceptance.cpp:80-104): a full
retrieval meets the point-wise bound; every planned retrieval's measured error is within
bound_for_plan, which is within the requested target; a refine chain lands bit-identical
to the fresh retrieval at each step; loaded bytes equal plan_payload_bytes.
"""
import numpy as np
import pytest

import oracle
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

pytestmark = pytest.mark.gpu


def _bits(t):
    import torch

    return t.view(torch.int32 if t.dtype == torch.float32 else torch.int64)


@pytest.mark.parametrize("cfg", [1, 3, 4, 5, 2])
def test_full_size_config(cfg, ctx):
    import torch

    c = synth.CONFIGS[cfg]
    dims = c["dims"]
    f = synth.make_field(cfg)
    eb = synth.abs_eb(f, c["rel_eb"])
    ft = torch.from_numpy(f).cuda()
    n = f.size
    reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)
    arch = reader.to_bytes()
    ref = oracle.load("ref") if oracle.ref_available() else None
    if ref is not None:
        assert arch == ref.compress(f, dims, eb, c["interp"]), f"cfg{cfg}: archive differs from the reference"

    full = ipc.reconstruct_field(reader, ipc.full_plan(reader), device=True, keep_session=False)
    assert ipc.compute_metrics(ft, full.values, ctx=ctx).max_error <= eb

    rng = reader.header().range
    rt = c["retrieve"]
    plans = []
    for rel in rt.get("rel", []):
        plans.append(("rel", rel, ipc.plan_for_error(reader, rel * rng)))
    for b in rt.get("bitrate", []):
        plans.append(("bitrate", b, ipc.plan_for_size(reader, int(b * n / 8))))
    prev = None
    for kind, t, plan in plans:
        fresh = ipc.reconstruct_field(reader, plan, device=True)
        assert fresh.stats.payload_bytes_loaded == ipc.plan_payload_bytes(reader, plan)
        err = ipc.compute_metrics(ft, fresh.values, ctx=ctx).max_error
        bound = ipc.bound_for_plan(reader, plan)
        assert err <= bound, (cfg, kind, t, err, bound)
        if kind == "rel":
            assert bound <= t * rng, (cfg, t, bound)
        else:
            assert ipc.plan_payload_bytes(reader, plan) <= int(t * n / 8)
        want = want_merged = None
        if ref is not None:  # every target of every config, against the reference's own code
            want, want_merged, _ = ref.reconstruct(arch, plan.k, f.dtype, n)
            assert fresh.values.cpu().numpy().tobytes() == want.tobytes(), (cfg, kind, t)
            for l in range(1, reader.header().progressive_levels + 1):
                assert np.array_equal(fresh.session.merged(l), want_merged[l - 1]), (cfg, kind, t, l)
        if prev is not None and all(a >= b for a, b in zip(plan.k, prev.session.planes_loaded())):
            refined = ipc.refine_field(reader, prev.session, prev.values, plan)
            assert torch.equal(_bits(refined.values), _bits(fresh.values)), (cfg, kind, t)
            if ref is not None:  # the reference's refine_field from the previous step's session
                pk = prev.session.planes_loaded()
                pm = [prev.session.merged(l) for l in range(1, reader.levels + 1)]
                got_ref, _, _ = ref.refine(arch, pk, pm, prev.values.cpu().numpy(), plan.k)
                assert refined.values.cpu().numpy().tobytes() == got_ref.tobytes(), (cfg, kind, t)
        prev = fresh


def test_cfg3_nonfill_range_variant(ctx):
    """SURVEY.md §8d cfg3 caveat: the 1e20 fill enters the range, so every bitrate returns the
    whole archive.  The caller-side variant with eb = 1e-3 x (range of the non-fill values)
    exercises partial plans at 0.5-4 bits/value."""
    import torch

    c = synth.CONFIGS[3]
    dims = c["dims"]
    f = synth.make_field(3)
    ok = f < 1e19
    eb = 1e-3 * float(f[ok].max() - f[ok].min())
    ft = torch.from_numpy(f).cuda()
    reader = ipc.compress_field(ft, dims, eb, c["interp"], ctx=ctx)
    arch = reader.to_bytes()
    n = f.size
    prev_bytes = -1
    mandatory = ipc.plan_payload_bytes(
        reader, [0 if l + 1 <= reader.header().progressive_levels else 32 for l in range(reader.levels)])
    for b in c["retrieve"]["bitrate"]:
        try:
            plan = ipc.plan_for_size(reader, int(b * n / 8))
        except ipc.InfeasibleRequest:  # planner.cpp: budget below the mandatory bytes
            assert int(b * n / 8) < mandatory
            continue
        got = ipc.reconstruct_field(reader, plan, device=True, keep_session=False)
        if oracle.ref_available():  # partial bitrate plans, bit for bit against the reference
            want, _, _ = oracle.load("ref").reconstruct(arch, plan.k, f.dtype, n)
            assert got.values.cpu().numpy().tobytes() == want.tobytes(), b
        loaded = got.stats.payload_bytes_loaded
        assert loaded == ipc.plan_payload_bytes(reader, plan) >= prev_bytes
        prev_bytes = loaded
        # the loss table replays the dropped digits in double (pipeline.hpp:85-124) while values are
        # rounded to f32 (quantizer.hpp:57-60), so an f32 retrieval may exceed bound_for_plan by a
        # few ulps of the values it rounds (bit-exact with the reference all the same)
        ulp = float(np.spacing(np.float32(np.abs(f[ok]).max())))
        assert ipc.compute_metrics(ft, got.values, ctx=ctx).max_error <= ipc.bound_for_plan(reader, plan) + 4 * ulp
    if oracle.ref_available():
        assert arch == oracle.load("ref").compress(f, dims, eb, c["interp"])
