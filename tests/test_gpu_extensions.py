"""GPU tests of what sits next to the hot path and of the host-async
output mode, against the CPU oracle (oracle/), bit for bit where the reference is exact."""
import numpy as np
import pytest

import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

pytestmark = pytest.mark.gpu


def _field(dims, seed, dtype):
    return synth.smooth_field(dims, seed).astype(dtype)


def _eb(f, rel):
    r = float(np.max(f)) - float(np.min(f))
    return rel * r if r > 0 else 1e-3


@pytest.mark.parametrize("lp", [0, 2])
def test_host_async_chain_matches_oracle(lp, oracle_lib):
    """Retrievals into pinned host buffers in host-async mode: each call returns before its
    copy-out lands; a refine whose `previous` is a host buffer still being written (lp=2
    keeps non-progressive levels, so `previous` is read) must wait for it."""
    import torch

    ctx = ipc.Context(0)
    ctx.set_host_async(True)
    dims = (40, 36, 30)
    f = _field(dims, 31, np.float32)
    eb = _eb(f, 1e-4)
    arch = oracle_lib.compress(f, dims, eb, 1, lp)
    reader = ipc.ArchiveReader(arch, ctx=ctx)
    L = reader.levels
    plans = [[min(32, 4 + 9 * s) if l + 1 <= reader.header().progressive_levels else 32 for l in range(L)]
             for s in range(4)]
    outs = [torch.empty(f.size, dtype=torch.float32).pin_memory() for _ in plans]
    shared = torch.empty(f.size, dtype=torch.float32).pin_memory()
    r = ipc.reconstruct_field(reader, plans[0], out=outs[0])
    rs = ipc.reconstruct_field(reader, plans[0], out=shared)
    for i in range(1, len(plans)):
        r = ipc.refine_field(reader, r.session, outs[i - 1], plans[i], out=outs[i])
        rs = ipc.refine_field(reader, rs.session, shared, plans[i], out=shared)  # like bench.py's e2e
    ctx.synchronize()
    k_prev, m_prev, want_prev = None, None, None
    for i, k in enumerate(plans):
        if i == 0:
            want, m, _ = oracle_lib.reconstruct(arch, k, np.float32, f.size)
        else:
            want, m, _ = oracle_lib.refine(arch, k_prev, m_prev, want_prev, k)
        assert outs[i].numpy().tobytes() == want.tobytes(), i
        k_prev, m_prev, want_prev = k, m, want
    assert shared.numpy().tobytes() == want_prev.tobytes()
    ctx.set_host_async(False)
    sync = ipc.reconstruct_field(reader, plans[-1])
    assert sync.values.tobytes() == want_prev.tobytes()


@pytest.mark.parametrize("dtype,dims", [(np.float32, (40, 36, 30)), (np.float64, (70, 130))])
def test_staged_field_compresses_like_a_direct_upload(dtype, dims, oracle_lib):
    """ipcg_stage_field: a host field uploaded ahead of its compress gives the oracle's archive
    bytes; a compress of another buffer ignores (and drops) the staged copy; a staged field is
    used once."""
    import torch

    ctx = ipc.Context(0)
    f = torch.from_numpy(_field(dims, 7, dtype).reshape(-1)).pin_memory()
    g = torch.from_numpy(_field(dims, 8, dtype).reshape(-1)).pin_memory()
    eb = _eb(f.numpy(), 1e-4)
    want_f = oracle_lib.compress(f.numpy(), dims, eb, 1)
    want_g = oracle_lib.compress(g.numpy(), dims, eb, 1)
    for _ in range(2):  # (the second round re-stages over a consumed copy)
        ctx.stage_field(f)
        assert ipc.compress_field(f, dims, eb, ipc.CUBIC, ctx=ctx).to_bytes() == want_f
    assert ipc.compress_field(f, dims, eb, ipc.CUBIC, ctx=ctx).to_bytes() == want_f  # nothing staged
    ctx.stage_field(f)
    assert ipc.compress_field(g, dims, eb, ipc.CUBIC, ctx=ctx).to_bytes() == want_g  # another buffer
    assert ipc.compress_field(f, dims, eb, ipc.CUBIC, ctx=ctx).to_bytes() == want_f  # the copy was dropped
    ctx.stage_field(f)
    ctx.stage_field(g)  # replaces the pending one
    assert ipc.compress_field(g, dims, eb, ipc.CUBIC, ctx=ctx).to_bytes() == want_g
    with pytest.raises(ValueError):
        ctx.stage_field(f.cuda())


# ---- session file: write_session / read_session, session.cpp:8-61
import hashlib  # noqa: E402
import json  # noqa: E402
import os  # noqa: E402

import oracle  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


@pytest.mark.parametrize("case", MANIFEST, ids=[c["name"] for c in MANIFEST])
def test_session_file_matches_reference_golden(case, oracle_lib, ctx):
    arch = open(os.path.join(GOLDEN, case["name"] + ".ipc"), "rb").read()
    want = open(os.path.join(GOLDEN, case["name"] + ".ips"), "rb").read()
    k = case["session"]["k"]
    f = np.load(os.path.join(GOLDEN, case["name"] + ".input.npy"))
    reader = ipc.ArchiveReader(arch, ctx=ctx)
    got = ipc.reconstruct_field(reader, k)
    assert ipc.write_session(got.session) == want  # deflated on the GPU, byte-identical
    back = ipc.read_session(want, reader)
    assert back.planes_loaded() == k
    _, m, _ = oracle_lib.reconstruct(arch, k, f.dtype, f.size)
    for level in range(1, reader.levels + 1):
        mg = back.merged(level)
        assert (mg is None and m[level - 1] is None) or np.array_equal(mg, m[level - 1])
    # a refine from the session read back equals the oracle's refine
    rf = case["refine"]
    if rf["k1"] == k:
        v2 = ipc.refine_field(reader, back, got.values, rf["k2"])
        assert hashlib.sha256(v2.values.tobytes()).hexdigest() == rf["sha256"]


def test_session_file_large_device_resident(oracle_lib, ctx):
    """cfg2 generator at 96^3: level-1 codeword arrays of ~0.4 MB per level through the GPU
    deflate; device-resident destination and source."""
    import torch

    dims = (96, 96, 96)
    c = synth.CONFIGS[2]
    f = synth.make_field(2, dims=dims)
    eb = synth.abs_eb(f, c["rel_eb"])
    reader = ipc.compress_field(f, dims, eb, c["interp"], ctx=ctx)
    arch = reader.to_bytes()
    for rel in (1e-1, 1e-3):
        k = ipc.plan_for_error(reader, rel * reader.header().range).k
        got = ipc.reconstruct_field(reader, k)
        _, m, _ = oracle_lib.reconstruct(arch, k, np.float32, f.size)
        want = oracle_lib.write_session(arch, k, m)
        dst = torch.empty(ipc.library().ipcg_session_write_bound(got.session.h), dtype=torch.uint8, device="cuda")
        size = ipc.write_session(got.session, dst)
        assert size == len(want)
        assert dst[:size].cpu().numpy().tobytes() == want
        back = ipc.read_session(dst[:size], reader)  # device-resident file
        assert back.planes_loaded() == k
        for level in range(1, reader.levels + 1):
            assert np.array_equal(back.merged(level), m[level - 1])


@pytest.mark.parametrize("lp", [0, 2])
def test_session_reader_errors_match_oracle(lp, oracle_lib, ctx):
    from test_oracle import _session_corruptions

    dims = (20, 24, 18)
    f = synth.smooth_field(dims, 3).astype(np.float32)
    arch = oracle_lib.compress(f, dims, 1e-3 * float(f.max() - f.min()), 1, lp)
    L = oracle.archive_levels(arch)
    k = [5 + 3 * i if i < (lp or L) else 32 for i in range(L)]
    _, m, _ = oracle_lib.reconstruct(arch, k, np.float32, f.size)
    good = oracle_lib.write_session(arch, k, m)
    reader = ipc.ArchiveReader(arch, ctx=ctx)
    other = ipc.ArchiveReader(oracle_lib.compress(f, dims, 2e-3 * float(f.max() - f.min()), 1, lp), ctx=ctx)
    with pytest.raises(RuntimeError, match="session does not belong to this archive"):
        ipc.read_session(good, other)
    for bad in _session_corruptions(good):
        try:
            oracle_lib.read_session(arch, bad)
            want = "ok"
        except oracle.OracleError as e:
            want = str(e)
        try:
            ipc.read_session(bad, reader)
            got = "ok"
        except RuntimeError as e:
            got = str(e)
        assert got == want, len(bad)


# ---- compute_metrics, pipeline.hpp:354-372
def test_metrics_known_answers(ctx):  # test_pipeline.cpp:355-390
    a = np.array([1.0, 2.0, 3.0])
    m = ipc.compute_metrics(a, a, ctx=ctx)
    assert m.max_error == 0.0 and m.mse == 0.0 and np.isinf(m.psnr)
    a = np.array([0.0, 10.0, 5.0, 2.5])
    b = a.copy()
    b[2] += 0.125
    m = ipc.compute_metrics(a, b, ctx=ctx)
    assert m.max_error == 0.125
    assert m.mse == pytest.approx(0.125 * 0.125 / 4.0, rel=1e-12)
    assert m.psnr == pytest.approx(20.0 * np.log10(10.0 / np.sqrt(0.125 * 0.125 / 4.0)), rel=1e-12)
    with pytest.raises(ValueError, match="metrics inputs differ in size"):
        ipc.compute_metrics(a, a[:3], ctx=ctx)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [0, 1, 5, 1000, 4099, 3_000_001])
def test_metrics_match_oracle(dtype, n, oracle_lib, ctx):
    """max_error bit-exact; mse/psnr to the summation-order tolerance (the reference's own
    test allows 1e-12 at n=1000; the bound grows like n*eps, 1e-10 covers 3e6)."""
    import torch

    rng = np.random.default_rng(n)
    a = rng.uniform(-3, 3, n).astype(dtype)
    b = (a + 0.01 * rng.uniform(-3, 3, n)).astype(dtype)
    want = oracle_lib.compute_metrics(a, b)
    tol = 1e-12 if n <= 5000 else 1e-10
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for x, y in ((a, b), (ta, tb), (a[1:], b[1:]), (ta[1:], tb[1:])):  # device slices are misaligned
        got = ipc.compute_metrics(x, y, ctx=ctx)
        w = want if x.shape[0] == n else oracle_lib.compute_metrics(a[1:], b[1:])
        assert got.max_error == w[0]
        assert got.mse == pytest.approx(w[1], rel=tol, abs=0)
        assert got.psnr == pytest.approx(w[2], rel=tol) or (np.isinf(got.psnr) and np.isinf(w[2]))


def test_metrics_nonfinite_like_reference(oracle_lib, ctx):
    a = np.linspace(-1, 1, 777)
    b = a + 1e-3
    b[10], a[20], b[30] = np.nan, np.inf, -np.inf
    got = ipc.compute_metrics(a, b, ctx=ctx)
    want = oracle_lib.compute_metrics(a, b)
    assert got.max_error == want[0]
    assert np.isnan(got.mse) == np.isnan(want[1]) and np.isnan(got.psnr) == np.isnan(want[2])
