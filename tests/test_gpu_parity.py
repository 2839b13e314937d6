"""GPU parity: the sm_100a path against the CPU oracle (oracle/), bit for bit.

Compares, on the same seeded inputs: whole archive bytes (codes, outliers, loss
tables, every bitplane block incl. the zlib-1.3 deflate streams and CRCs), the
reconstructed values for random plans, refine chains, planner outputs and error
behaviour.  Mirrors the reference's own tests (proj/tests/test_pipeline.cpp).
"""
import numpy as np
import pytest

import oracle
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

pytestmark = pytest.mark.gpu

SHAPES = [(1,), (2,), (3, 1), (1, 1, 1, 5), (9,), (17, 9), (65,), (257,), (33, 21), (17, 18, 19), (5, 6, 7),
          (2, 3, 4, 5), (31, 22), (129,), (513,), (64, 64), (9, 7, 33)]


def _field(dims, seed, dtype):
    f = synth.smooth_field(dims, seed).astype(dtype)
    return f


def _eb(f, rel):
    r = float(np.max(f)) - float(np.min(f))
    return rel * r if r > 0 else 1e-3


@pytest.mark.parametrize("dims", SHAPES)
@pytest.mark.parametrize("interp", [0, 1])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_archive_bytes_match_oracle(dims, interp, dtype, oracle_lib, ctx):
    f = _field(dims, 17 + len(dims), dtype)
    eb = _eb(f, 1e-4)
    want = oracle_lib.compress(f, dims, eb, interp)
    got = ipc.compress_field(f, dims, eb, interp, ctx=ctx).to_bytes()
    assert got == want


@pytest.mark.parametrize("rel", [1e-1, 1e-3, 1e-6])
@pytest.mark.parametrize("lp", [0, 1, 2])
def test_archive_bytes_eb_and_progressive_levels(rel, lp, oracle_lib, ctx):
    dims = (24, 40, 36)
    f = _field(dims, 5, np.float32)
    eb = _eb(f, rel)
    want = oracle_lib.compress(f, dims, eb, 1, lp)
    got = ipc.compress_field(f, dims, eb, 1, lp, ctx=ctx).to_bytes()
    assert got == want


@pytest.mark.parametrize("cfg,dims", [(1, (64, 64, 64)), (2, (64, 64, 64)), (3, (90, 180)), (4, (20, 60, 60)),
                                      (5, (24, 36, 36))])
def test_baseline_config_generators_match(cfg, dims, oracle_lib, ctx):
    c = synth.CONFIGS[cfg]
    f = synth.make_field(cfg, dims=dims)
    eb = synth.abs_eb(f, c["rel_eb"])
    want = oracle_lib.compress(f, dims, eb, c["interp"])
    got = ipc.compress_field(f, dims, eb, c["interp"], ctx=ctx).to_bytes()
    assert got == want


def test_outliers_nonfinite_and_spikes(oracle_lib, ctx):
    for dt in (np.float32, np.float64):
        v = np.ones(40, dtype=dt)
        v[7] = np.inf
        v[21] = 1e30 if dt == np.float32 else 1e60
        v[22] = -v[21]
        v[30] = np.nan
        want = oracle_lib.compress(v, (40,), 1e-6, 1)
        got = ipc.compress_field(v, (40,), 1e-6, 1, ctx=ctx).to_bytes()
        assert got == want


def _random_plan(rng, L, lp):
    return [32 if l + 1 > lp else int(rng.integers(0, 33)) for l in range(L)]


def _widen(rng, k, lp):
    return [x + (int(rng.integers(0, 33 - x)) if i + 1 <= lp else 0) for i, x in enumerate(k)]


@pytest.mark.parametrize("dims,interp,dtype", [((65, 33), 0, np.float64), ((17, 13, 11), 1, np.float64),
                                               ((64, 64, 64), 1, np.float32), ((33,), 1, np.float32),
                                               ((2, 3, 4, 5), 0, np.float32),
                                               # whole-row level-1 kernels (last extent a multiple of
                                               # the 16-byte vector): f64 pairs, f32 quads, rows longer
                                               # than one 1024-element chunk, 1-D and 2-D boxes
                                               ((24, 40, 36), 1, np.float64), ((24, 40, 36), 0, np.float64),
                                               ((6, 10, 2056), 1, np.float32), ((48, 64), 0, np.float32),
                                               ((4100,), 1, np.float32), ((7, 9, 4), 1, np.float32)])
def test_reconstruct_and_refine_match_oracle(dims, interp, dtype, oracle_lib, ctx):
    f = _field(dims, 606, dtype)
    eb = _eb(f, 1e-4)
    arch = oracle_lib.compress(f, dims, eb, interp)
    reader = ipc.ArchiveReader(arch, ctx=ctx)
    info = oracle_lib.info(arch)
    L, lp = info.levels, info.progressive_levels
    rng = np.random.default_rng(7)
    n = f.size
    for trial in range(4):
        k1 = _random_plan(rng, L, lp)
        k2 = _widen(rng, k1, lp)
        want1, m1, loaded1 = oracle_lib.reconstruct(arch, k1, dtype, n)
        got1 = ipc.reconstruct_field(reader, k1)
        assert got1.values.tobytes() == want1.tobytes()
        assert got1.stats.payload_bytes_loaded == loaded1
        for l in range(L):
            if m1[l] is not None:
                assert np.array_equal(got1.session.merged(l + 1), m1[l])
        want2, _, loaded2 = oracle_lib.refine(arch, k1, m1, want1, k2)
        got2 = ipc.refine_field(reader, got1.session, got1.values, k2)
        assert got2.values.tobytes() == want2.tobytes()
        assert got2.stats.payload_bytes_loaded == loaded2
        direct2, _, _ = oracle_lib.reconstruct(arch, k2, dtype, n)
        assert got2.values.tobytes() == direct2.tobytes()


def test_gpu_archive_round_trip_device_resident(oracle_lib, ctx):
    import torch

    dims = (48, 40, 32)
    f = _field(dims, 3, np.float32)
    eb = _eb(f, 1e-3)
    ft = torch.from_numpy(f).cuda()
    reader = ipc.compress_field(ft, dims, eb, 1, ctx=ctx)  # device in, device archive
    arch = reader.to_bytes()
    assert arch == oracle_lib.compress(f, dims, eb, 1)
    k = ipc.full_plan(reader).k
    out = ipc.reconstruct_field(reader, k, device=True)
    want, _, _ = oracle_lib.reconstruct(arch, k, np.float32, f.size)
    assert out.values.cpu().numpy().tobytes() == want.tobytes()
    assert float(np.max(np.abs(out.values.cpu().numpy().astype(np.float64) - f))) <= eb


def test_planner_matches_oracle(oracle_lib, ctx):
    dims = (33, 29, 17)
    f = _field(dims, 42, np.float64)
    eb = _eb(f, 1e-4)
    arch = oracle_lib.compress(f, dims, eb, 0)
    reader = ipc.ArchiveReader(arch, ctx=ctx)
    for factor in (4.0, 64.0, 1024.0, 65536.0):
        assert ipc.plan_for_error(reader, factor * eb).k == oracle_lib.plan_for_error(arch, factor * eb)
    total = oracle_lib.plan_payload_bytes(arch, [32] * reader.levels)
    for frac in (0.2, 0.5, 0.9, 1.0):
        b = int(total * frac)
        try:
            want = oracle_lib.plan_for_size(arch, b)
        except oracle.InfeasibleRequest:
            with pytest.raises(ipc.InfeasibleRequest):
                ipc.plan_for_size(reader, b)
            continue
        assert ipc.plan_for_size(reader, b).k == want
    with pytest.raises(ipc.InfeasibleRequest):
        ipc.plan_for_error(reader, eb * 0.5)


def _host_plan(m, *, max_error=None, byte_budget=None):
    k = (ipc.C.c_int * ipc.MAX_LEVELS)()
    lib = ipc.library()
    if byte_budget is None:
        rc = lib.ipcg_model_plan_for_error(ipc.C.byref(m), float(max_error), k)
    else:
        rc = lib.ipcg_model_plan_for_size(ipc.C.byref(m), int(byte_budget), k)
    if rc:
        return rc, (lib.ipcg_last_error(None) or b"").decode(), None
    return 0, "", list(k)[:m.levels]


def _device_plan(ctx, m, **kw):
    try:
        return 0, "", ipc.plan_on_device(m, ctx=ctx, **kw).k
    except ipc.InfeasibleRequest as e:
        return 4, str(e), None
    except RuntimeError as e:
        return 2, str(e), None


def test_device_planner_matches_host_and_oracle(oracle_lib, ctx):
    """plan_for_error / plan_for_size as one GPU launch (planner.cu) give the
    host planner's plans (and the oracle's), error kinds and messages."""
    for dims, dtype, interp, lp in [((33, 29, 17), np.float64, 0, 0), ((40, 36, 30), np.float32, 1, 0),
                                    ((70, 130), np.float32, 1, 2), ((9,), np.float32, 0, 0)]:
        f = _field(dims, 42, dtype)
        eb = _eb(f, 1e-4)
        arch = oracle_lib.compress(f, dims, eb, interp, lp)
        reader = ipc.ArchiveReader(arch, ctx=ctx)
        for factor in (1.0, 1.5, 4.0, 64.0, 1024.0, 65536.0, 1e30, float("inf")):
            assert ipc.plan_on_device(reader, max_error=factor * eb).k == oracle_lib.plan_for_error(arch, factor * eb)
        for bad in (eb * 0.5, float("nan")):
            with pytest.raises(ipc.InfeasibleRequest, match="below the archive's compression bound"):
                ipc.plan_on_device(reader, max_error=bad)
        total = oracle_lib.plan_payload_bytes(arch, [32] * reader.levels)
        m = ipc.error_model_c(reader)
        for b in [0, 1, total // 7, total // 3, total // 2, int(total * 0.9), total - 1, total, 2 * total, 2**63]:
            rc, msg, want = _host_plan(m, byte_budget=b)
            drc, dmsg, got = _device_plan(ctx, m, byte_budget=b)
            assert (drc, got) == (rc, want), (dims, b)
            if rc:
                assert dmsg == msg
            else:
                assert got == oracle_lib.plan_for_size(arch, b)


def test_device_planner_random_models(ctx):
    """Hand-built ErrorModels (planner.hpp:13-32): ties between choices, zero-length planes,
    zero deltas, a single level, 16 levels -- device plans equal the host planner's."""
    rng = np.random.default_rng(5)
    for case in range(60):
        m = ipc.ErrorModelC()
        m.levels = int(rng.integers(1, ipc.MAX_LEVELS + 1))
        m.progressive_levels = int(rng.integers(0, m.levels + 1))
        m.eb = float(10.0 ** rng.uniform(-9, 0))
        m.amplification = float(rng.choice([1.0, 1.25]))
        for l in range(m.levels):
            lc = m.level[l]
            steps = rng.choice([0.0, 1.0, 2.0], size=32, p=[0.3, 0.4, 0.3]) * 10.0 ** rng.uniform(-9, 1)
            d = np.concatenate([[0.0], np.cumsum(steps)])  # non-decreasing, with plateaus (ties)
            for i in range(33):
                lc.delta[i] = float(d[i])
            pb = rng.integers(0, 1 << int(rng.integers(1, 28)), size=32) * rng.choice([0, 1], size=32, p=[0.2, 0.8])
            for i in range(32):
                lc.plane_bytes[i] = int(pb[i])
            lc.outlier_bytes = int(rng.integers(0, 1000))
            lc.progressive = 1 if l + 1 <= m.progressive_levels else 0
        total = int(ipc.library().ipcg_model_total_payload_bytes(ipc.C.byref(m)))
        for q in range(6):
            target = m.eb * float(10.0 ** rng.uniform(-0.3, 12))
            assert _device_plan(ctx, m, max_error=target) == _host_plan(m, max_error=target), (case, q)
            b = int(rng.integers(0, max(2, 2 * total)))
            assert _device_plan(ctx, m, byte_budget=b) == _host_plan(m, byte_budget=b), (case, q, b)


def test_backend_encode_matches_zlib(ctx):
    import zlib

    rng = np.random.default_rng(0)
    cases = [bytes(1), bytes(100), bytes(70000), rng.integers(0, 256, 5000, dtype=np.uint8).tobytes(),
             np.packbits((rng.random(8 * 200000) < 0.05).astype(np.uint8), bitorder="little").tobytes(),
             (b"abcabcabd" * 30000)[:250000],
             # stored blocks (random stretches) between compressed ones: every later block's bit
             # position goes through a byte alignment
             rng.integers(0, 256, 40000, dtype=np.uint8).tobytes() + bytes(60000) +
             rng.integers(0, 256, 50000, dtype=np.uint8).tobytes() + b"xyz" * 20000]
    for raw in cases:
        (be, payload, crc), = ipc.backend_encode(np.frombuffer(raw, np.uint8), ctx=ctx)
        z = zlib.compress(raw, 6)
        if len(z) < len(raw):
            assert be == 1 and payload == z
        else:
            assert be == 0 and payload == raw
        assert crc == zlib.crc32(payload)


def test_errors_mirror_reference(oracle_lib, ctx):
    f = _field((33,), 3, np.float64)
    with pytest.raises(ipc.InvalidArgument, match="error bound must be positive and finite"):
        ipc.compress_field(f, (33,), 0.0, ctx=ctx)
    with pytest.raises(ipc.InvalidArgument, match="grid must have between 1 and 4 dimensions"):
        ipc.compress_field(np.zeros(243), (3, 3, 3, 3, 3), 1e-3, ctx=ctx)
    arch = oracle_lib.compress(f, (33,), 1e-3, 1)
    reader = ipc.ArchiveReader(arch, ctx=ctx)
    with pytest.raises(ipc.InvalidArgument, match="scalar kind does not match archive"):
        ipc.reconstruct_field(reader, ipc.full_plan(reader), dtype=np.float32)
    with pytest.raises(ipc.InvalidArgument, match="plan plane count out of range"):
        ipc.reconstruct_field(reader, [33] * reader.levels)
    bad = bytearray(arch)
    bad[0] = ord("X")
    with pytest.raises(RuntimeError, match="not an archive: bad magic"):
        ipc.ArchiveReader(bytes(bad), ctx=ctx)
    # corrupt one payload byte of the finest level's plane 0 -> checksum mismatch
    info = oracle_lib.info(arch)
    off = info.index_bytes + info.plane_offset[0][31] + 21
    bad = bytearray(arch)
    bad[off] ^= 0xFF
    r2 = ipc.ArchiveReader(bytes(bad), ctx=ctx)
    with pytest.raises(RuntimeError, match="block checksum mismatch"):
        ipc.reconstruct_field(r2, ipc.full_plan(r2))
    out = ipc.reconstruct_field(reader, [16] * reader.levels)
    with pytest.raises(ipc.InvalidArgument, match="refinement plan must not drop planes"):
        ipc.refine_field(reader, out.session, out.values, [8] + [16] * (reader.levels - 1))


def test_inflate_against_zlib_streams(ctx):
    """GPU inflate on zlib streams of every level / block mix, stored/fixed/dynamic, and corruptions."""
    import zlib

    rng = np.random.default_rng(11)
    datas = [b"", b"a", bytes(10), bytes(100000), rng.integers(0, 256, 70000, dtype=np.uint8).tobytes(),
             np.packbits((rng.random(8 * 300000) < 0.03).astype(np.uint8), bitorder="little").tobytes(),
             np.packbits((rng.random(8 * 200000) < 0.3).astype(np.uint8), bitorder="little").tobytes(),
             (b"the quick brown fox %d " * 20000)[:300000],
             np.repeat(rng.integers(0, 3, 5000, dtype=np.uint8), rng.integers(1, 300, 5000)).tobytes()]
    blocks, want = [], []
    def deflate(d, level, strategy):
        c = zlib.compressobj(level, zlib.DEFLATED, 15, 8, strategy)
        return c.compress(d) + c.flush()

    for d in datas:
        for level in (1, 6, 9):
            z = zlib.compress(d, level)
            blocks.append((1, z, zlib.crc32(z), len(d)))
            want.append(d)
        # fixed-Huffman-only streams (long static blocks the chain decodes itself),
        # Huffman-only (no matches) and RLE (distance-1 runs)
        for strategy in (zlib.Z_FIXED, zlib.Z_HUFFMAN_ONLY, zlib.Z_RLE):
            z = deflate(d, 6, strategy)
            blocks.append((1, z, zlib.crc32(z), len(d)))
            want.append(d)
        blocks.append((0, d, zlib.crc32(d), len(d)))
        want.append(d)
    got = ipc.backend_decode(blocks, ctx=ctx)
    for g, w in zip(got, want):
        assert g == w
    z = bytearray(zlib.compress(datas[6], 6))
    z[len(z) // 2] ^= 0x55
    bad = [(1, bytes(z), zlib.crc32(bytes(z)), len(datas[6])),          # corrupt stream, valid CRC
           (1, zlib.compress(datas[6], 6), 123, len(datas[6])),          # CRC mismatch
           (1, zlib.compress(datas[6], 6)[:-5], zlib.crc32(zlib.compress(datas[6], 6)[:-5]), len(datas[6])),
           (1, zlib.compress(datas[6], 6), zlib.crc32(zlib.compress(datas[6], 6)), len(datas[6]) - 1),
           (0, b"abc", zlib.crc32(b"abc"), 4)]
    got = ipc.backend_decode(bad, ctx=ctx)
    assert [str(g) for g in got] == ["deflate backend failed to decompress block", "block checksum mismatch",
                                     "deflate backend failed to decompress block",
                                     "deflate backend failed to decompress block", "identity block has wrong length"]


def test_inflate_lane_parallel_decode_edge_streams(ctx):
    """The lane-parallel candidate decode (inflate.cu k_decode_cands) on streams that defeat
    self-synchronisation: long runs coded as a few-bit repeated match (phase-locked paths),
    periodic symbol patterns of several periods, near-fixed-length literal codes, a dynamic block
    of exactly the maximum symbol count, and corruptions deep inside long dynamic blocks."""
    import zlib

    rng = np.random.default_rng(23)
    datas = [bytes(3_000_000),                                         # 258-byte dist-1 matches
             (b"\x01" + bytes(257)) * 6000,                            # run + literal
             bytes([0, 0, 0, 7]) * 200000,                             # 4-periodic
             bytes(rng.integers(0, 2, 300000, dtype=np.uint8)),       # 1-bit literal codes
             bytes(rng.integers(0, 4, 300000, dtype=np.uint8) * 64),  # 2-bit literal codes
             rng.integers(0, 256, 200000, dtype=np.uint8).tobytes(),   # ~8-bit codes
             bytes(rng.permutation(np.repeat(np.arange(256, dtype=np.uint8), 64)))]
    blocks, want = [], []
    for d in datas:
        for level, strategy in ((6, zlib.Z_DEFAULT_STRATEGY), (1, zlib.Z_DEFAULT_STRATEGY),
                                (6, zlib.Z_HUFFMAN_ONLY), (6, zlib.Z_RLE)):
            c = zlib.compressobj(level, zlib.DEFLATED, 15, 8, strategy)
            z = c.compress(d) + c.flush()
            blocks.append((1, z, zlib.crc32(z), len(d)))
            want.append(d)
    got = ipc.backend_decode(blocks, ctx=ctx)
    for g, w in zip(got, want):
        assert g == w
    # corruptions at several depths of a long dynamic stream: the error must surface exactly
    # as zlib reports it (any failure -> the reference's message), never as wrong bytes
    d = datas[5]
    z0 = zlib.compress(d, 6)
    bad = []
    for frac in (0.01, 0.3, 0.62, 0.97):
        z = bytearray(z0)
        z[int(len(z) * frac)] ^= 0x10
        bad.append((1, bytes(z), zlib.crc32(bytes(z)), len(d)))
    got = ipc.backend_decode(bad, ctx=ctx)
    for (be, z, crc, n), g in zip(bad, got):
        try:
            ok = zlib.decompress(z) == d
        except zlib.error:
            ok = False
        if ok:
            assert g == d
        else:
            assert str(g) == "deflate backend failed to decompress block"
