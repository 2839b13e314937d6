"""CPU: pin the oracle (oracle/, the C restatement) before trusting it.

1. Against the golden fixtures the UNMODIFIED reference wrote (tests/golden/, made by
   tests/golden/make_golden.py from oracle/_ref): archive bytes, reconstruction and refine
   digests, planner outputs.
2. Against the compiled reference itself (oracle/_ref) when it is present in this container.
3. The reference's own known-answer tests for the path (proj/tests/test_pipeline.cpp,
   test_quantizer.cpp, test_bitplane.cpp), restated through the oracle's traces.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_2502_04093_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


@pytest.mark.parametrize("case", MANIFEST, ids=[c["name"] for c in MANIFEST])
def test_oracle_reproduces_golden_reference_outputs(case, oracle_lib):
    f = np.load(os.path.join(GOLDEN, case["name"] + ".input.npy"))
    arch = oracle_lib.compress(f, tuple(case["dims"]), case["eb"], case["interp"], case["lp"])
    want = open(os.path.join(GOLDEN, case["name"] + ".ipc"), "rb").read()
    assert arch == want
    for r in case["recon"]:
        v, _, loaded = oracle_lib.reconstruct(arch, r["k"], f.dtype, f.size)
        assert hashlib.sha256(v.tobytes()).hexdigest() == r["sha256"]
        assert loaded == r["loaded"]
    rf = case["refine"]
    v1, m1, _ = oracle_lib.reconstruct(arch, rf["k1"], f.dtype, f.size)
    v2, _, loaded2 = oracle_lib.refine(arch, rf["k1"], m1, v1, rf["k2"])
    assert hashlib.sha256(v2.tobytes()).hexdigest() == rf["sha256"] and loaded2 == rf["loaded"]
    for key, want_k in case["planner"].items():
        if key.startswith("error_x"):
            fac = float(key[len("error_x"):])
            assert oracle_lib.plan_for_error(arch, fac * case["eb"]) == want_k
        else:
            frac = float(key[len("size_"):])
            tot = oracle_lib.plan_payload_bytes(arch, [32] * len(case["recon"][0]["k"]))
            try:
                got = oracle_lib.plan_for_size(arch, int(tot * frac))
            except oracle.InfeasibleRequest:
                got = "infeasible"
            assert got == want_k


@pytest.mark.parametrize("case", MANIFEST, ids=[c["name"] for c in MANIFEST])
def test_oracle_session_file_matches_golden(case, oracle_lib):
    """write_session / read_session (session.cpp:8-61) against the session file the reference wrote."""
    arch = open(os.path.join(GOLDEN, case["name"] + ".ipc"), "rb").read()
    want = open(os.path.join(GOLDEN, case["name"] + ".ips"), "rb").read()
    sess = case["session"]
    assert hashlib.sha256(want).hexdigest() == sess["sha256"]
    f = np.load(os.path.join(GOLDEN, case["name"] + ".input.npy"))
    _, m, _ = oracle_lib.reconstruct(arch, sess["k"], f.dtype, f.size)
    assert oracle_lib.write_session(arch, sess["k"], m) == want
    k, m2 = oracle_lib.read_session(arch, want)
    assert k == sess["k"]
    for a, b in zip(m, m2):
        assert (a is None and b is None) or np.array_equal(a, b)


def _session_corruptions(good: bytes):
    yield good[:3]
    yield b"XPS1" + good[4:]
    yield good[:4] + bytes(4) + good[8:]
    yield good[:-1]
    yield good + b"\0"
    yield good[:8] + bytes([33]) + good[9:]   # plane count out of range
    yield good[:9] + bytes([7]) + good[10:]   # unknown backend id
    yield good[:20] + bytes([good[20] ^ 1]) + good[21:]  # payload length
    yield good[:-2] + bytes([good[-2] ^ 0x40]) + good[-1:]  # payload byte -> checksum
    for cut in (9, 12, 20, 29):
        yield good[:cut]


def test_oracle_metrics_known_answers(oracle_lib):  # test_pipeline.cpp:355-390
    a = np.array([1.0, 2.0, 3.0])
    m = oracle_lib.compute_metrics(a, a)
    assert m[0] == 0.0 and m[1] == 0.0 and np.isinf(m[2])
    a = np.array([0.0, 10.0, 5.0, 2.5])
    b = a.copy()
    b[2] += 0.125
    m = oracle_lib.compute_metrics(a, b)
    assert m[0] == 0.125 and m[1] == 0.125 * 0.125 / 4.0
    assert m[2] == pytest.approx(20.0 * np.log10(10.0 / np.sqrt(0.125 * 0.125 / 4.0)), rel=1e-12)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (reference tree absent)")
def test_oracle_metrics_equal_reference(oracle_lib):
    ref = oracle.load("ref")
    rng = np.random.default_rng(19)
    for dt in (np.float32, np.float64):
        a = rng.uniform(-3, 3, 5000).astype(dt)
        b = (a + 0.01 * rng.uniform(-3, 3, a.size)).astype(dt)
        b[11], a[12], b[13] = np.nan, np.inf, -np.inf
        for x, y in ((a, b), (a[:100], a[:100]), (a[:0], b[:0])):
            got, want = oracle_lib.compute_metrics(x, y), ref.compute_metrics(x, y)
            assert np.array_equal(np.array(got), np.array(want), equal_nan=True)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (reference tree absent)")
@pytest.mark.parametrize("lp", [0, 2])
def test_oracle_session_reader_errors_match_reference(lp, oracle_lib):
    ref = oracle.load("ref")
    dims = (20, 24, 18)
    f = synth.smooth_field(dims, 3).astype(np.float32)
    arch = oracle_lib.compress(f, dims, 1e-3 * float(f.max() - f.min()), 1, lp)
    L = oracle.archive_levels(arch)
    k = [5 + 3 * i if i < (lp or L) else 32 for i in range(L)]
    _, m, _ = oracle_lib.reconstruct(arch, k, np.float32, f.size)
    good = ref.write_session(arch, k, m)
    assert oracle_lib.write_session(arch, k, m) == good
    for bad in _session_corruptions(good):
        res = []
        for impl in (oracle_lib, ref):
            try:
                impl.read_session(arch, bad)
                res.append("ok")
            except oracle.OracleError as e:
                res.append(str(e))
        assert res[0] == res[1], (len(bad), res)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (reference tree absent)")
@pytest.mark.parametrize("dims,interp,dtype", [((1,), 1, np.float64), ((3, 1), 0, np.float32), ((65,), 1, np.float64),
                                               ((9, 7, 33), 1, np.float32), ((2, 3, 4, 5), 0, np.float64),
                                               ((40, 36), 1, np.float32)])
def test_oracle_matches_compiled_reference(dims, interp, dtype, oracle_lib):
    ref = oracle.load("ref")
    f = synth.smooth_field(dims, 99).astype(dtype)
    eb = 1e-5 * (float(f.max()) - float(f.min())) or 1e-3
    a = oracle_lib.compress(f, dims, eb, interp)
    assert a == ref.compress(f, dims, eb, interp)
    L = oracle.archive_levels(a)
    rng = np.random.default_rng(1)
    for _ in range(3):
        k = [int(x) for x in rng.integers(0, 33, L)]
        va, ma, la = oracle_lib.reconstruct(a, k, dtype, f.size)
        vb, mb, lb = ref.reconstruct(a, k, dtype, f.size)
        assert va.tobytes() == vb.tobytes() and la == lb


# ---- known answers from the reference's own tests ---------------------------------
def test_linear_ramp_codes_are_zero_below_anchor(oracle_lib):  # test_pipeline.cpp:65-79
    v = np.arange(65, dtype=np.float64)
    for interp in (0, 1):
        _, tr = oracle_lib.compress(v, (65,), 0.5, interp, trace=True)
        for lt in tr[:-1]:
            assert not lt.codes.any() and lt.delta[32] == 0.0
        assert tr[-1].delta[32] > 0.0


def test_negabinary_codewords(oracle_lib):  # test_quantizer.cpp:87-93
    # codes 1, -1, 2 at the anchors of a 3-point grid: to_negabinary(1)=0b1, (-1)=0b11, (2)=0b110
    v = np.array([2.0, -2.0, 4.0])  # eb 1 -> bins of width 2 -> codes 1, -1, 2 (coarsest predicts 0)
    _, tr = oracle_lib.compress(v, (3,), 1.0, 1, trace=True)
    top = tr[-1]
    assert list(top.codes) == [1, 2]
    assert list(top.negabinary) == [0b1, 0b110]
    # level 1 predicts (2+4)/2 = 3, residual -5 -> round(-2.5) = -3 (half away from zero)
    assert list(tr[0].codes) == [-3]

    def value(w):  # definitional base -2 evaluation (test_quantizer.cpp:14-22)
        return sum((-2) ** k for k in range(32) if (int(w) >> k) & 1)

    assert value(tr[0].negabinary[0]) == -3
    for q in (0, 1, -1, 2, -2, 1 << 30, -(1 << 30), 12345, -98765):
        v = np.zeros(2)
        v[0] = 2.0 * q
        _, t = oracle_lib.compress(v, (2,), 1.0, 1, trace=True)
        assert value(t[-1].negabinary[0]) == q


def test_xor_plane_coding_by_hand(oracle_lib):  # test_bitplane.cpp:59-70 semantics on planes
    rng = np.random.default_rng(4)
    v = rng.normal(size=4096)
    _, tr = oracle_lib.compress(v, (4096,), 1e-6, 1, trace=True)
    lt = tr[0]
    # rebuild planes from the codewords and apply e_p = b_p ^ b_{p-1} ^ b_{p-2}
    nb = lt.negabinary
    b = np.zeros((32, (lt.count + 7) // 8), np.uint8)
    for p in range(32):
        bits = ((nb >> (31 - p)) & 1).astype(np.uint8)
        b[p] = np.packbits(bits, bitorder="little")[: b.shape[1]]
    e = b.copy()
    for p in range(1, 32):
        e[p] ^= b[p - 1]
        if p >= 2:
            e[p] ^= b[p - 2]
    assert np.array_equal(e, lt.xor_planes)


def test_one_dimensional_loss_table_equals_suffix_measurement(oracle_lib):  # test_pipeline.cpp:476-505
    f = synth.smooth_field((201,), 1881)
    eb = 1e-4 * (f.max() - f.min())
    for interp in (0, 1):
        _, tr = oracle_lib.compress(f, (201,), eb, interp, trace=True)
        for lt in tr:
            running = 0.0
            for d in range(33):
                mask = 0 if d == 32 else (~((1 << d) - 1)) & 0xFFFFFFFF
                t = ((lt.negabinary & np.uint32(mask)) ^ np.uint32(0xAAAAAAAA)).astype(np.int64) - 0xAAAAAAAA
                t = ((t + 2**31) % 2**32) - 2**31
                worst = np.max(np.abs(2.0 * eb * (t - lt.codes.astype(np.int64)))) if lt.count else 0.0
                running = max(running, worst)
                assert lt.delta[d] == running


def test_full_retrieval_within_bound(oracle_lib):  # test_pipeline.cpp:81-96
    for dims in ((257,), (33, 21), (17, 18, 19)):
        f = synth.smooth_field(dims, 1000)
        eb = 1e-4 * (f.max() - f.min())
        a = oracle_lib.compress(f, dims, eb, 1)
        L = oracle.archive_levels(a)
        v, _, _ = oracle_lib.reconstruct(a, [32] * L, np.float64, f.size)
        assert np.max(np.abs(v - f)) <= eb
