"""CPU: the position-parallel deflate decomposition (paper_2502_04093_b200/csrc/deflate_core.cuh,
run sequentially by tests/native/zmodel.cpp) must produce exactly zlib 1.3's compress2(level 6)
bytes -- the reference's lossless stage (proj/src/backend.cpp:15-22).  The GPU kernels call the
same device functions, so this pins their semantics without a GPU.  zlib is the system libz the
reference links (not vendored, version not pinned by the reference; 1.3 in this image).
"""
import ctypes as C
import os
import subprocess
import zlib

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "zmodel.cpp")
LIB = os.path.join(HERE, "native", "libzmodel.so")


@pytest.fixture(scope="module")
def zmodel():
    core = os.path.join(os.path.dirname(HERE), "paper_2502_04093_b200", "csrc", "deflate_core.cuh")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(core)):
        subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-o", LIB, SRC], check=True)
    lib = C.CDLL(LIB)
    lib.zmodel_compress.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_char_p, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    lib.zmodel_crc_combine.restype = C.c_uint32
    lib.zmodel_crc_combine.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]

    lib.zmodel_compress_od.argtypes = lib.zmodel_compress.argtypes

    def run(data: bytes, chunk: int = 2048, ondemand: bool = False) -> bytes:
        cap = 2 * len(data) + 1024
        out = C.create_string_buffer(cap)
        n = C.c_uint64()
        st = (C.c_uint64 * 6)()
        f = lib.zmodel_compress_od if ondemand else lib.zmodel_compress
        assert f(data, len(data), chunk, out, cap, C.byref(n), st) == 0
        return out.raw[: n.value]

    run.lib = lib
    return run


def _cases():
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 4, 100, 4095, 16384, 65535, 65536, 65537, 65800, 131072 + 65536 + 100, 300000):
        yield f"zeros{n}", bytes(n)
        yield f"rand{n}", rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        for p in (0.02, 0.3):
            bits = (rng.random(n * 8) < p).astype(np.uint8)
            yield f"bits{p}_{n}", np.packbits(bits, bitorder="little").tobytes()
        yield f"runs{n}", np.repeat(rng.integers(0, 3, n // 50 + 1, dtype=np.uint8),
                                    rng.integers(1, 300, n // 50 + 1))[:n].tobytes()
        yield f"text{n}", (b"the quick brown fox %d jumps over " * (n // 30 + 1))[:n]
        yield f"longruns{n}", np.repeat(rng.integers(0, 4, n // 500 + 1, dtype=np.uint8),
                                        rng.integers(1, 5000, n // 500 + 1))[:n].tobytes()
    # window-slide boundaries: tail slides with the head exactly at MAX_DIST
    for k in range(3):
        base = 32768 * k + 65536
        for d in (-262, -261, -1, 0, 1, 261, 262):
            n = base + d
            yield f"edge_rand{n}", rng.integers(0, 256, n, dtype=np.uint8).tobytes()
            yield f"edge_runs{n}", np.repeat(rng.integers(0, 3, n // 40 + 1, dtype=np.uint8),
                                             rng.integers(1, 200, n // 40 + 1))[:n].tobytes()


CASES = list(_cases())


@pytest.mark.parametrize("name,data", CASES, ids=[c[0] for c in CASES])
def test_model_equals_zlib_level6(zmodel, name, data):
    want = zlib.compress(data, 6)
    assert zmodel(data) == want
    assert zmodel(data, chunk=257) == want
    # the on-demand chunked parse (what the GPU runs for streams < 2^31 bytes), with chunk sizes
    # that put joins inside matches, across several chunks and at the stream end
    for ch in (64, 300, 1024, 8192):
        assert zmodel(data, chunk=ch, ondemand=True) == want, ch


def test_model_on_real_bitplanes(zmodel, oracle_lib):
    from paper_2502_04093_b200 import synth

    for cfg, dims in ((2, (48, 48, 48)), (4, (20, 50, 50)), (5, (24, 32, 32))):
        f = synth.make_field(cfg, dims=dims)
        eb = synth.abs_eb(f, synth.CONFIGS[cfg]["rel_eb"])
        _, tr = oracle_lib.compress(f, dims, eb, synth.CONFIGS[cfg]["interp"], trace=True)
        for lt in tr:
            for p in range(32):
                raw = lt.xor_planes[p].tobytes()
                if raw:
                    want = zlib.compress(raw, 6)
                    assert zmodel(raw) == want, (cfg, lt.count, p)
                    assert zmodel(raw, chunk=1024, ondemand=True) == want, (cfg, lt.count, p)


def test_crc_combine(zmodel):
    rng = np.random.default_rng(3)
    for la, lb in ((1, 1), (4096, 411), (100000, 3), (0, 7), (7, 0), (4096, 4096)):
        a = rng.integers(0, 256, la, dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, lb, dtype=np.uint8).tobytes()
        assert zmodel.lib.zmodel_crc_combine(zlib.crc32(a), zlib.crc32(b), lb) == zlib.crc32(a + b)


def test_fast_match_search_equals_reference_form(zmodel):
    """match_search32 (what k_match runs) gives the same record as match_search at every
    position: runs, sparse bit patterns, periodic text, tails shorter than a word."""
    lib = zmodel.lib
    lib.zmodel_match_check.restype = C.c_uint64
    lib.zmodel_match_check.argtypes = [C.c_char_p, C.c_uint64]
    rng = np.random.default_rng(11)
    datas = [d for _, d in CASES if len(d) <= 70000]
    for n in (5, 6, 7, 9, 258, 259, 261, 263, 1000):
        for p in (0.01, 0.05, 0.5):
            bits = (rng.random(n * 8) < p).astype(np.uint8)
            datas.append(np.packbits(bits, bitorder="little").tobytes())
        datas.append(bytes([7]) * n)
        datas.append((b"ab" * n)[:n])
    for d in datas:
        assert lib.zmodel_match_check(d, len(d)) == 0, len(d)
