"""CPU ORACLE -- test infrastructure only.

ctypes access to
  * ``oracle/liboracle.so``: the plain-C restatement of the reference IPComp hot
    path (``oracle/ipcomp_oracle.c``), and
  * ``oracle/_ref/libipcomp_ref.so``: the UNMODIFIED reference compiled from
    ``/root/reference/proj/src`` (``make -C oracle ref``), used to pin the
    restatement and as the CPU baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs import this package, and only as the checker.  The
product package ``paper_2502_04093_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libipcomp_ref.so")
MAX_LEVELS = 16

ERROR_KINDS = {1: ValueError, 2: RuntimeError, 3: ArithmeticError, 4: RuntimeError}


class InfeasibleRequest(RuntimeError):
    pass


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Trace(C.Structure):
    _fields_ = [
        ("levels", C.c_int),
        ("count", C.c_uint64 * MAX_LEVELS),
        ("codes", C.POINTER(C.c_int32) * MAX_LEVELS),
        ("negabinary", C.POINTER(C.c_uint32) * MAX_LEVELS),
        ("n_outliers", C.c_uint64 * MAX_LEVELS),
        ("outlier_ordinal", C.POINTER(C.c_uint64) * MAX_LEVELS),
        ("outlier_bytes", C.POINTER(C.c_uint8) * MAX_LEVELS),
        ("xor_planes", C.POINTER(C.c_uint8) * MAX_LEVELS),
        ("delta", (C.c_double * 33) * MAX_LEVELS),
    ]


class Info(C.Structure):
    _fields_ = [
        ("scalar", C.c_int), ("interp", C.c_int), ("ndims", C.c_int), ("levels", C.c_int),
        ("progressive_levels", C.c_int), ("anchor_cap", C.c_int),
        ("dims", C.c_uint64 * 4),
        ("eb", C.c_double), ("range", C.c_double),
        ("index_bytes", C.c_uint64), ("payload_bytes", C.c_uint64),
        ("identity", C.c_uint32),
        ("count", C.c_uint64 * MAX_LEVELS),
        ("delta", (C.c_double * 33) * MAX_LEVELS),
        ("outlier_offset", C.c_uint64 * MAX_LEVELS),
        ("outlier_length", C.c_uint64 * MAX_LEVELS),
        ("outlier_count", C.c_uint64 * MAX_LEVELS),
        ("plane_offset", (C.c_uint64 * 32) * MAX_LEVELS),
        ("plane_length", (C.c_uint64 * 32) * MAX_LEVELS),
    ]


def build(ref: bool | None = None) -> None:
    """Compile the restatement (and, when the reference tree exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _setup(lib: C.CDLL, pfx: str) -> C.CDLL:
    u8p = C.POINTER(C.c_uint8)
    f = getattr(lib, pfx + "compress")
    f.restype = C.c_int
    lib_args = [C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64,
                C.POINTER(u8p), C.POINTER(C.c_uint64)]
    if pfx == "orc_":
        lib_args.append(C.POINTER(Trace))
    lib_args += [C.c_char_p, C.c_int]
    f.argtypes = lib_args
    f = getattr(lib, pfx + "reconstruct")
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_int), C.c_void_p,
                  C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
    f = getattr(lib, pfx + "refine")
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_uint32)),
                  C.c_void_p, C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.POINTER(C.c_uint32)),
                  C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
    for name, extra in (("plan_for_error", C.c_double), ("plan_for_size", C.c_uint64)):
        f = getattr(lib, pfx + name)
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_uint64, extra, C.POINTER(C.c_int), C.c_char_p, C.c_int]
    f = getattr(lib, pfx + "bound_for_plan")
    f.restype = C.c_double
    f.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]
    f = getattr(lib, pfx + "plan_payload_bytes")
    f.restype = C.c_uint64
    f.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]
    f = getattr(lib, pfx + "backend_encode")
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(u8p), C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                  C.POINTER(C.c_uint32)]
    getattr(lib, pfx + "free").argtypes = [C.c_void_p]
    f = getattr(lib, pfx + "compute_metrics")
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_double)]
    f = getattr(lib, pfx + "read_session")
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.POINTER(C.c_int),
                  C.POINTER(C.POINTER(C.c_uint32)), C.c_char_p, C.c_int]
    if pfx == "ref_":
        lib.ref_write_session.restype = C.c_int
        lib.ref_write_session.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int),
                                          C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(u8p), C.POINTER(C.c_uint64),
                                          C.c_char_p, C.c_int]
    if pfx == "orc_":
        lib.orc_trace_free.argtypes = [C.POINTER(Trace)]
        lib.orc_archive_info.restype = C.c_int
        lib.orc_archive_info.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(Info), C.c_char_p, C.c_int]
        lib.orc_crc32.restype = C.c_uint32
        lib.orc_crc32.argtypes = [C.c_void_p, C.c_uint64]
        lib.orc_write_session.restype = C.c_int
        lib.orc_write_session.argtypes = [C.c_uint32, C.c_int, C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_uint32)),
                                          C.POINTER(C.c_uint64), C.POINTER(u8p), C.POINTER(C.c_uint64)]
    return lib


@dataclass
class LevelTrace:
    count: int
    codes: np.ndarray
    negabinary: np.ndarray
    outlier_ordinal: np.ndarray
    outlier_bytes: bytes
    xor_planes: np.ndarray  # (32, plane_bytes) uint8
    delta: np.ndarray


@dataclass
class Oracle:
    """One loaded CPU implementation (restatement or reference) behind one interface."""

    lib: C.CDLL
    pfx: str
    name: str
    _bufs: list = field(default_factory=list)

    def _err(self, rc: int, buf) -> None:
        if rc == 0:
            return
        msg = buf.value.decode(errors="replace")
        if rc == 4:
            raise InfeasibleRequest(msg)
        raise OracleError(rc, msg)

    def compress(self, values: np.ndarray, dims, eb: float, interp: int = 1, progressive_levels: int = 0,
                 anchor_cap: int = 64, trace: bool = False):
        values = np.ascontiguousarray(values)
        scalar = 0 if values.dtype == np.float32 else 1
        assert values.dtype in (np.float32, np.float64)
        d = (C.c_uint64 * len(dims))(*dims)
        out = C.POINTER(C.c_uint8)()
        size = C.c_uint64()
        err = C.create_string_buffer(512)
        f = getattr(self.lib, self.pfx + "compress")
        args = [scalar, values.ctypes.data, d, len(dims), eb, interp, progressive_levels, anchor_cap,
                C.byref(out), C.byref(size)]
        tr = Trace() if trace else None
        if self.pfx == "orc_":
            args.append(C.byref(tr) if trace else None)
        elif trace:
            raise ValueError("trace is only available from the restatement")
        rc = f(*args, err, 512)
        self._err(rc, err)
        data = C.string_at(out, size.value)
        getattr(self.lib, self.pfx + "free")(out)
        if not trace:
            return data
        levels = []
        for li in range(tr.levels):
            cnt = tr.count[li]
            pb = (cnt + 7) // 8
            no = tr.n_outliers[li]
            w = 4 if scalar == 0 else 8
            levels.append(LevelTrace(
                count=cnt,
                codes=np.ctypeslib.as_array(tr.codes[li], (max(cnt, 1),))[:cnt].copy(),
                negabinary=np.ctypeslib.as_array(tr.negabinary[li], (max(cnt, 1),))[:cnt].copy(),
                outlier_ordinal=(np.ctypeslib.as_array(tr.outlier_ordinal[li], (no,)).copy() if no
                                 else np.zeros(0, np.uint64)),
                outlier_bytes=C.string_at(tr.outlier_bytes[li], no * (8 + w)) if no else b"",
                xor_planes=np.ctypeslib.as_array(tr.xor_planes[li], (32 * max(pb, 1),))[:32 * pb].reshape(32, pb).copy(),
                delta=np.array(tr.delta[li][:], dtype=np.float64),
            ))
        self.lib.orc_trace_free(C.byref(tr))
        return data, levels

    def info(self, archive: bytes) -> Info:
        inf = Info()
        err = C.create_string_buffer(512)
        rc = self.lib.orc_archive_info(archive, len(archive), C.byref(inf), err, 512)
        self._err(rc, err)
        return inf

    def _levels(self, archive: bytes) -> int:
        return archive_levels(archive)

    def reconstruct(self, archive: bytes, k, dtype, n: int):
        L = len(k)
        kk = (C.c_int * L)(*k)
        out = np.empty(n, dtype=dtype)
        merged = (C.POINTER(C.c_uint32) * MAX_LEVELS)()
        loaded = C.c_uint64()
        err = C.create_string_buffer(512)
        f = getattr(self.lib, self.pfx + "reconstruct")
        rc = f(archive, len(archive), 0 if dtype == np.float32 else 1, kk, out.ctypes.data, merged,
               C.byref(loaded), err, 512)
        self._err(rc, err)
        return out, self._collect_merged(archive, merged, L), loaded.value

    def _collect_merged(self, archive, merged, L):
        counts = archive_counts(archive)
        res = []
        for li in range(L):
            if merged[li]:
                cnt = counts[li]
                res.append(np.ctypeslib.as_array(merged[li], (max(cnt, 1),))[:cnt].copy())
                getattr(self.lib, self.pfx + "free")(merged[li])
            else:
                res.append(None)
        return res

    def refine(self, archive: bytes, session_k, session_merged, previous: np.ndarray, target_k):
        L = len(target_k)
        sk = (C.c_int * L)(*session_k)
        tk = (C.c_int * L)(*target_k)
        keep = []
        sm = (C.POINTER(C.c_uint32) * MAX_LEVELS)()
        for li, m in enumerate(session_merged):
            if m is not None:
                a = np.ascontiguousarray(m, dtype=np.uint32)
                keep.append(a)
                sm[li] = a.ctypes.data_as(C.POINTER(C.c_uint32))
        prev = np.ascontiguousarray(previous)
        out = np.empty_like(prev)
        merged = (C.POINTER(C.c_uint32) * MAX_LEVELS)()
        loaded = C.c_uint64()
        err = C.create_string_buffer(512)
        f = getattr(self.lib, self.pfx + "refine")
        rc = f(archive, len(archive), 0 if prev.dtype == np.float32 else 1, sk, sm, prev.ctypes.data, tk,
               out.ctypes.data, merged, C.byref(loaded), err, 512)
        self._err(rc, err)
        return out, self._collect_merged(archive, merged, L), loaded.value

    def write_session(self, archive: bytes, session_k, session_merged) -> bytes:
        """write_session (session.cpp:8-24) of the session {k, merged} bound to `archive`."""
        L = archive_levels(archive)
        sk = (C.c_int * L)(*session_k)
        keep = []
        sm = (C.POINTER(C.c_uint32) * MAX_LEVELS)()
        for li, m in enumerate(session_merged):
            if m is not None:
                a = np.ascontiguousarray(m, dtype=np.uint32)
                keep.append(a)
                sm[li] = a.ctypes.data_as(C.POINTER(C.c_uint32))
        out = C.POINTER(C.c_uint8)()
        size = C.c_uint64()
        if self.pfx == "ref_":
            err = C.create_string_buffer(512)
            rc = self.lib.ref_write_session(archive, len(archive), sk, sm, C.byref(out), C.byref(size), err, 512)
            self._err(rc, err)
        else:
            counts = (C.c_uint64 * MAX_LEVELS)(*archive_counts(archive))
            self.lib.orc_write_session(self.info(archive).identity, L, sk, sm, counts, C.byref(out), C.byref(size))
        data = C.string_at(out, size.value)
        getattr(self.lib, self.pfx + "free")(out)
        return data

    def read_session(self, archive: bytes, data: bytes):
        """read_session (session.cpp:26-61) -> (planes_loaded, merged per level or None)."""
        L = archive_levels(archive)
        k = (C.c_int * MAX_LEVELS)()
        merged = (C.POINTER(C.c_uint32) * MAX_LEVELS)()
        err = C.create_string_buffer(512)
        rc = getattr(self.lib, self.pfx + "read_session")(archive, len(archive), data, len(data), k, merged, err, 512)
        self._err(rc, err)
        return list(k)[:L], self._collect_merged(archive, merged, L)

    def compute_metrics(self, original: np.ndarray, decoded: np.ndarray):
        """compute_metrics<T> (pipeline.hpp:354-372) -> (max_error, mse, psnr)."""
        a, b = np.ascontiguousarray(original), np.ascontiguousarray(decoded)
        assert a.dtype == b.dtype and a.size == b.size
        out = (C.c_double * 3)()
        getattr(self.lib, self.pfx + "compute_metrics")(0 if a.dtype == np.float32 else 1, a.ctypes.data,
                                                         b.ctypes.data, a.size, out)
        return tuple(out)

    def plan_for_error(self, archive: bytes, max_error: float):
        L = archive_levels(archive)
        k = (C.c_int * L)()
        err = C.create_string_buffer(512)
        rc = getattr(self.lib, self.pfx + "plan_for_error")(archive, len(archive), max_error, k, err, 512)
        self._err(rc, err)
        return list(k)

    def plan_for_size(self, archive: bytes, budget: int):
        L = archive_levels(archive)
        k = (C.c_int * L)()
        err = C.create_string_buffer(512)
        rc = getattr(self.lib, self.pfx + "plan_for_size")(archive, len(archive), int(budget), k, err, 512)
        self._err(rc, err)
        return list(k)

    def bound_for_plan(self, archive: bytes, k) -> float:
        kk = (C.c_int * len(k))(*k)
        return getattr(self.lib, self.pfx + "bound_for_plan")(archive, len(archive), kk)

    def plan_payload_bytes(self, archive: bytes, k) -> int:
        kk = (C.c_int * len(k))(*k)
        return getattr(self.lib, self.pfx + "plan_payload_bytes")(archive, len(archive), kk)

    def backend_encode(self, raw: bytes, preferred: int = 1):
        out = C.POINTER(C.c_uint8)()
        n = C.c_uint64()
        be = C.c_int()
        crc = C.c_uint32()
        getattr(self.lib, self.pfx + "backend_encode")(raw, len(raw), preferred, C.byref(out), C.byref(n),
                                                       C.byref(be), C.byref(crc))
        data = C.string_at(out, n.value)
        getattr(self.lib, self.pfx + "free")(out)
        return be.value, data, crc.value


def archive_levels(archive: bytes) -> int:
    nd = archive[8]
    return archive[12 + 8 * nd + 8]


def archive_counts(archive: bytes) -> list[int]:
    """Per-level point counts [l-1] read straight from the index layout (README.md:93-101)."""
    nd = archive[8]
    L = archive_levels(archive)
    pos = 12 + 8 * nd + 8 + 4 + 8
    rec = 8 * (1 + 33 + 3 + 64)
    counts = [0] * L
    for level in range(L, 0, -1):
        counts[level - 1] = int.from_bytes(archive[pos:pos + 8], "little")
        pos += rec
    return counts


_cache: dict = {}


def load(which: str = "oracle") -> Oracle:
    """'oracle' -> C restatement; 'ref' -> the compiled reference (oracle/_ref)."""
    if which in _cache:
        return _cache[which]
    if which == "oracle":
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        o = Oracle(_setup(C.CDLL(LIB_PATH), "orc_"), "orc_", "oracle")
    elif which == "ref":
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError(REF_PATH)
        o = Oracle(_setup(C.CDLL(REF_PATH), "ref_"), "ref_", "ref")
    else:
        raise ValueError(which)
    _cache[which] = o
    return o


def ref_available() -> bool:
    return os.path.exists(REF_PATH)
