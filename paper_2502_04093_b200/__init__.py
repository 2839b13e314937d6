"""B200-native IPComp hot path (arXiv 2502.04093) -- Python binding of the C-ABI.

Mirrors the reference's public interface (proj/include/ipcomp/pipeline.hpp, archive.hpp,
planner.hpp, session.hpp): ``compress_field``, ``ArchiveReader``, ``build_error_model``,
``plan_for_error``, ``plan_for_size``, ``bound_for_plan``, ``plan_payload_bytes``,
``full_plan``, ``reconstruct_field``, ``refine_field``; errors raise the Python
counterparts of the reference's exception types.  All compute runs in the in-tree
sm_100a library ``libipcomp_b200.so`` (include/ipcomp_b200.h); there is no CPU path --
importing works without a GPU, but every compute call fails loudly without one.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libipcomp_b200.so")
MAX_LEVELS = 16


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ArithmeticError):
    """std::domain_error"""


class InfeasibleRequest(RuntimeError):
    """ipcomp::InfeasibleRequest (common.hpp:23-25)"""


class CudaError(RuntimeError):
    """device failure (no reference counterpart)"""


_KIND = {1: InvalidArgument, 2: RuntimeError, 3: DomainError, 4: InfeasibleRequest, 5: CudaError}

LINEAR, CUBIC = 0, 1


class LevelRecord(C.Structure):
    _fields_ = [("count", C.c_uint64), ("delta", C.c_double * 33), ("outlier_offset", C.c_uint64),
                ("outlier_length", C.c_uint64), ("outlier_count", C.c_uint64),
                ("plane_offset", C.c_uint64 * 32), ("plane_length", C.c_uint64 * 32)]


class Index(C.Structure):
    _fields_ = [("version", C.c_uint16), ("scalar", C.c_uint8), ("interp", C.c_uint8), ("ndims", C.c_uint8),
                ("levels", C.c_uint8), ("progressive_levels", C.c_uint8), ("anchor_cap", C.c_uint8),
                ("dims", C.c_uint64 * 4), ("eb", C.c_double), ("range", C.c_double),
                ("payload_bytes", C.c_uint64), ("index_bytes", C.c_uint64), ("identity", C.c_uint32),
                ("records", LevelRecord * MAX_LEVELS)]


class RetrieveStats(C.Structure):
    _fields_ = [("payload_bytes_loaded", C.c_uint64), ("level_visits", C.c_int * MAX_LEVELS)]


class LevelCosts(C.Structure):
    _fields_ = [("delta", C.c_double * 33), ("plane_bytes", C.c_uint64 * 32), ("outlier_bytes", C.c_uint64),
                ("progressive", C.c_int)]


class ErrorModelC(C.Structure):
    _fields_ = [("levels", C.c_int), ("progressive_levels", C.c_int), ("eb", C.c_double),
                ("amplification", C.c_double), ("level", LevelCosts * MAX_LEVELS)]


READ_FN = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64)

_lib = None


def library() -> C.CDLL:
    """Load the sm_100a library; raises if it was not built (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run paper_2502_04093_b200.build.build() (nvcc, sm_100a)")
    lib = C.CDLL(LIB_PATH)
    vp, u64, i32, dbl = C.c_void_p, C.c_uint64, C.c_int, C.c_double
    P = C.POINTER
    sig = {
        "ipcg_ctx_create": (i32, [i32, P(vp)]),
        "ipcg_ctx_destroy": (None, [vp]),
        "ipcg_last_error": (C.c_char_p, [vp]),
        "ipcg_set_stream": (i32, [vp, vp]),
        "ipcg_synchronize": (i32, [vp]),
        "ipcg_set_host_async": (i32, [vp, i32]),
        "ipcg_stage_field": (i32, [vp, vp, u64]),
        "ipcg_compress": (i32, [vp, i32, vp, i32, P(u64), i32, dbl, i32, i32, u64, P(vp)]),
        "ipcg_archive_open": (i32, [vp, vp, u64, i32, P(vp)]),
        "ipcg_archive_open_source": (i32, [vp, READ_FN, vp, P(vp)]),
        "ipcg_archive_read_range": (i32, [vp, vp, u64, u64, vp]),
        "ipcg_archive_copy": (i32, [vp, vp, u64, u64, vp, i32]),
        "ipcg_index_serialize": (i32, [P(Index), vp, u64, P(u64)]),
        "ipcg_index_parse": (i32, [vp, u64, P(Index)]),
        "ipcg_crc32": (C.c_uint32, [vp, u64]),
        "ipcg_archive_index": (i32, [vp, P(Index)]),
        "ipcg_archive_size": (u64, [vp]),
        "ipcg_archive_write": (i32, [vp, vp, vp, i32, u64]),
        "ipcg_archive_payload_bytes_read": (u64, [vp]),
        "ipcg_archive_free": (None, [vp]),
        "ipcg_reconstruct": (i32, [vp, vp, i32, P(i32), vp, i32, u64, P(vp), P(RetrieveStats)]),
        "ipcg_refine": (i32, [vp, vp, i32, vp, vp, i32, u64, P(i32), vp, i32, u64, P(vp), P(RetrieveStats)]),
        "ipcg_session_create": (i32, [vp, vp, P(i32), P(P(C.c_uint32)), P(vp)]),
        "ipcg_session_levels": (i32, [vp]),
        "ipcg_session_archive_crc": (C.c_uint32, [vp]),
        "ipcg_session_planes_loaded": (i32, [vp, P(i32)]),
        "ipcg_session_count": (u64, [vp, i32]),
        "ipcg_session_merged": (i32, [vp, vp, i32, vp, i32]),
        "ipcg_session_free": (None, [vp]),
        "ipcg_session_write_bound": (u64, [vp]),
        "ipcg_session_write": (i32, [vp, vp, vp, i32, u64, P(u64)]),
        "ipcg_session_read": (i32, [vp, vp, vp, u64, i32, P(vp)]),
        "ipcg_compute_metrics": (i32, [vp, i32, vp, i32, u64, vp, i32, u64, P(dbl), P(dbl), P(dbl)]),
        "ipcg_plan_for_error": (i32, [vp, vp, dbl, P(i32)]),
        "ipcg_plan_for_size": (i32, [vp, vp, u64, P(i32)]),
        "ipcg_bound_for_plan": (dbl, [vp, P(i32)]),
        "ipcg_plan_payload_bytes": (u64, [vp, P(i32)]),
        "ipcg_build_error_model": (i32, [P(Index), P(ErrorModelC)]),
        "ipcg_model_plan_for_error": (i32, [P(ErrorModelC), dbl, P(i32)]),
        "ipcg_model_plan_for_size": (i32, [P(ErrorModelC), u64, P(i32)]),
        "ipcg_model_plan_device": (i32, [vp, P(ErrorModelC), i32, dbl, u64, P(i32)]),
        "ipcg_model_bound_for_plan": (dbl, [P(ErrorModelC), P(i32)]),
        "ipcg_model_plan_payload_bytes": (u64, [P(ErrorModelC), P(i32)]),
        "ipcg_model_mandatory_payload_bytes": (u64, [P(ErrorModelC)]),
        "ipcg_model_total_payload_bytes": (u64, [P(ErrorModelC)]),
        "ipcg_split": (i32, [vp, vp, u64, i32, P(C.c_void_p)]),
        "ipcg_plane_xor": (i32, [vp, P(C.c_void_p), u64, i32, i32]),
        "ipcg_merge": (i32, [vp, P(C.c_void_p), u64, i32, vp]),
        "ipcg_backend_encode": (i32, [vp, vp, i32, u64, u64, i32, vp, vp, vp, vp, u64]),
        "ipcg_kernel_launches": (u64, [vp]),
        "ipcg_profile_enable": (i32, [vp, i32]),
        "ipcg_backend_decode": (i32, [vp, vp, vp, vp, vp, vp, i32, vp, vp]),
        "ipcg_profile_read": (i32, [vp, C.c_char_p, u64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


EXPORTED_SYMBOLS = [
    "ipcg_ctx_create", "ipcg_ctx_destroy", "ipcg_last_error", "ipcg_set_stream", "ipcg_synchronize",
    "ipcg_set_host_async", "ipcg_stage_field",
    "ipcg_compress", "ipcg_archive_open", "ipcg_archive_index", "ipcg_archive_size", "ipcg_archive_write",
    "ipcg_archive_open_source", "ipcg_archive_read_range", "ipcg_archive_copy", "ipcg_index_serialize",
    "ipcg_index_parse", "ipcg_crc32", "ipcg_build_error_model", "ipcg_model_plan_for_error",
    "ipcg_model_plan_for_size", "ipcg_model_plan_device", "ipcg_model_bound_for_plan", "ipcg_model_plan_payload_bytes",
    "ipcg_model_mandatory_payload_bytes", "ipcg_model_total_payload_bytes", "ipcg_split", "ipcg_plane_xor",
    "ipcg_merge",
    "ipcg_archive_payload_bytes_read", "ipcg_archive_free", "ipcg_reconstruct", "ipcg_refine",
    "ipcg_session_create", "ipcg_session_levels", "ipcg_session_archive_crc", "ipcg_session_planes_loaded",
    "ipcg_session_count", "ipcg_session_merged", "ipcg_session_free",
    "ipcg_session_write_bound", "ipcg_session_write", "ipcg_session_read", "ipcg_compute_metrics", "ipcg_plan_for_error",
    "ipcg_plan_for_size", "ipcg_bound_for_plan", "ipcg_plan_payload_bytes", "ipcg_backend_encode",
    "ipcg_kernel_launches", "ipcg_profile_enable", "ipcg_profile_read", "ipcg_backend_decode",
]


class Context:
    """One CUDA device + stream (ipcg_ctx)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        lib = library()
        h = C.c_void_p()
        rc = lib.ipcg_ctx_create(device, C.byref(h))
        if rc:
            raise CudaError(f"cannot create context on cuda:{device} (rc={rc})")
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def check(self, rc: int) -> None:
        if rc:
            msg = library().ipcg_last_error(self.h).decode(errors="replace")
            raise _KIND.get(rc, RuntimeError)(msg)

    def set_stream(self, stream_ptr: int) -> None:
        self.check(library().ipcg_set_stream(self.h, C.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        self.check(library().ipcg_synchronize(self.h))

    def set_host_async(self, enable: bool = True) -> None:
        """Host-async mode (ipcg_set_host_async): retrievals into host buffers return once the
        values are final on the device; the copy-out lands by the next synchronize()."""
        self.check(library().ipcg_set_host_async(self.h, 1 if enable else 0))

    def stage_field(self, values) -> None:
        """Start uploading a HOST field (ipcg_stage_field); the next compress_field of the same
        buffer on this context compresses the staged device copy."""
        addr, on_dev, nbytes = _ptr(values)
        if on_dev:
            raise ValueError("stage_field takes a host field")
        self.check(library().ipcg_stage_field(self.h, C.c_void_p(addr), nbytes))

    def kernel_launches(self) -> int:
        return int(library().ipcg_kernel_launches(self.h))

    def profile(self, enable: bool = True) -> None:
        self.check(library().ipcg_profile_enable(self.h, 1 if enable else 0))

    def profile_read(self) -> dict:
        import json

        buf = C.create_string_buffer(1 << 16)
        self.check(library().ipcg_profile_read(self.h, buf, 1 << 16))
        return {k: {"ms": v[0], "scopes": v[1], "bytes": v[2]} for k, v in json.loads(buf.value.decode()).items()}

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib is not None:
                _lib.ipcg_ctx_destroy(self.h)
        except Exception:
            pass


class HostContext:
    """Context-free handle for host-only calls (index parsing, planning): no device needed."""

    h = None
    device = 0

    def check(self, rc: int) -> None:
        if rc:
            msg = library().ipcg_last_error(None).decode(errors="replace")
            raise _KIND.get(rc, RuntimeError)(msg)


def _ptr(x):
    """(address, on_device, nbytes) of a numpy array or torch tensor."""
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data, 0, x.nbytes
    try:
        import torch

        if isinstance(x, torch.Tensor):
            assert x.is_contiguous()
            return x.data_ptr(), 1 if x.is_cuda else 0, x.numel() * x.element_size()
    except ImportError:
        pass
    if isinstance(x, (bytes, bytearray)):
        buf = np.frombuffer(x, dtype=np.uint8)
        return buf.ctypes.data, 0, len(x)
    raise TypeError(f"unsupported buffer type {type(x)}")


def _scalar_of(x) -> int:
    dt = getattr(x, "dtype", None)
    s = str(dt)
    if "float32" in s:
        return 0
    if "float64" in s:
        return 1
    raise InvalidArgument("field scalars must be f32 or f64")


@dataclass
class ArchiveHeader:
    scalar: int
    interp: int
    dims: tuple
    eb: float
    range: float
    levels: int
    progressive_levels: int
    anchor_cap: int
    payload_bytes: int
    version: int = 1


class ArchiveReader:
    """ArchiveReader (archive.hpp:63-113): parsed index over archive bytes held in host
    memory (bytes / numpy) or device memory (torch CUDA tensor).  The bytes are borrowed
    and kept alive by this object.  Also the owner of a freshly compressed archive."""

    def __init__(self, data=None, ctx: Context | None = None, _handle=None):
        self.ctx = ctx or Context.default()
        lib = library()
        self._keep = data
        if _handle is not None:
            self.h = _handle
        else:
            if isinstance(data, (bytes, bytearray)):
                data = np.frombuffer(bytes(data), dtype=np.uint8)
                self._keep = data
            addr, on_dev, nbytes = _ptr(data)
            h = C.c_void_p()
            self.ctx.check(lib.ipcg_archive_open(self.ctx.h, C.c_void_p(addr), nbytes, on_dev, C.byref(h)))
            self.h = h
        self._ix = Index()
        lib.ipcg_archive_index(self.h, C.byref(self._ix))

    # -- reference accessors
    def header(self) -> ArchiveHeader:
        ix = self._ix
        return ArchiveHeader(ix.scalar, ix.interp, tuple(ix.dims[: ix.ndims]), ix.eb, ix.range, ix.levels,
                             ix.progressive_levels, ix.anchor_cap, ix.payload_bytes, ix.version)

    def record(self, level: int) -> LevelRecord:
        return self._ix.records[level - 1]

    def identity(self) -> int:
        return int(self._ix.identity)

    def index_bytes(self) -> int:
        return int(self._ix.index_bytes)

    def payload_bytes_read(self) -> int:
        return int(library().ipcg_archive_payload_bytes_read(self.h))

    @property
    def levels(self) -> int:
        return int(self._ix.levels)

    @property
    def dims(self) -> tuple:
        return tuple(self._ix.dims[: self._ix.ndims])

    @property
    def dtype(self):
        return np.float32 if self._ix.scalar == 0 else np.float64

    def size(self) -> int:
        return int(library().ipcg_archive_size(self.h))

    def to_bytes(self) -> bytes:
        """write_archive (archive.cpp:72-81)"""
        n = self.size()
        out = np.empty(n, dtype=np.uint8)
        self.ctx.check(library().ipcg_archive_write(self.ctx.h, self.h, C.c_void_p(out.ctypes.data), 0, n))
        return out.tobytes()

    def write_to(self, dst) -> None:
        addr, on_dev, nbytes = _ptr(dst)
        self.ctx.check(library().ipcg_archive_write(self.ctx.h, self.h, C.c_void_p(addr), on_dev, nbytes))

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib is not None:
                _lib.ipcg_archive_free(self.h)
        except Exception:
            pass


def compress_field(values, dims, eb: float, interp: int = CUBIC, progressive_levels: int = 0,
                   anchor_cap: int = 64, ctx: Context | None = None) -> ArchiveReader:
    """compress_field<T> (pipeline.hpp:140-223); values: numpy (host) or torch CUDA tensor."""
    ctx = ctx or Context.default()
    addr, on_dev, nbytes = _ptr(values)
    d = (C.c_uint64 * len(dims))(*[int(x) for x in dims])
    h = C.c_void_p()
    ctx.check(library().ipcg_compress(ctx.h, _scalar_of(values), C.c_void_p(addr), on_dev, d, len(dims), float(eb),
                                      int(interp), int(progressive_levels), int(anchor_cap), C.byref(h)))
    return ArchiveReader(ctx=ctx, _handle=h)


@dataclass
class RetrievalPlan:
    k: list


@dataclass
class ReconstructStats:
    level_visits: list
    payload_bytes_loaded: int


class RetrievalSession:
    """RetrievalSession (session.hpp:19-34); merged codewords stay device-resident."""

    def __init__(self, h, ctx: Context):
        self.h = h
        self.ctx = ctx

    @property
    def archive_crc(self) -> int:
        return int(library().ipcg_session_archive_crc(self.h))

    def planes_loaded(self) -> list:
        n = library().ipcg_session_levels(self.h)
        k = (C.c_int * n)()
        library().ipcg_session_planes_loaded(self.h, k)
        return list(k)

    def plan(self) -> RetrievalPlan:
        return RetrievalPlan(self.planes_loaded())

    def merged(self, level: int):
        cnt = library().ipcg_session_count(self.h, level)
        out = np.empty(cnt, dtype=np.uint32)
        if cnt:
            self.ctx.check(library().ipcg_session_merged(self.ctx.h, self.h, level, C.c_void_p(out.ctypes.data), 0))
            return out
        return None

    @classmethod
    def from_host(cls, reader: ArchiveReader, planes_loaded, merged) -> "RetrievalSession":
        L = reader.levels
        k = (C.c_int * L)(*planes_loaded)
        arr = (C.POINTER(C.c_uint32) * L)()
        keep = []
        for i, m in enumerate(merged):
            if m is not None:
                a = np.ascontiguousarray(m, dtype=np.uint32)
                keep.append(a)
                arr[i] = a.ctypes.data_as(C.POINTER(C.c_uint32))
        h = C.c_void_p()
        reader.ctx.check(library().ipcg_session_create(reader.ctx.h, reader.h, k, arr, C.byref(h)))
        return cls(h, reader.ctx)

    def to_bytes(self) -> bytes:
        """write_session (session.cpp:8-24); codewords deflated on the GPU."""
        return write_session(self)

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib is not None:
                _lib.ipcg_session_free(self.h)
        except Exception:
            pass


def write_session(session: RetrievalSession, dst=None) -> bytes | int:
    """write_session (session.cpp:8-24).  Returns the file bytes, or, with `dst` (a host or
    device buffer: numpy array / torch tensor), writes into it and returns the size."""
    lib = library()
    ctx = session.ctx
    size = C.c_uint64()
    if dst is None:
        buf = np.empty(max(1, int(lib.ipcg_session_write_bound(session.h))), np.uint8)
        ctx.check(lib.ipcg_session_write(ctx.h, session.h, C.c_void_p(buf.ctypes.data), 0, buf.nbytes,
                                         C.byref(size)))
        return buf[:size.value].tobytes()
    addr, on_dev, nbytes = _ptr(dst)
    ctx.check(lib.ipcg_session_write(ctx.h, session.h, C.c_void_p(addr), on_dev, nbytes, C.byref(size)))
    return int(size.value)


def read_session(data, reader: "ArchiveReader") -> RetrievalSession:
    """read_session (session.cpp:26-61): `data` is bytes or a host/device buffer."""
    addr, on_dev, nbytes = _ptr(data)
    h = C.c_void_p()
    reader.ctx.check(library().ipcg_session_read(reader.ctx.h, reader.h, C.c_void_p(addr), nbytes, on_dev,
                                                 C.byref(h)))
    return RetrievalSession(h, reader.ctx)


@dataclass
class Retrieved:
    values: object
    session: RetrievalSession | None
    stats: ReconstructStats = field(default_factory=lambda: ReconstructStats([], 0))


def _plan_arr(plan, L):
    k = plan.k if isinstance(plan, RetrievalPlan) else list(plan)
    if len(k) != L:
        raise InvalidArgument("plan level count does not match archive")
    return (C.c_int * L)(*[int(x) for x in k])


def _out_buffer(reader: ArchiveReader, out, device: bool):
    n = int(np.prod(reader.dims))
    if out is not None:
        return out
    if device:
        import torch

        return torch.empty(n, dtype=torch.float32 if reader.dtype == np.float32 else torch.float64,
                           device=f"cuda:{reader.ctx.device}")
    return np.empty(n, dtype=reader.dtype)


def reconstruct_field(reader: ArchiveReader, plan, dtype=None, out=None, device: bool = False,
                      keep_session: bool = True) -> Retrieved:
    """reconstruct_field<T> (pipeline.hpp:260-287)."""
    lib = library()
    scalar = reader._ix.scalar if dtype is None else (0 if np.dtype(dtype) == np.float32 else 1)
    k = _plan_arr(plan, reader.levels)
    out = _out_buffer(reader, out, device)
    addr, on_dev, nbytes = _ptr(out)
    sess = C.c_void_p()
    st = RetrieveStats()
    w = 4 if scalar == 0 else 8
    reader.ctx.check(lib.ipcg_reconstruct(reader.ctx.h, reader.h, scalar, k, C.c_void_p(addr), on_dev, nbytes // w,
                                          C.byref(sess) if keep_session else None, C.byref(st)))
    s = RetrievalSession(sess, reader.ctx) if keep_session else None
    return Retrieved(out, s, ReconstructStats(list(st.level_visits[: reader.levels]), int(st.payload_bytes_loaded)))


def refine_field(reader: ArchiveReader, session: RetrievalSession, previous, plan, out=None,
                 keep_session: bool = True) -> Retrieved:
    """refine_field<T> (pipeline.hpp:294-352)."""
    lib = library()
    k = _plan_arr(plan, reader.levels)
    paddr, pdev, pbytes = _ptr(previous)
    if out is None:
        out = np.empty_like(previous) if isinstance(previous, np.ndarray) else previous.clone()
    addr, on_dev, nbytes = _ptr(out)
    sess = C.c_void_p()
    st = RetrieveStats()
    scalar = _scalar_of(previous)
    w = 4 if scalar == 0 else 8
    reader.ctx.check(lib.ipcg_refine(reader.ctx.h, reader.h, scalar, session.h, C.c_void_p(paddr), pdev,
                                     pbytes // w, k, C.c_void_p(addr), on_dev, nbytes // w,
                                     C.byref(sess) if keep_session else None, C.byref(st)))
    s = RetrievalSession(sess, reader.ctx) if keep_session else None
    return Retrieved(out, s, ReconstructStats(list(st.level_visits[: reader.levels]), int(st.payload_bytes_loaded)))


@dataclass
class FieldMetrics:
    """FieldMetrics (pipeline.hpp:49-53)."""
    max_error: float
    mse: float
    psnr: float


def compute_metrics(original, decoded, ctx: Context | None = None) -> FieldMetrics:
    """compute_metrics<T> (pipeline.hpp:354-372) on the GPU; numpy arrays or torch tensors."""
    ctx = ctx or Context.default()
    pa, da, na = _ptr(original)
    pb, db, nb = _ptr(decoded)
    sa, sb = _scalar_of(original), _scalar_of(decoded)
    if sa != sb:
        raise InvalidArgument("metrics inputs differ in scalar type")
    w = 4 if sa == 0 else 8
    m, e, p = C.c_double(), C.c_double(), C.c_double()
    ctx.check(library().ipcg_compute_metrics(ctx.h, sa, C.c_void_p(pa), da, na // w, C.c_void_p(pb), db, nb // w,
                                             C.byref(m), C.byref(e), C.byref(p)))
    return FieldMetrics(m.value, e.value, p.value)


# ------------------------------------------------------------------ planner
def build_error_model(reader: ArchiveReader) -> ArchiveReader:
    """build_error_model (planner.cpp:30-45): the model is the parsed index itself."""
    return reader


def full_plan(model: ArchiveReader) -> RetrievalPlan:
    return RetrievalPlan([32] * model.levels)


def plan_for_error(model: ArchiveReader, max_error: float) -> RetrievalPlan:
    k = (C.c_int * model.levels)()
    model.ctx.check(library().ipcg_plan_for_error(model.ctx.h, model.h, float(max_error), k))
    return RetrievalPlan(list(k))


def plan_for_size(model: ArchiveReader, byte_budget: int) -> RetrievalPlan:
    k = (C.c_int * model.levels)()
    model.ctx.check(library().ipcg_plan_for_size(model.ctx.h, model.h, int(byte_budget), k))
    return RetrievalPlan(list(k))


def error_model_c(reader: ArchiveReader) -> ErrorModelC:
    """The plain ErrorModel (planner.hpp:13-32) of an archive's index."""
    m = ErrorModelC()
    reader.ctx.check(library().ipcg_build_error_model(C.byref(reader._ix), C.byref(m)))
    return m


def plan_on_device(model, *, max_error: float | None = None, byte_budget: int | None = None,
                   ctx: Context | None = None) -> RetrievalPlan:
    """plan_for_error / plan_for_size as one GPU launch (ipcg_model_plan_device);
    `model` is an ArchiveReader or an ErrorModelC.  Same plans and errors as the host planner."""
    if (max_error is None) == (byte_budget is None):
        raise ValueError("give exactly one of max_error and byte_budget")
    if isinstance(model, ArchiveReader):
        ctx = ctx or model.ctx
        model = error_model_c(model)
    ctx = ctx or Context.default()
    k = (C.c_int * MAX_LEVELS)()
    by_size = byte_budget is not None
    ctx.check(library().ipcg_model_plan_device(ctx.h, C.byref(model), 1 if by_size else 0,
                                               0.0 if by_size else float(max_error), int(byte_budget or 0), k))
    return RetrievalPlan(list(k)[:model.levels])


def bound_for_plan(model: ArchiveReader, plan) -> float:
    return float(library().ipcg_bound_for_plan(model.h, _plan_arr(plan, model.levels)))


def plan_payload_bytes(model: ArchiveReader, plan) -> int:
    return int(library().ipcg_plan_payload_bytes(model.h, _plan_arr(plan, model.levels)))


def backend_encode(planes: np.ndarray, ctx: Context | None = None):
    """backend_encode (backend.cpp:34-53) for a (count, plane_bytes) uint8 array of planes.
    Returns a list of (backend, payload bytes, crc32)."""
    ctx = ctx or Context.default()
    planes = np.ascontiguousarray(planes, dtype=np.uint8)
    if planes.ndim == 1:
        planes = planes[None, :]
    count, nbytes = planes.shape
    be = np.zeros(count, np.uint8)
    ln = np.zeros(count, np.uint64)
    cr = np.zeros(count, np.uint32)
    cap = max(1, count * nbytes)
    out = np.empty(cap, np.uint8)
    ctx.check(library().ipcg_backend_encode(ctx.h, C.c_void_p(planes.ctypes.data), 0, nbytes, nbytes, count,
                                            C.c_void_p(be.ctypes.data), C.c_void_p(ln.ctypes.data),
                                            C.c_void_p(cr.ctypes.data), C.c_void_p(out.ctypes.data), cap))
    res, o = [], 0
    for i in range(count):
        L = int(ln[i])
        res.append((int(be[i]), out[o:o + L].tobytes(), int(cr[i])))
        o += L
    return res


DECODE_ERRORS = {1: "block checksum mismatch", 2: "deflate backend failed to decompress block",
                 3: "identity block has wrong length"}


def backend_decode(blocks, ctx: Context | None = None):
    """backend_decode (backend.cpp:55-65) for a list of (backend, payload bytes, crc32, raw_bytes).
    Returns a list of decoded byte strings, or raises RuntimeError with the reference's message."""
    ctx = ctx or Context.default()
    n = len(blocks)
    payload = np.frombuffer(b"".join(b[1] for b in blocks) + b"\0", dtype=np.uint8)
    plen = np.array([len(b[1]) for b in blocks], np.uint64)
    be = np.array([b[0] for b in blocks], np.uint8)
    crc = np.array([b[2] for b in blocks], np.uint32)
    raw = np.array([b[3] for b in blocks], np.uint64)
    out = np.empty(int(raw.sum()) + 1, np.uint8)
    status = np.zeros(n, np.int32)
    ctx.check(library().ipcg_backend_decode(ctx.h, C.c_void_p(payload.ctypes.data), C.c_void_p(plen.ctypes.data),
                                            C.c_void_p(be.ctypes.data), C.c_void_p(crc.ctypes.data),
                                            C.c_void_p(raw.ctypes.data), n, C.c_void_p(out.ctypes.data),
                                            C.c_void_p(status.ctypes.data)))
    res, o = [], 0
    for i in range(n):
        if status[i]:
            res.append(RuntimeError(DECODE_ERRORS[int(status[i])]))
        else:
            res.append(out[o:o + int(raw[i])].tobytes())
        o += int(raw[i])
    return res
