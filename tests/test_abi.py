"""CPU: the C-ABI boundary (include/ipcomp_b200.h).

* the sm_100a library loads without a GPU and exports every symbol the header declares;
* the host half of the boundary (index parsing = ArchiveReader, planner = planner.cpp)
  agrees with the oracle on real archives, through context-free calls (no device needed);
* the planner's edge behaviour mirrors the reference (InfeasibleRequest).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ipcomp_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ipcg_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ipc.library()
    names = declared_symbols()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(ipc.EXPORTED_SYMBOLS) == names


def test_library_is_sm100a_and_links_no_zlib():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", ipc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", ipc.LIB_PATH], capture_output=True, text=True).stdout
    assert "libz" not in deps  # the lossless stage is our own GPU deflate/inflate


class HostReader(ipc.ArchiveReader):
    def __init__(self, data: bytes):
        super().__init__(data, ctx=ipc.HostContext())


@pytest.mark.parametrize("dims,interp,lp", [((65, 33), 0, 0), ((17, 13, 11), 1, 0), ((6, 7, 8, 9), 1, 2), ((3, 1), 1, 0)])
def test_index_and_planner_match_oracle(dims, interp, lp, oracle_lib):
    f = synth.smooth_field(dims, 12)
    eb = 1e-4 * (f.max() - f.min())
    arch = oracle_lib.compress(f, dims, eb, interp, lp)
    r = HostReader(arch)
    info = oracle_lib.info(arch)
    assert r.levels == info.levels and r.identity() == info.identity
    assert r.index_bytes() == info.index_bytes and r.header().payload_bytes == info.payload_bytes
    for l in range(info.levels):
        rec = r.record(l + 1)
        assert list(rec.delta) == list(info.delta[l])
        assert list(rec.plane_length) == list(info.plane_length[l])
    for fac in (1.0, 4.0, 64.0, 1024.0, 1e6):
        assert ipc.plan_for_error(r, fac * eb).k == oracle_lib.plan_for_error(arch, fac * eb)
        k = oracle_lib.plan_for_error(arch, fac * eb)
        assert ipc.bound_for_plan(r, k) == oracle_lib.bound_for_plan(arch, k)
        assert ipc.plan_payload_bytes(r, k) == oracle_lib.plan_payload_bytes(arch, k)
    total = oracle_lib.plan_payload_bytes(arch, [32] * info.levels)
    for frac in (0.0, 0.3, 0.7, 1.0):
        b = int(total * frac)
        try:
            want = oracle_lib.plan_for_size(arch, b)
        except oracle.InfeasibleRequest:
            with pytest.raises(ipc.InfeasibleRequest):
                ipc.plan_for_size(r, b)
            continue
        assert ipc.plan_for_size(r, b).k == want


def test_malformed_index_is_rejected_like_the_reference(oracle_lib):
    f = synth.smooth_field((33,), 3)
    arch = oracle_lib.compress(f, (33,), 1e-3, 1)
    with pytest.raises(RuntimeError, match="not an archive: bad magic"):
        HostReader(b"X" + arch[1:])
    with pytest.raises(RuntimeError, match="unsupported archive version"):
        HostReader(arch[:4] + bytes([9]) + arch[5:])
    with pytest.raises(RuntimeError, match="truncated archive index"):
        HostReader(arch[:40])
    r = HostReader(arch)
    with pytest.raises(ipc.InfeasibleRequest):
        ipc.plan_for_error(r, 1e-9)
