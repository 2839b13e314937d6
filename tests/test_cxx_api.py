"""The header-only C++ mirror of the reference API (include/ipcomp_b200.hpp) used as a
reference user would use <ipcomp/pipeline.hpp>: builds against the C-ABI library on the
CPU; on the GPU its archive / reconstruction / refinement must equal the oracle's."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "cxx_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2502_04093_b200")


@pytest.fixture(scope="module")
def cxx_api(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cxx") / "cxx_api")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lipcomp_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cxx_header_builds_and_fails_loudly_without_gpu(cxx_api, tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    f = tmp_path / "f.bin"
    np.zeros(64, np.float32).tofile(f)
    r = subprocess.run([cxx_api, str(f), "4", "4", "4", "0.1", "1", str(tmp_path / "o")],
                       capture_output=True, text=True)
    assert r.returncode == 10 and "cannot create" in r.stderr  # CudaError, no CPU fallback


@pytest.mark.gpu
def test_cxx_api_matches_oracle(cxx_api, tmp_path, oracle_lib):
    from paper_2502_04093_b200 import synth

    dims = (20, 33, 27)
    f = synth.make_field(2, dims=dims)
    eb = synth.abs_eb(f, 1e-4)
    rng = float(f.max() - f.min())
    path = tmp_path / "f.bin"
    f.tofile(path)
    pre = str(tmp_path / "o")
    r = subprocess.run([cxx_api, str(path), *map(str, dims), repr(eb), repr(1e-2 * rng), pre],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    arch = open(pre + ".archive", "rb").read()
    assert arch == oracle_lib.compress(f, dims, eb, 1)
    k = [int(x) for x in r.stdout.split("plan")[1].split("bytes_read")[0].split()]
    want1, m1, _ = oracle_lib.reconstruct(arch, k, np.float32, f.size)
    assert open(pre + ".recon", "rb").read() == want1.tobytes()
    want2, _, _ = oracle_lib.refine(arch, k, m1, want1, [32] * len(k))
    assert open(pre + ".refine", "rb").read() == want2.tobytes()
    assert open(pre + ".session", "rb").read() == oracle_lib.write_session(arch, k, m1)
    assert open(pre + ".refine2", "rb").read() == want2.tobytes()
    line = next(ln for ln in r.stdout.splitlines() if ln.startswith("max_error"))
    vals = [float(x) for x in line.split()[1::2]]
    want_m = oracle_lib.compute_metrics(f, want2)
    assert vals[0] == want_m[0] and vals[1] == pytest.approx(want_m[1], rel=1e-12)
