"""Compress graphs (ipcg.cu compress_entry): a device-resident field of a shape compressed before
replays the captured kernel sequence of its compress as one CUDA graph.  Every call -- the
first (normal, tallying its scratch), the second (captured, then replayed) and later replays --
must give the oracle's archive bytes, for changing field contents of one shape, across graph
evictions, for outlier-heavy fields whose replay falls back to the exact-size assembly, and the
archives a replay returns must stay valid across later replays (they are copied out of the
graph's slab)."""
import numpy as np
import pytest

import paper_2502_04093_b200 as ipc
from paper_2502_04093_b200 import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _eb(f, rel):
    return rel * (float(np.max(f)) - float(np.min(f)))


@pytest.mark.parametrize("dims,dtype,interp", [((64, 64, 64), np.float32, 1), ((90, 180), np.float32, 1),
                                               ((24, 36, 36), np.float64, 1), ((17, 18, 19), np.float32, 0),
                                               ((513,), np.float64, 0)])
def test_replays_match_oracle(dims, dtype, interp, oracle_lib):
    ctx = ipc.Context(0)
    fields = [synth.smooth_field(dims, s).astype(dtype) for s in (3, 4)]
    eb = _eb(fields[0], 1e-4)
    archives = []
    for it in range(5):
        f = fields[it % 2]
        l0 = ctx.kernel_launches()
        r = ipc.compress_field(torch.from_numpy(f).cuda(), dims, eb, interp, ctx=ctx)
        assert ctx.kernel_launches() > l0
        got = r.to_bytes()
        assert got == oracle_lib.compress(f, dims, eb, interp), f"call {it}"
        archives.append((r, got))
    for r, want in archives:  # earlier replays' archives were not overwritten by later ones
        assert r.to_bytes() == want
    # a retrieval from a replayed archive
    r, want = archives[-1]
    f = fields[0]
    plan = ipc.full_plan(r)
    out = ipc.reconstruct_field(r, plan)
    ref, _, _ = oracle_lib.reconstruct(want, plan.k, dtype, f.size)
    assert out.values.tobytes() == ref.tobytes()


def test_eviction_and_many_keys(oracle_lib):
    ctx = ipc.Context(0)
    dims = (33, 21, 9)
    f = synth.smooth_field(dims, 9).astype(np.float32)
    ft = torch.from_numpy(f).cuda()
    rels = [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 3e-3]  # more keys than the context keeps
    for rep in range(3):
        for rel in rels:
            eb = _eb(f, rel)
            assert ipc.compress_field(ft, dims, eb, 1, ctx=ctx).to_bytes() == oracle_lib.compress(f, dims, eb, 1)
    for lp in (1, 2, 0, 1):  # progressive-level option is part of the key
        eb = _eb(f, 1e-4)
        assert ipc.compress_field(ft, dims, eb, 1, lp, ctx=ctx).to_bytes() == oracle_lib.compress(f, dims, eb, 1, lp)


def test_outlier_heavy_replay_falls_back(oracle_lib):
    ctx = ipc.Context(0)
    dims = (40, 50, 30)
    rng = np.random.default_rng(5)
    smooth = synth.smooth_field(dims, 2).astype(np.float32)
    spiky = smooth.copy()
    idx = rng.choice(spiky.size, spiky.size // 8, replace=False)  # 1/8 outliers: over the 1/64 allowance
    spiky.reshape(-1)[idx] = rng.normal(0, 1e6, idx.size).astype(np.float32)
    eb = _eb(smooth, 1e-4)
    for f in (smooth, smooth, spiky, smooth, spiky, spiky):
        got = ipc.compress_field(torch.from_numpy(f).cuda(), dims, eb, 1, ctx=ctx).to_bytes()
        assert got == oracle_lib.compress(f, dims, eb, 1)
