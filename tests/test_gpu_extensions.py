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
