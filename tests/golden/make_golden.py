"""Generate tests/golden/ fixtures from the UNMODIFIED reference (oracle/_ref, compiled
from /root/reference/proj/src by `make -C oracle ref`).

Each case stores the input field, the compression options, the archive bytes the
reference writes, the session file it writes for one plan (.ips), and SHA-256 digests of the reference's reconstructions for a few
plans (incl. one refine step) plus its planner outputs.  The fixtures pin the C
restatement (oracle/) and the GPU path without needing the reference tree, which does
not exist on the GPU box.  Re-run only when the reference changes:

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2502_04093_b200 import synth  # noqa: E402

CASES = [
    # name, field builder, dims, dtype, rel eb, interp, lp
    ("smooth_1d_cubic", lambda: synth.smooth_field((257,), 1000), (257,), np.float64, 1e-4, 1, 0),
    ("smooth_2d_linear", lambda: synth.smooth_field((33, 21), 1001), (33, 21), np.float64, 1e-4, 0, 0),
    ("smooth_3d_f32_cubic", lambda: synth.smooth_field((17, 18, 19), 1002), (17, 18, 19), np.float32, 1e-3, 1, 0),
    ("smooth_4d_lp2", lambda: synth.smooth_field((6, 7, 8, 9), 1003), (6, 7, 8, 9), np.float64, 1e-5, 1, 2),
    ("cfg1_32cube", lambda: synth.make_field(1, dims=(32, 32, 32)), (32, 32, 32), np.float32, 1e-3, 0, 0),
    ("cfg4_spikes", lambda: synth.make_field(4, dims=(12, 30, 30)), (12, 30, 30), np.float32, 1e-5, 1, 0),
    ("cfg5_gradient_f64", lambda: synth.make_field(5, dims=(16, 24, 24)), (16, 24, 24), np.float64, 1e-7, 1, 0),
    ("outliers_nonfinite", None, (40,), np.float64, None, 1, 0),
    ("tiny_2", lambda: np.array([-1.0, -0.5]), (2,), np.float64, None, 1, 0),
]


def field_for(name, builder, dims, dtype):
    if name == "outliers_nonfinite":
        v = np.ones(40)
        v[7] = np.inf
        v[21] = 1e60
        v[22] = -1e60
        v[30] = np.nan
        return v.astype(dtype)
    return np.ascontiguousarray(builder()).astype(dtype)


def main():
    ref = oracle.load("ref")
    manifest = []
    rng = np.random.default_rng(2502)
    for name, builder, dims, dtype, rel, interp, lp in CASES:
        f = field_for(name, builder, dims, dtype)
        finite = f[np.isfinite(f)].astype(np.float64)
        eb = 1e-6 if rel is None else rel * float(finite.max() - finite.min())
        if name == "tiny_2":
            eb = 1e-4
        arch = ref.compress(f, dims, eb, interp, lp)
        info = oracle.load("oracle").info(arch)
        L, LP = info.levels, info.progressive_levels
        plans = [[32] * L, [0 if l + 1 <= LP else 32 for l in range(L)]]
        plans.append([32 if l + 1 > LP else int(rng.integers(0, 33)) for l in range(L)])
        recon = []
        for k in plans:
            v, merged, loaded = ref.reconstruct(arch, k, dtype, f.size)
            recon.append({"k": k, "sha256": hashlib.sha256(v.tobytes()).hexdigest(), "loaded": int(loaded)})
        k1 = plans[2]
        v1, m1, _ = ref.reconstruct(arch, k1, dtype, f.size)
        k2 = [min(32, x + 7) if l + 1 <= LP else 32 for l, x in enumerate(k1)]
        v2, _, loaded2 = ref.refine(arch, k1, m1, v1, k2)
        refine = {"k1": k1, "k2": k2, "sha256": hashlib.sha256(v2.tobytes()).hexdigest(), "loaded": int(loaded2)}
        sess = ref.write_session(arch, k1, m1)  # write_session (session.cpp:8-24) of the k1 session
        with open(os.path.join(HERE, f"{name}.ips"), "wb") as fh:
            fh.write(sess)
        session = {"k": k1, "sha256": hashlib.sha256(sess).hexdigest(), "bytes": len(sess)}
        planner = {}
        for fac in (4.0, 64.0, 4096.0):
            planner[f"error_x{int(fac)}"] = ref.plan_for_error(arch, fac * eb)
        tot = ref.plan_payload_bytes(arch, [32] * L)
        for frac in (0.5, 1.0):
            try:
                planner[f"size_{frac}"] = ref.plan_for_size(arch, int(tot * frac))
            except oracle.InfeasibleRequest:
                planner[f"size_{frac}"] = "infeasible"
        np.save(os.path.join(HERE, f"{name}.input.npy"), f)
        with open(os.path.join(HERE, f"{name}.ipc"), "wb") as fh:
            fh.write(arch)
        manifest.append({"name": name, "dims": list(dims), "dtype": np.dtype(dtype).name, "eb": eb,
                         "interp": interp, "lp": lp, "archive_sha256": hashlib.sha256(arch).hexdigest(),
                         "archive_bytes": len(arch), "recon": recon, "refine": refine, "planner": planner,
                         "session": session})
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("wrote", len(manifest), "golden cases")


if __name__ == "__main__":
    main()
