"""Seeded synthetic fields standing in for the BASELINE.json workloads.

The reference measures on SDRBench-class datasets that are not
in this image; these generators reproduce the shapes, dtypes and value statistics
BASELINE.json names for configs 1-5.  They are workload
generators for bench.py and the tests, not part of the compression path.
"""
from __future__ import annotations

import math

import numpy as np

# BASELINE.json configs: dims, dtype, interp (1 = cubic, the reference default), relative eb
CONFIGS = {
    1: dict(dims=(64, 64, 64), dtype=np.float32, interp=0, rel_eb=1e-3,
            retrieve=dict(rel=[1e-2, 1e-3])),
    2: dict(dims=(512, 512, 512), dtype=np.float32, interp=1, rel_eb=1e-4,
            retrieve=dict(rel=[1e-1, 1e-2, 1e-3, 1e-4])),
    3: dict(dims=(1800, 3600), dtype=np.float32, interp=1, rel_eb=1e-3,
            retrieve=dict(bitrate=[0.5, 1.0, 2.0, 4.0])),
    4: dict(dims=(100, 500, 500), dtype=np.float32, interp=1, rel_eb=1e-5,
            retrieve=dict(rel=[1e-5])),
    5: dict(dims=(256, 384, 384), dtype=np.float64, interp=1, rel_eb=1e-7,
            retrieve=dict(rel=[1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7])),
}


def smooth_field(dims, seed: int, max_waves: int = 8) -> np.ndarray:
    """Sum of 1..max_waves random sinusoids over the unit cube (the reference's only
    test-field family, tests/field_util.hpp:14-51; own seeded generator)."""
    rng = np.random.default_rng(seed)
    waves = 1 + int(rng.integers(0, max_waves))
    grids = np.meshgrid(*[np.arange(d, dtype=np.float64) / d for d in dims], indexing="ij")
    out = np.zeros(dims, dtype=np.float64)
    for _ in range(waves):
        a = rng.uniform(0.2, 1.0)
        p = rng.uniform(0.0, 2 * math.pi)
        arg = np.full(dims, p)
        for g in grids:
            arg = arg + rng.uniform(0.5, 4.0) * 2 * math.pi * g
        out += a * np.sin(arg)
    return out.reshape(-1)


def spectral_field(dims, alpha: float, seed: int, device: str | None = None) -> np.ndarray:
    """Gaussian random field with isotropic power spectrum P(k) ~ k^-alpha (k != 0),
    by FFT synthesis of seeded white noise.  Returns float64 flattened, zero mean."""
    import torch

    dev = device or ("cuda" if torch.cuda.is_available() else "cpu")
    g = torch.Generator(device="cpu").manual_seed(seed)
    noise = torch.randn(*dims, generator=g, dtype=torch.float32)
    x = noise.to(dev)
    spec = torch.fft.rfftn(x)
    ks = []
    for i, d in enumerate(dims):
        if i == len(dims) - 1:
            k = torch.fft.rfftfreq(d, device=dev) * d
        else:
            k = torch.fft.fftfreq(d, device=dev) * d
        shape = [1] * len(dims)
        shape[i] = -1
        ks.append(k.reshape(shape).to(torch.float32))
    k2 = sum(k * k for k in ks)
    amp = torch.where(k2 > 0, k2.clamp_min(1e-12) ** (-alpha / 4.0), torch.zeros_like(k2))
    spec = spec * amp
    out = torch.fft.irfftn(spec, s=dims)
    res = out.double().cpu().numpy().reshape(-1)
    del x, spec, out
    return res


def make_field(cfg: int, seed: int = 0, dims=None, device: str | None = None) -> np.ndarray:
    """Synthetic field of BASELINE config `cfg` (optionally at reduced dims for parity tests)."""
    c = CONFIGS[cfg]
    dims = tuple(dims or c["dims"])
    rng = np.random.default_rng(1000 + seed)
    if cfg == 1:
        # sum of 4 random-phase sinusoids, wavelengths 8-64 cells, amplitude 1, + N(0, 1e-3)
        grids = np.meshgrid(*[np.arange(d, dtype=np.float64) for d in dims], indexing="ij")
        v = np.zeros(dims)
        for _ in range(4):
            lam = rng.uniform(8.0, 64.0)
            direc = rng.normal(size=len(dims))
            direc /= np.linalg.norm(direc)
            ph = rng.uniform(0, 2 * math.pi)
            arg = ph + sum(direc[i] * grids[i] for i in range(len(dims))) * (2 * math.pi / lam)
            v += np.sin(arg)
        v += rng.normal(0.0, 1e-3, size=dims)
        out = v.reshape(-1)
    elif cfg == 2:
        f = spectral_field(dims, 11.0 / 3.0, seed, device)
        out = (f - f.min()) / (f.max() - f.min())
    elif cfg == 3:
        ny, nx = dims
        lat = (np.arange(ny) + 0.5) / ny * math.pi - math.pi / 2
        base = np.cos(lat)[:, None] * np.ones((1, nx))
        pert = spectral_field(dims, 3.0, seed, device).reshape(dims)
        pert = pert / (pert.std() + 1e-30) * (base.std() / 10.0)
        v = base + pert
        mask = np.zeros(dims, dtype=bool)
        target = int(0.05 * ny * nx)
        while mask.sum() < target:
            h = int(rng.integers(max(2, ny // 60), max(3, ny // 12)))
            w = int(rng.integers(max(2, nx // 60), max(3, nx // 12)))
            y0 = int(rng.integers(0, ny - h + 1))
            x0 = int(rng.integers(0, nx - w + 1))
            mask[y0:y0 + h, x0:x0 + w] = True
        v[mask] = 1e20
        out = v.reshape(-1)
    elif cfg == 4:
        f = spectral_field(dims, 5.0 / 3.0, seed, device).reshape(dims)
        std = f.std()
        grids = [np.arange(d, dtype=np.float64) for d in dims]
        for _ in range(200):
            ctr = [rng.uniform(0, d) for d in dims]
            sig = rng.uniform(2.0, 6.0)
            amp = 50.0 * std * (1 if rng.random() < 0.5 else -1)
            sl = []
            gs = []
            for i, d in enumerate(dims):
                lo = max(0, int(ctr[i] - 4 * sig))
                hi = min(d, int(ctr[i] + 4 * sig) + 1)
                sl.append(slice(lo, hi))
                gs.append(grids[i][lo:hi] - ctr[i])
            r2 = gs[0][:, None, None] ** 2 + gs[1][None, :, None] ** 2 + gs[2][None, None, :] ** 2
            f[tuple(sl)] += amp * np.exp(-r2 / (2 * sig * sig))
        out = f.reshape(-1)
    elif cfg == 5:
        f = spectral_field(dims, 2.0, seed, device).reshape(dims)
        f = f / (f.std() + 1e-30)
        z = np.linspace(0.0, 1e6, dims[0])[:, None, None]
        out = (f + z).reshape(-1)
    else:
        raise ValueError(cfg)
    return np.ascontiguousarray(out.astype(c["dtype"]))


def abs_eb(values: np.ndarray, rel: float) -> float:
    """Relative bound -> absolute, as the reference CLI does (tools/main.cpp:125-134):
    rel * (max - min) with lo/hi seeded from values[0]."""
    v = values.astype(np.float64)
    return float(rel * (v.max() - v.min()))
