"""Seeded synthetic fields with the shapes and value distributions of
BASELINE.json's configs (the paper's datasets are not available; these stand
in for them).  Parameters are drawn on the host from
numpy's PCG64 (``np.random.default_rng(seed)``); fields are evaluated in fp64
with torch on the requested device and cast to the config dtype.  Grid
coordinates are x_i = idx_i / (n_i - 1) unless stated.

config 1  129^3 f64: 16 Gaussian bumps + 1e-3 N(0,1) noise
config 2  513^3 f32: config-1 bumps + sum_k (1/k) sin(2 pi k (d_k . x) + phi_k), k=1..8 + 1e-4 noise
config 3  4097^2 f64 on nonuniform coordinates: 64-mode Fourier series, amplitude ~ k^-2
config 4a 100x500x500 f32: exp(-z/0.3) x 2-D Gaussian random fields (power ~ k^-3)
config 4b 288x115x69x69 f32: 32 random waves (amp U[.2,1], freq U[.5,3], phase U[0,2pi))
"""
from __future__ import annotations

import math

import numpy as np


def _torch():
    import torch

    return torch


def _axes(dims, device):
    torch = _torch()
    return [torch.linspace(0.0, 1.0, n, dtype=torch.float64, device=device) if n > 1 else
            torch.zeros(1, dtype=torch.float64, device=device) for n in dims]


def _noise(dims, scale, seed, device):
    torch = _torch()
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 7919 + 17)
    return scale * torch.randn(tuple(dims), generator=g, dtype=torch.float64, device=device)


def bumps(dims, seed=0, n_bumps=16, device="cpu", rng=None):
    """sum_b a_b exp(-|x - c_b|^2 / (2 w_b^2)), c ~ U[0,1]^d, w ~ U[.05,.2], a ~ N(0,1)."""
    torch = _torch()
    rng = rng or np.random.default_rng(seed)
    d = len(dims)
    xs = _axes(dims, device)
    out = torch.zeros(tuple(dims), dtype=torch.float64, device=device)
    for _ in range(n_bumps):
        c = rng.uniform(0.0, 1.0, d)
        w = rng.uniform(0.05, 0.2)
        a = rng.normal()
        term = None
        for i in range(d):
            e = torch.exp(-((xs[i] - c[i]) ** 2) / (2.0 * w * w))
            shape = [1] * d
            shape[i] = dims[i]
            e = e.reshape(shape)
            term = e if term is None else term * e
        out += a * term
    return out


def config1_field(dims=(129, 129, 129), seed=0, device="cpu", dtype=None):
    torch = _torch()
    rng = np.random.default_rng(seed)
    f = bumps(dims, seed, 16, device, rng) + _noise(dims, 1e-3, seed, device)
    return f.to(dtype or torch.float64)


def config2_field(dims=(513, 513, 513), seed=0, device="cpu", dtype=None):
    """Bumps + 8 oblique sine modes + 1e-4 noise, evaluated in fp64."""
    torch = _torch()
    rng = np.random.default_rng(seed)
    f = bumps(dims, seed, 16, device, rng)
    xs = _axes(dims, device)
    d = len(dims)
    for k in range(1, 9):
        dirn = rng.normal(size=d)
        dirn /= np.linalg.norm(dirn)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        arg = None
        for i in range(d):
            shape = [1] * d
            shape[i] = dims[i]
            t = (2.0 * math.pi * k * dirn[i]) * xs[i].reshape(shape)
            arg = t if arg is None else arg + t
        f += (1.0 / k) * torch.sin(arg + phi)
    f += _noise(dims, 1e-4, seed, device)
    return f.to(dtype or torch.float32)


def nonuniform_coords(n, seed=0, axis=0):
    """Sorted cumulative sums of U[0.5, 1.5] spacings, normalised to [0, 1]."""
    rng = np.random.default_rng([seed, axis, 3])
    h = rng.uniform(0.5, 1.5, n - 1)
    x = np.concatenate([[0.0], np.cumsum(h)])
    return x / x[-1]


def config3_field(dims=(4097, 4097), seed=0, device="cpu", dtype=None):
    """64-mode random Fourier series on nonuniform coordinates; returns
    (field, coords).  Modes k in [1,16]^2, a_m = N(0,1)/|k|^2."""
    torch = _torch()
    rng = np.random.default_rng(seed)
    coords = [nonuniform_coords(n, seed, a) for a, n in enumerate(dims)]
    xs = [torch.tensor(c, dtype=torch.float64, device=device) for c in coords]
    f = torch.zeros(tuple(dims), dtype=torch.float64, device=device)
    for _ in range(64):
        k = rng.integers(1, 17, size=2)
        a = rng.normal() / float(k[0] ** 2 + k[1] ** 2)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        arg = (2.0 * math.pi * k[0]) * xs[0][:, None] + (2.0 * math.pi * k[1]) * xs[1][None, :]
        f += a * torch.sin(arg + phi)
    return f.to(dtype or torch.float64), coords


def _grf2d(ny, nx, rng, torch, device):
    """2-D Gaussian random field with power ~ |k|^-3: white noise filtered by
    |k|^-1.5 in Fourier space."""
    white = torch.tensor(rng.normal(size=(ny, nx)), dtype=torch.float64, device=device)
    ky = torch.fft.fftfreq(ny, device=device, dtype=torch.float64)[:, None] * ny
    kx = torch.fft.fftfreq(nx, device=device, dtype=torch.float64)[None, :] * nx
    k = torch.sqrt(kx * kx + ky * ky)
    k[0, 0] = 1.0
    amp = k ** -1.5
    amp[0, 0] = 0.0
    g = torch.fft.ifft2(torch.fft.fft2(white) * amp).real
    return g / g.std()


def config4a_field(dims=(100, 500, 500), seed=0, device="cpu", dtype=None):
    """exp(-z/0.3) * (cos(theta_z) G_a + sin(theta_z) G_b), theta_z = pi z / 2."""
    torch = _torch()
    rng = np.random.default_rng(seed)
    nz, ny, nx = dims
    ga = _grf2d(ny, nx, rng, torch, device)
    gb = _grf2d(ny, nx, rng, torch, device)
    z = torch.linspace(0.0, 1.0, nz, dtype=torch.float64, device=device)
    th = (math.pi / 2.0) * z
    decay = torch.exp(-z / 0.3)
    f = decay[:, None, None] * (torch.cos(th)[:, None, None] * ga[None] + torch.sin(th)[:, None, None] * gb[None])
    return f.to(dtype or torch.float32)


def config4b_field(dims=(288, 115, 69, 69), seed=0, device="cpu", dtype=None, waves=32):
    """Sum of random sinusoids over the index lattice (the smooth_field recipe
    of the reference's tests, oracles.hpp:184-220, with numpy draws)."""
    torch = _torch()
    rng = np.random.default_rng(seed)
    d = len(dims)
    f = torch.zeros(tuple(dims), dtype=torch.float64, device=device)
    idx = [torch.arange(n, dtype=torch.float64, device=device) / float(n - 1) for n in dims]
    for _ in range(waves):
        amp = rng.uniform(0.2, 1.0)
        phi = rng.uniform(0.0, 2.0 * math.pi)
        ks = rng.uniform(0.5, 3.0, d)
        arg = None
        for i in range(d):
            shape = [1] * d
            shape[i] = dims[i]
            t = (ks[i] * 2.0 * math.pi) * idx[i].reshape(shape)
            arg = t if arg is None else arg + t
        f += amp * torch.sin(arg + phi)
    return f.to(dtype or torch.float32)
