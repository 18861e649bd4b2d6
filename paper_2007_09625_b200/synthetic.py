"""Deterministic synthetic fields (reference: sdqz/synthetic.py:16-88).

Test/bench data source only (SURVEY.md §2a marks it out of the hot path).
The random draws happen in the reference's order, so a given (profile,
dims, seed, value) yields the reference's field.  `smooth_rows` evaluates a
row range of axis 0 of the smooth profile (slab-wise generation of fields too
large for host memory, e.g. the 2048x2048x1024 config).
"""

from __future__ import annotations

import math

import numpy as np

from .core import SdqzError

PROFILES = ("smooth", "ramp", "sparse-near-zero", "constant", "gaussian-noise")
_TWO_PI = 2.0 * math.pi


def _grid(dims):
    return list(np.ix_(*(np.arange(d, dtype=np.float64) / d for d in dims)))


def smooth_params(seed: int, rank: int):
    """(amp, phase, [freq per axis]) for the 6 waves of the smooth profile."""
    rng = np.random.default_rng(seed)
    waves = []
    for _ in range(6):
        amp = rng.uniform(0.5, 1.0)
        phase = rng.uniform(0.0, _TWO_PI)
        freqs = [rng.uniform(1.0, 4.0) for _ in range(rank)]
        waves.append((amp, phase, freqs))
    return waves


def smooth_rows(dims, seed: int, rows=None) -> np.ndarray:
    """Smooth profile over rows [r0, r1) of axis 0 (whole field if rows is None)."""
    dims = tuple(int(d) for d in dims)
    grid = _grid(dims)
    if rows is not None:
        grid[0] = grid[0][rows[0]:rows[1]]
    shape = tuple(g.shape[i] for i, g in enumerate(grid))
    out = np.zeros(shape)
    for amp, phase, freqs in smooth_params(seed, len(dims)):
        arg = phase
        for f, t in zip(freqs, grid):
            arg = arg + f * 2.0 * math.pi * t
        out += amp * np.sin(arg)
    return out


def _ramp(rng, dims):
    out = rng.uniform(-0.5, 0.5) * np.ones(dims)
    for t in _grid(dims):
        out = out + rng.uniform(0.5, 1.5) * t
    return out


def _sparse(rng, dims):
    grid = _grid(dims)
    acc = np.zeros(dims)
    for _ in range(8):
        centre = [rng.uniform(0.0, 1.0) for _ in dims]
        width = rng.uniform(0.04, 0.12)
        r2 = np.zeros(dims)
        for t, c in zip(grid, centre):
            d = np.abs(t - c)
            d = np.minimum(d, 1.0 - d)
            r2 = r2 + d * d
        acc += rng.uniform(0.5, 1.0) * np.exp(-r2 / (2.0 * width * width))
    floor = np.quantile(acc, 0.90)
    out = np.maximum(acc - floor, 0.0)
    return out / out.max()


def generate_field(profile: str, dims, seed: int = 0, value: float = 0.0) -> np.ndarray:
    """One shaped float64 field; identical arguments give identical values."""
    dims = tuple(int(d) for d in dims)
    if any(d < 1 for d in dims) or not 1 <= len(dims) <= 3:
        raise SdqzError(f"profile fields are rank 1-3 with positive extents, got {dims}")
    if profile == "smooth":
        return smooth_rows(dims, seed)
    rng = np.random.default_rng(seed)
    if profile == "ramp":
        return _ramp(rng, dims)
    if profile == "sparse-near-zero":
        return _sparse(rng, dims)
    if profile == "constant":
        return np.full(dims, float(value))
    if profile == "gaussian-noise":
        return rng.normal(0.0, 1.0, size=dims)
    raise SdqzError(f"unknown profile {profile!r}; choose from {', '.join(PROFILES)}")


def smooth_field_device(dims, seed: int = 1, rows=None, device=None, dtype=None):
    """The smooth profile evaluated on the GPU in fp64 (same parameters as
    `smooth_rows`; values agree to ~1 ulp, not bitwise -- bench data only)."""
    import torch
    dims = tuple(int(d) for d in dims)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    r0, r1 = rows if rows is not None else (0, dims[0])
    axes = []
    for a, d in enumerate(dims):
        t = torch.arange(d, dtype=torch.float64, device=dev) / d
        if a == 0:
            t = t[r0:r1]
        shape = [1] * len(dims)
        shape[a] = t.numel()
        axes.append(t.view(shape))
    shape = tuple(ax.shape[a] for a, ax in enumerate(axes))
    out = torch.zeros(shape, dtype=torch.float64, device=dev)
    for amp, phase, freqs in smooth_params(seed, len(dims)):
        arg = torch.full((1,) * len(dims), phase, dtype=torch.float64, device=dev)
        for f, t in zip(freqs, axes):
            arg = arg + (f * 2.0 * math.pi) * t
        out += amp * torch.sin(arg)
    return out.to(dtype) if dtype is not None else out
