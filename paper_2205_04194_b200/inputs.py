"""Seeded synthetic inputs of the BASELINE.json configs.

Both implementations (this library and the reference arm) consume the same
arrays; the SplitMix64 stream is the reference's random_vector
(reference.cpp:94-108), evaluated here in closed (counter) form.
"""
from __future__ import annotations

import math

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix_stream(seed: int, start: int, count: int) -> np.ndarray:
    """Values start..start+count-1 of random_vector(., seed) on [-1, 1)."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def random_vector(n: int, seed: int) -> np.ndarray:
    return splitmix_stream(seed, 0, n)


def uniform_points(n: int, seed: int = 0) -> np.ndarray:
    """(0.5 + 0.5 r[2i], 0.5 + 0.5 r[2i+1]), r = random_vector(2n, seed)."""
    return 0.5 + 0.5 * random_vector(2 * n, seed)


def gaussian_mixture(n: int, seed: int = 1, k: int = 8, sigma: float = 0.05) -> np.ndarray:
    """Config 3: k isotropic Gaussians, centres U[0.15,0.85]^2, point i from
    component i mod k, Box-Muller, rejection-clipped to [0,1]^2, one stream."""
    pos = 0
    c = 0.5 + 0.5 * splitmix_stream(seed, pos, 2 * k)
    pos += 2 * k
    cx = 0.15 + 0.7 * c[0::2]
    cy = 0.15 + 0.7 * c[1::2]
    out = np.empty(2 * n)
    i = 0
    chunk = 1 << 16
    while i < n:
        m = min(chunk, n - i)
        u = 0.5 + 0.5 * splitmix_stream(seed, pos, 2 * m)
        r = np.sqrt(-2.0 * np.log1p(-u[0::2]))
        th = 2.0 * math.pi * u[1::2]
        comp = (np.arange(i, i + m)) % k
        px = cx[comp] + sigma * r * np.cos(th)
        py = cy[comp] + sigma * r * np.sin(th)
        ok = (px >= 0.0) & (px <= 1.0) & (py >= 0.0) & (py <= 1.0)
        bad = np.flatnonzero(~ok)
        take = m if bad.size == 0 else int(bad[0])
        out[2 * i:2 * (i + take):2] = px[:take]
        out[2 * i + 1:2 * (i + take):2] = py[:take]
        i += take
        pos += 2 * take
        if take < m:  # attempt for point i rejected: consume its two values, redraw
            pos += 2
    return out


def cfg2_rhs(xy) -> np.ndarray:
    """f(x,y) = sin(2 pi x) cos(2 pi y) + 0.5 exp(-((x-.5)^2+(y-.5)^2)/0.02)."""
    x, y = xy[0::2], xy[1::2]
    return (np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
            + 0.5 * np.exp(-((x - 0.5) ** 2 + (y - 0.5) ** 2) / 0.02))


CONFIGS = {
    1: dict(n=4096, t=0.1, m=10, levels=2, points="uniform", seed=0),
    2: dict(n=65536, t=0.05, m=12, levels=0, points="uniform", seed=0),
    3: dict(n=1048576, t=0.02, m=14, levels=6, points="mixture", seed=1),
    4: dict(n=16777216, t=0.01, m=16, levels=8, points="uniform", seed=0),
    5: dict(n=4194304, t=None, m=None, levels=7, points="uniform", seed=0),
}


def config_points(cfg: int, n: int | None = None) -> np.ndarray:
    c = CONFIGS[cfg]
    n = n or c["n"]
    return uniform_points(n, c["seed"]) if c["points"] == "uniform" else gaussian_mixture(n, c["seed"])
