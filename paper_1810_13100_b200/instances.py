"""Problem instances (x_true, b) and circulant masks for the pinned configs.

Host-side setup only: the masks follow the reference formulas
``radon_mask`` / ``laplacian_mask_2d`` / ``metric_mask`` (circulant.cpp:57-84,
pipeline.cpp:112-118); the projection used to synthesise ``b`` is passed in
(the GPU forward in bench.py, the oracle in tests).
"""
from __future__ import annotations

import math

import numpy as np

from . import datagen
from .configs import Config


def laplacian_mask(n: int) -> np.ndarray:
    """4 (sin^2(pi j/N) + sin^2(pi k/N)) (circulant.cpp:57-68)."""
    s2 = np.array([math.sin(math.pi * j / n) ** 2 for j in range(n)])
    return (4.0 * (s2[:, None] + s2[None, :])).astype(np.complex128)


def radon_mask(n: int, scale: float, dc: float) -> np.ndarray:
    """scale / sqrt(m_j^2 + m_k^2), DC pinned to dc (circulant.cpp:70-84)."""
    j = np.arange(n, dtype=np.float64)
    mj = np.minimum(j, n - j)
    r = np.sqrt(mj[:, None] * mj[:, None] + mj[None, :] * mj[None, :])
    with np.errstate(divide="ignore"):
        h = scale / r
    h[0, 0] = dc
    return h.astype(np.complex128)


def metric_mask(cfg: Config, positivity: bool = False) -> np.ndarray:
    """measurement mask + (beta/alpha)^2 Laplacian (+1 with positivity)
    (pipeline.cpp:112-118).  The TV-denoise data block is the identity, whose
    circulant part is exactly 1."""
    if cfg.kind == "ct":
        meas = radon_mask(cfg.n, cfg.mask_scale, cfg.dc)
    else:
        meas = np.ones((cfg.n, cfg.n), np.complex128)
    w = cfg.beta / cfg.alpha
    mask = meas + (w * w) * laplacian_mask(cfg.n)
    if positivity:
        mask = mask + 1.0
    return mask


def make_instance(cfg: Config, forward=None, problem: int = 0):
    """(x_true, b) for problem ``problem`` of ``cfg``; ``forward(x)`` must
    return R x (float64 angles x det) for CT configs."""
    x = datagen.phantom(cfg.n, cfg.ellipses, cfg.phantom_seed + problem)
    if cfg.kind == "ct":
        clean = np.asarray(forward(x), dtype=np.float64).reshape(cfg.angles, cfg.det)
        b, _ = datagen.add_sinogram_noise(clean, cfg.noise_frac, cfg.noise_seed + problem)
    else:
        b = x + cfg.image_sigma * datagen.stream_noise(x.shape, cfg.noise_seed + problem)
    return x, b
