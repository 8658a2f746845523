"""Seeded synthetic inputs for the five BASELINE.json configs.

The reference ships no benchmark data (its paper's Mayo/XCAT/PET sets are out
of scope), so these generators stand in for it with the shapes and
value distributions BASELINE.json states:

* random-ellipse phantoms: K ellipses, each drawn from its own counter-based
  stream ``RngStream(seed, e)`` (the reference RNG, rng.cpp:9-45): centre
  uniform in the inner 80 % of the image, semi-axes 5-40 px, rotation uniform,
  additive intensity U[0,1]; rasterised exactly as ``make_phantom``
  (phantom.cpp:29-51) does, then clipped to [0,1];
* sinogram noise ``b_i = (R x)_i + sigma * RngStream(seed, i).next_normal()``
  (``simulate_ct``, phantom.cpp:53-63) with ``sigma = frac * max(R x)``;
* image noise for TV denoising with the same per-element stream rule.

Everything here is host-side numpy: input generation, not the hot path.
"""
from __future__ import annotations

import math

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (rng.cpp:9-14), vectorised over uint64 arrays."""
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


class Streams:
    """A batch of ``RngStream(seed, id)`` (rng.cpp:16-45) advanced in lock step."""

    def __init__(self, seed: int, ids):
        ids = np.asarray(ids, dtype=np.uint64)
        with np.errstate(over="ignore"):
            self.state = _mix(_mix(np.array([seed], dtype=np.uint64)) + ids)

    def next_u64(self) -> np.ndarray:
        with np.errstate(over="ignore"):
            self.state = self.state + _GOLD
            z = self.state
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            return z ^ (z >> np.uint64(31))

    def next_double(self) -> np.ndarray:
        bits = self.next_u64() >> np.uint64(11)
        bits = np.where(bits == 0, np.uint64(1), bits)
        return bits.astype(np.float64) * 2.0 ** -53

    def first_normal(self) -> np.ndarray:
        """The first ``next_normal()`` of every stream (Box-Muller cosine branch)."""
        u1 = self.next_double()
        u2 = self.next_double()
        r = np.sqrt(-2.0 * np.log(u1))
        return r * np.cos(2.0 * math.pi * u2)


def normals(seed: int, stream: int, count: int) -> np.ndarray:
    """``count`` successive normals of one stream (pairs cached, rng.cpp:33-45)."""
    s = Streams(seed, [stream])
    out = np.empty(count)
    i = 0
    while i < count:
        u1 = s.next_double()[0]
        u2 = s.next_double()[0]
        r = math.sqrt(-2.0 * math.log(u1))
        t = 2.0 * math.pi * u2
        out[i] = r * math.cos(t)
        if i + 1 < count:
            out[i + 1] = r * math.sin(t)
        i += 2
    return out


def random_ellipses(n: int, count: int, seed: int) -> np.ndarray:
    """(count, 6) rows {intensity, x0, y0, a, b, rot_deg} in make_phantom's
    [-1,1]^2 frame (phantom.hpp:11-18); one pixel is 2/N."""
    s = Streams(seed, np.arange(count))
    u = np.stack([s.next_double() for _ in range(6)], axis=1)
    cx = n * (0.1 + 0.8 * u[:, 0])
    cy = n * (0.1 + 0.8 * u[:, 1])
    a_px = 5.0 + 35.0 * u[:, 2]
    b_px = 5.0 + 35.0 * u[:, 3]
    rot = 180.0 * u[:, 4]
    inten = u[:, 5]
    x0 = (2.0 * cx - (n - 1)) / n
    y0 = ((n - 1) - 2.0 * cy) / n
    return np.stack([inten, x0, y0, 2.0 * a_px / n, 2.0 * b_px / n, rot], axis=1)


def make_phantom(n: int, ellipses: np.ndarray) -> np.ndarray:
    """Indicator rasterisation at pixel centres, ellipses add (phantom.cpp:29-51)."""
    img = np.zeros((n, n))
    i = np.arange(n, dtype=np.float64)
    v = ((n - 1.0) - 2.0 * i) / n  # row coordinate
    u = (2.0 * i - (n - 1.0)) / n  # column coordinate
    for inten, x0, y0, a, b, rot in np.asarray(ellipses, np.float64).reshape(-1, 6):
        if a <= 0.0 or b <= 0.0:
            raise ValueError("ellipse semi-axes must be positive")
        phi = rot * math.pi / 180.0
        c, s = math.cos(phi), math.sin(phi)
        du = u[None, :] - x0
        dv = v[:, None] - y0
        xi = (c * du + s * dv) / a
        eta = (-s * du + c * dv) / b
        img[xi * xi + eta * eta <= 1.0] += inten
    return img


def phantom(n: int, count: int, seed: int) -> np.ndarray:
    """Seeded random-ellipse phantom clipped to [0, 1] (BASELINE.json configs)."""
    return np.clip(make_phantom(n, random_ellipses(n, count, seed)), 0.0, 1.0)


def stream_noise(shape, seed: int) -> np.ndarray:
    """Element i gets the first normal of RngStream(seed, i) (phantom.cpp:57-61)."""
    total = int(np.prod(shape))
    out = np.empty(total)
    step = 1 << 22
    for lo in range(0, total, step):
        hi = min(total, lo + step)
        out[lo:hi] = Streams(seed, np.arange(lo, hi)).first_normal()
    return out.reshape(shape)


def add_sinogram_noise(clean: np.ndarray, frac: float, seed: int) -> tuple[np.ndarray, float]:
    """simulate_ct noise with sigma = frac * max(R x) (tools/main.cpp:186-193)."""
    sigma = frac * float(np.max(clean))
    return clean + sigma * stream_noise(clean.shape, seed), sigma
