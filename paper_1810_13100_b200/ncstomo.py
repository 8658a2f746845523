"""GPU drop-in for the reference's Python module ``ncstomo``
(proj/python/bindings.cpp:180-336): the same names, arguments, defaults and
errors, with every operator application and solve on the B200 path
(``ncsg`` C ABI).  ``import paper_1810_13100_b200.ncstomo as ncstomo``.

* ``Geometry(kind, image_size, angles, detectors)`` -- "parallel"
  (RadonMap) or "fan" (build_fanbeam's SparseMap), ``forward``/``adjoint``
  (bindings.cpp:219-259, pipeline.cpp:40-51);
* ``simulate_ct`` / ``simulate_pet`` (phantom.cpp:53-90) -- GPU projection,
  host noise from the reference's per-bin RngStream rule;
* ``default_params`` (pipeline.cpp:54-67), ``measurement_mask``
  (pipeline.cpp:100-110: calibrate_scale for parallel beam, empirical_mask
  otherwise), ``make_phantom`` (phantom.cpp:29-51);
* ``reconstruct(...)`` (bindings.cpp:120-177) -> ``Result`` with image,
  objective, records (iter, objective, rel_subopt, seminorm_step, wall_ms),
  warnings (step-condition screen) and iters; solvers "ncs", "pdhg", "admm"
  (run_named_solver, pipeline.cpp:132-141).

Arithmetic is fp32 on the device (parity bar in DESIGN.md §4); the reference
is fp64 on the host.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import datagen, ncsg
from .instances import laplacian_mask, radon_mask

__version__ = "0.1.0+b200"
DivergenceError = ncsg.DivergenceError
RECORD_COLUMNS = ("iter", "objective", "rel_subopt", "seminorm_step", "wall_ms")


@dataclass
class Ellipse:
    """Ellipse(intensity, x0, y0, a, b, rot_deg) (phantom.hpp)."""
    intensity: float = 1.0
    x0: float = 0.0
    y0: float = 0.0
    a: float = 0.5
    b: float = 0.5
    rot_deg: float = 0.0


def make_phantom(n: int, ellipses) -> np.ndarray:
    """Additive ellipse indicators sampled at pixel centres (phantom.cpp:29-51)."""
    rows = [[e.intensity, e.x0, e.y0, e.a, e.b, e.rot_deg] if isinstance(e, Ellipse) else list(e)
            for e in ellipses]
    return datagen.make_phantom(n, np.asarray(rows, np.float64).reshape(-1, 6))


class Geometry:
    """Acquisition geometry (bindings.cpp:219-259; build_geometry, pipeline.cpp:40-51);
    detectors = 0 picks the default width."""

    def __init__(self, kind: str = "parallel", image_size: int = 0, angles: int = 60,
                 detectors: int = 0, device: int = 0):
        if kind not in ("parallel", "fan"):
            raise ValueError(f'unknown geometry kind "{kind}"')
        if image_size < 1 or angles < 1:
            raise ValueError("geometry sizes must be positive")
        det = detectors if detectors > 0 else ncsg.default_detector_count(image_size)
        self.kind, self.image_size = kind, image_size
        if kind == "parallel":
            self.map = ncsg.RadonMap(image_size, angles, det, device=device)
        else:
            self.map = ncsg.FanBeam(image_size, angles, det, device=device)

    @property
    def n_angles(self) -> int:
        return self.map.n_angles

    @property
    def n_detectors(self) -> int:
        return self.map.n_det

    def forward(self, image) -> np.ndarray:
        image = np.asarray(image, np.float64)
        if image.shape != (self.image_size, self.image_size):
            raise ValueError("image size does not match the geometry")
        return self.map.forward(image)

    def adjoint(self, sino) -> np.ndarray:
        sino = np.asarray(sino, np.float64)
        if sino.shape != (self.n_angles, self.n_detectors):
            raise ValueError("sinogram shape does not match the geometry")
        return self.map.adjoint(sino)

    def __repr__(self):
        return (f'Geometry(kind="{self.kind}", image_size={self.image_size}, '
                f"angles={self.n_angles}, detectors={self.n_detectors})")


def simulate_ct(image, geometry: Geometry, sigma: float = 0.0, seed: int = 0) -> np.ndarray:
    """Projection + sigma * RngStream(seed, i).next_normal() per bin (phantom.cpp:53-63)."""
    if sigma < 0.0:
        raise ValueError("sigma must be nonnegative")
    clean = geometry.forward(image)
    return clean + sigma * datagen.stream_noise(clean.shape, seed)


def _poisson(mean: float, s: datagen.Streams) -> int:
    """RngStream::next_poisson (rng.cpp:46-76): Knuth inversion below 30, PTRS above."""
    nd = lambda: float(s.next_double()[0])  # noqa: E731
    if mean < 30.0:
        limit, prod, k = math.exp(-mean), 1.0, 0
        while True:
            prod *= nd()
            if prod < limit:
                return k
            k += 1
    b = 0.931 + 2.53 * math.sqrt(mean)
    a = -0.059 + 0.02483 * b
    inv_alpha = 1.1239 + 1.1328 / (b - 3.4)
    v_r = 0.9277 - 3.6224 / (b - 2.0)
    while True:
        u = nd() - 0.5
        v = nd()
        us = 0.5 - abs(u)
        kf = math.floor((2.0 * a / us + b) * u + mean + 0.43)
        if us >= 0.07 and v <= v_r:
            return int(kf)
        if kf < 0.0 or (us < 0.013 and v > us):
            continue
        lhs = math.log(v * inv_alpha / (a / (us * us) + b))
        rhs = -mean + kf * math.log(mean) - math.lgamma(kf + 1.0)
        if lhs <= rhs:
            return int(kf)


def simulate_pet(image, geometry: Geometry, exposure_scale: float = 1.0,
                 seed: int = 0) -> np.ndarray:
    """Poisson counts with mean exposure_scale * projection (phantom.cpp:65-90);
    host sampling per bin (input generation, not the hot path)."""
    if exposure_scale <= 0.0:
        raise ValueError("exposure scale must be positive")
    clean = geometry.forward(image)
    peak = float(np.max(np.abs(clean))) if clean.size else 0.0
    out = np.zeros_like(clean)
    flat, res = clean.ravel(), out.ravel()
    for i in range(flat.size):
        mean = exposure_scale * flat[i]
        if mean < 0.0:
            if mean < -1e-12 * exposure_scale * max(1.0, peak):
                raise ValueError("negative projection mean in Poisson simulation")
            mean = 0.0
        if mean == 0.0:
            continue
        res[i] = _poisson(mean, datagen.Streams(seed, [i]))
    return out


def default_params(model: str = "ct") -> dict:
    """default_model_params (pipeline.cpp:54-67)."""
    p = {"model": model, "alpha": 1e-2, "beta": 1e-2, "gamma": 1.0, "lambda": 1.0, "dc": 1e-1,
         "positivity": False, "cg_iters": 10}
    if model == "ct":
        return p
    if model == "pet":
        p.update({"alpha": 1e-3, "beta": 1e-3, "gamma": 1e-4, "lambda": 1e-3, "dc": 1e-2})
        return p
    raise ValueError(f'unknown model "{model}"')


def measurement_mask(geometry: Geometry, dc: float = 1e-1, samples: int = 8,
                     seed: int = 0) -> np.ndarray:
    """Circulant surrogate of the measurement normal operator (pipeline.cpp:100-110)."""
    if samples < 1:
        raise ValueError("mask estimation needs samples >= 1")
    if geometry.kind == "parallel":
        scale = geometry.map.calibrate_scale(samples, seed)
        return radon_mask(geometry.image_size, scale, dc)
    return geometry.map.empirical_mask(samples, seed)[0]


def _metric_mask(meas: np.ndarray, p: dict) -> np.ndarray:
    """metric_mask (pipeline.cpp:112-118)."""
    w = p["beta"] / p["alpha"]
    mask = meas + (w * w) * laplacian_mask(meas.shape[0])
    if p["positivity"]:
        mask = mask + 1.0
    return mask


@dataclass
class Result:
    image: np.ndarray
    objective: float
    records: np.ndarray
    warnings: list = field(default_factory=list)
    iters: int = 0
    record_columns = RECORD_COLUMNS

    def __repr__(self):
        return f"Result(iters={self.iters}, objective={self.objective:.6f})"


def reconstruct(sino, geometry: Geometry, model: str = "ct", solver: str = "ncs",
                iters: int = 100, alpha=None, beta=None, gamma=None, lambda_=None, dc=None,
                positivity: bool = False, cg_iters=None, mask=None, mask_samples: int = 8,
                seed: int = 0, record_every: int = 1) -> Result:
    """reconstruct (bindings.cpp:120-177) on the GPU."""
    if iters < 0:
        raise ValueError("iters must be nonnegative")
    p = default_params(model)
    for k, v in (("alpha", alpha), ("beta", beta), ("gamma", gamma), ("lambda", lambda_),
                 ("dc", dc), ("cg_iters", cg_iters)):
        if v is not None:
            p[k] = v
    p["positivity"] = bool(positivity)
    sino = np.asarray(sino, np.float64)
    if sino.shape != (geometry.n_angles, geometry.n_detectors):
        raise ValueError("sinogram shape does not match the geometry")
    metric = None
    if mask is not None:
        if solver != "ncs":
            raise ValueError("mask only applies to the ncs solver")
        if isinstance(mask, str):
            if mask != "auto":
                raise ValueError('mask must be None, "auto", or a complex array')
            meas = measurement_mask(geometry, p["dc"], mask_samples, seed)
        else:
            meas = np.asarray(mask, np.complex128)
            if meas.shape != (geometry.image_size, geometry.image_size):
                raise ValueError("mask size does not match the geometry")
        metric = _metric_mask(meas, p)
    if solver not in ("ncs", "pdhg", "admm"):
        raise ValueError(f'unknown solver "{solver}"')
    if p["alpha"] <= 0.0 or p["beta"] <= 0.0:
        raise ValueError("alpha and beta must be positive")
    kind = ncsg.PET if model == "pet" else ncsg.CT
    if model not in ("ct", "pet"):
        raise ValueError(f'unknown model "{model}"')
    use_mask = metric if solver == "ncs" else None
    g = p["gamma"] if (solver != "admm" or p["gamma"] > 0.0) else 1.0
    sparse = geometry.map if geometry.kind == "fan" else None
    prob = ncsg.Problem(kind, geometry.image_size, p["alpha"], p["beta"], p["lambda"], g, sino,
                        mask=use_mask, n_angles=geometry.n_angles, n_det=geometry.n_detectors,
                        positivity=p["positivity"], sparse=sparse)
    if solver == "admm":
        prob.set_cg(int(p["cg_iters"]))
    prob.set_state()
    check = solver != "admm"  # the screen returns early in Cg mode (solvers.cpp:207)
    res = prob.solve(iters, record_every=record_every, check_step_condition=check, seed=seed)
    warnings = []
    if check and np.isfinite(res.screen_est):
        shift = p["gamma"] + (p["alpha"] * float(np.max(np.abs(use_mask))) if use_mask is not None
                              else 0.0)
        if res.screen_est > 1e-8 * max(1.0, shift):
            warnings.append("step condition M >= alpha A^T A appears violated (largest "
                            f"eigenvalue of alpha A^T A - M is about {res.screen_est:g})")
    return Result(image=res.x[0].reshape(geometry.image_size, geometry.image_size),
                  objective=float(res.objective[0]), records=res.rows[0], warnings=warnings,
                  iters=iters)
