"""ORACLE / TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.

ctypes bindings for
  * ``oracle/_build/libncsoracle.so`` -- the C restatement ``ncs_oracle.c``;
  * ``oracle/_ref/libncsref.so``      -- the reference's own sources compiled
    unchanged (oracle/Makefile).  Present only where it was built (this
    container builds it; the GPU box receives the prebuilt file).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libncsoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libncsref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def build(ref: bool | None = None) -> None:
    """Build the C restatement (and the reference library when its sources exist)."""
    targets = ["port"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets, "-j8"], check=True)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc == 4:
        raise OracleError(f"{what}: diverged")
    if rc != 0:
        raise OracleError(f"{what}: status {rc}")


@dataclass
class SolveOut:
    x: np.ndarray
    u: np.ndarray
    rows: np.ndarray  # (k, 5): iter, objective, rel_subopt, seminorm, wall_ms
    objective: float


class Port:
    """The C restatement (ncs_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_default_detector_count.restype = C.c_int
        for name in ("orc_radon_forward", "orc_radon_adjoint"):
            getattr(L, name).argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int]
        L.orc_radon_forward_rays.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int, _i64p, _dp,
                                             C.c_int]
        L.orc_radon_valid_counts.argtypes = [C.c_int, C.c_int, C.c_int, _i32p]
        L.orc_grad_forward.argtypes = [C.c_int, _dp, _dp]
        L.orc_grad_adjoint.argtypes = [C.c_int, _dp, _dp]
        L.orc_mask_apply.argtypes = [C.c_int, _dp, _dp, _dp]
        L.orc_pinv_mask.argtypes = [C.c_int, _dp, C.c_double, _dp]
        L.orc_laplacian_mask.argtypes = [C.c_int, _dp]
        L.orc_radon_mask.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.orc_calibrate_scale.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                          C.POINTER(C.c_double)]
        L.orc_make_phantom.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.orc_simulate_ct.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_double, C.c_uint64, _dp,
                                      C.c_int]
        L.orc_rng_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _dp]
        L.orc_screen.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                 C.c_double, C.c_int, _vp, C.c_double, _vp, C.c_int, C.c_uint64,
                                 C.c_int, C.POINTER(C.c_double)]
        L.orc_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.c_int, _vp, C.c_double, _vp, C.c_int, C.c_int, _vp,
                                _vp, _dp, _dp, _dp, C.c_int, C.POINTER(C.c_int),
                                C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
        L.orc_set_fan.argtypes = [C.c_double, C.c_double]
        L.orc_fan_defaults.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_fanbeam_triplets.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_int64, C.POINTER(C.c_int64), _vp, _vp, _vp]
        L.orc_fanbeam_apply.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_int, _dp, _dp, C.c_int]
        L.orc_fanbeam_empirical_mask.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                                 C.c_double, C.c_int, C.c_uint64, C.c_int, _dp,
                                                 C.POINTER(C.c_int)]
        L.orc_solve_ex.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_int, _vp, C.c_double, _vp, C.c_int, C.c_int,
                                   C.c_int, _vp, _vp, _dp, _dp, _dp, C.c_int, C.POINTER(C.c_int),
                                   C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
        L.orc_ncs_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_int, _vp, C.c_double, _vp, _dp, _dp, C.c_int,
                                   C.c_int]
        L.orc_objective.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_int, _vp, _dp, C.c_int,
                                    C.POINTER(C.c_double)]
        for name in ("orc_stacked_forward", "orc_stacked_adjoint"):
            getattr(L, name).argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_double, C.c_int, _dp, _dp, C.c_int]

    # -- operators -----------------------------------------------------
    def default_detector_count(self, n):
        return self.lib.orc_default_detector_count(n)

    # -- fan beam (fanbeam.cpp, sparse.cpp) ------------------------------
    def set_fan(self, radius, fan_angle):
        """Geometry of kind-3 (fan-beam CT-TV) problems."""
        self.lib.orc_set_fan(radius, fan_angle)

    def fan_defaults(self, n):
        r, f = C.c_double(), C.c_double()
        self.lib.orc_fan_defaults(n, C.byref(r), C.byref(f))
        return r.value, f.value

    def fanbeam_triplets(self, n, views, rays, radius, fan_angle):
        nnz = C.c_int64()
        _check(self.lib.orc_fanbeam_triplets(n, views, rays, radius, fan_angle, 0,
                                             C.byref(nnz), None, None, None), "fanbeam")
        k = nnz.value
        row, col, val = np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k)
        _check(self.lib.orc_fanbeam_triplets(n, views, rays, radius, fan_angle, k,
                                             C.byref(nnz), row.ctypes.data, col.ctypes.data,
                                             val.ctypes.data), "fanbeam")
        return row, col, val

    def fanbeam_empirical_mask(self, n, views, rays, radius, fan_angle, samples=8, seed=0,
                               threads=None):
        out = np.zeros((n, n), np.complex128)
        dead = C.c_int()
        _check(self.lib.orc_fanbeam_empirical_mask(n, views, rays, radius, fan_angle, samples,
                                                   seed, threads or default_threads(),
                                                   out.view(np.float64).ravel(),
                                                   C.byref(dead)), "empirical_mask")
        return out, dead.value

    def fanbeam_apply(self, n, views, rays, radius, fan_angle, v, adjoint=False, threads=None):
        v = np.ascontiguousarray(v, np.float64).ravel()
        out = np.zeros(n * n if adjoint else views * rays)
        _check(self.lib.orc_fanbeam_apply(n, views, rays, radius, fan_angle, int(adjoint), v,
                                          out, threads or default_threads()), "fanbeam_apply")
        return out

    def radon_forward(self, x, angles, det, threads=None):
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[-1]
        out = np.zeros((angles, det))
        _check(self.lib.orc_radon_forward(n, angles, det, x.ravel(), out.ravel(),
                                          threads or default_threads()), "radon_forward")
        return out

    def radon_forward_rays(self, x, angles, det, rays, threads=None):
        x = np.ascontiguousarray(x, np.float64)
        rays = np.ascontiguousarray(rays, np.int64)
        out = np.zeros(len(rays))
        _check(self.lib.orc_radon_forward_rays(x.shape[-1], angles, det, x.ravel(), len(rays),
                                               rays, out, threads or default_threads()),
               "radon_forward_rays")
        return out

    def radon_adjoint(self, u, n, threads=None):
        u = np.ascontiguousarray(u, np.float64)
        angles, det = u.shape
        out = np.zeros((n, n))
        _check(self.lib.orc_radon_adjoint(n, angles, det, u.ravel(), out.ravel(),
                                          threads or default_threads()), "radon_adjoint")
        return out

    def radon_valid_counts(self, n, angles, det):
        out = np.zeros(angles * det, np.int32)
        _check(self.lib.orc_radon_valid_counts(n, angles, det, out), "valid_counts")
        return out.reshape(angles, det)

    def grad_forward(self, x):
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[-1]
        out = np.zeros(2 * n * (n - 1))
        self.lib.orc_grad_forward(n, x.ravel(), out)
        return out

    def grad_adjoint(self, g, n):
        out = np.zeros((n, n))
        self.lib.orc_grad_adjoint(n, np.ascontiguousarray(g, np.float64).ravel(), out.ravel())
        return out

    def mask_apply(self, mask, x):
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[-1]
        h = np.ascontiguousarray(np.asarray(mask, np.complex128)).view(np.float64).ravel()
        out = np.zeros((n, n))
        self.lib.orc_mask_apply(n, h, x.ravel(), out.ravel())
        return out

    def pinv_mask(self, mask, rel_tol=1e-12):
        mask = np.ascontiguousarray(np.asarray(mask, np.complex128))
        out = np.zeros_like(mask)
        self.lib.orc_pinv_mask(mask.shape[0], mask.view(np.float64).ravel(), rel_tol,
                               out.view(np.float64).ravel())
        return out

    def laplacian_mask(self, n):
        out = np.zeros((n, n), np.complex128)
        self.lib.orc_laplacian_mask(n, out.view(np.float64).ravel())
        return out

    def radon_mask(self, n, scale, dc):
        out = np.zeros((n, n), np.complex128)
        self.lib.orc_radon_mask(n, scale, dc, out.view(np.float64).ravel())
        return out

    def calibrate_scale(self, n, angles, det, samples=8, seed=0, threads=None):
        r = C.c_double()
        _check(self.lib.orc_calibrate_scale(n, angles, det, samples, seed,
                                            threads or default_threads(), C.byref(r)),
               "calibrate_scale")
        return r.value

    def make_phantom(self, n, ellipses):
        e = np.ascontiguousarray(np.asarray(ellipses, np.float64).reshape(-1, 6))
        out = np.zeros((n, n))
        _check(self.lib.orc_make_phantom(n, len(e), e.ravel(), out.ravel()), "make_phantom")
        return out

    def simulate_ct(self, x, angles, det, sigma, seed, threads=None):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros((angles, det))
        _check(self.lib.orc_simulate_ct(x.shape[-1], angles, det, x.ravel(), sigma, seed,
                                        out.ravel(), threads or default_threads()), "simulate_ct")
        return out

    def rng_normals(self, seed, stream, count):
        out = np.zeros(count)
        self.lib.orc_rng_normals(seed, stream, count, out)
        return out

    # -- solver --------------------------------------------------------
    @staticmethod
    def _mask_arg(mask):
        if mask is None:
            return None, None
        h = np.ascontiguousarray(np.asarray(mask, np.complex128)).view(np.float64).ravel()
        return h, _ptr(h)

    def solve(self, prob, gamma, mask, max_iters, record_every=None, x0=None, u0=None,
              threads=None, pdhg=False, n_cg=0):
        """ncs_solve (pdhg=False, mask required) / pdhg_solve (mask=None) /
        admm_cg_solve (n_cg > 0, mask=None)."""
        p = prob
        if pdhg or n_cg:
            mask = None
        record_every = record_every or max(1, max_iters)
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        hk, hp = self._mask_arg(mask)
        x = np.zeros(p.n * p.n)
        u = np.zeros(p.range_size)
        max_rows = max_iters // record_every + 3
        rows = np.zeros((max_rows, 5))
        nr = C.c_int()
        obj = C.c_double()
        div = C.c_int64(-1)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64).ravel()
        u0a = None if u0 is None else np.ascontiguousarray(u0, np.float64).ravel()
        rc = self.lib.orc_solve_ex(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                                   int(p.positivity), _ptr(b), gamma, hp, n_cg, max_iters,
                                   record_every, _ptr(x0a), _ptr(u0a), x, u, rows.ravel(),
                                   max_rows, C.byref(nr), C.byref(obj), C.byref(div),
                                   threads or default_threads())
        if rc == 4:
            raise OracleError(f"diverged at iteration {div.value}")
        _check(rc, "solve")
        return SolveOut(x.reshape(p.n, p.n), u, rows[: nr.value].copy(), obj.value)

    def ncs_step(self, prob, gamma, mask, x, u, steps=1, threads=None):
        p = prob
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        hk, hp = self._mask_arg(mask)
        x = np.ascontiguousarray(x, np.float64).ravel().copy()
        u = np.ascontiguousarray(u, np.float64).ravel().copy()
        _check(self.lib.orc_ncs_step(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                                     int(p.positivity), _ptr(b), gamma, hp, x, u, steps,
                                     threads or default_threads()), "ncs_step")
        return x.reshape(p.n, p.n), u

    def objective(self, prob, x, threads=None):
        p = prob
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        f = C.c_double()
        self.lib.orc_objective(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                               int(p.positivity), _ptr(b),
                               np.ascontiguousarray(x, np.float64).ravel(),
                               threads or default_threads(), C.byref(f))
        return f.value

    def screen(self, prob, gamma, mask, iters=40, seed=0, threads=None):
        p = prob
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        hk, hp = self._mask_arg(mask)
        est = C.c_double()
        self.lib.orc_screen(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                            int(p.positivity), _ptr(b), gamma, hp, iters, seed,
                            threads or default_threads(), C.byref(est))
        return est.value

    def stacked_forward(self, prob, x, threads=None):
        p = prob
        out = np.zeros(p.range_size)
        self.lib.orc_stacked_forward(p.kind, p.n, p.angles, p.det, p.alpha, p.beta,
                                     int(p.positivity), np.ascontiguousarray(x, np.float64).ravel(),
                                     out, threads or default_threads())
        return out

    def stacked_adjoint(self, prob, u, threads=None):
        p = prob
        out = np.zeros((p.n, p.n))
        self.lib.orc_stacked_adjoint(p.kind, p.n, p.angles, p.det, p.alpha, p.beta,
                                     int(p.positivity), np.ascontiguousarray(u, np.float64).ravel(),
                                     out.ravel(), threads or default_threads())
        return out


class Ref:
    """The reference's own sources, compiled unchanged (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        for name in ("ref_radon_forward", "ref_radon_adjoint"):
            getattr(L, name).argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.ref_grad_forward.argtypes = [C.c_int, _dp, _dp]
        L.ref_grad_adjoint.argtypes = [C.c_int, _dp, _dp]
        L.ref_mask_apply.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_pinv_mask.argtypes = [C.c_int, _dp, C.c_double, _dp]
        L.ref_laplacian_mask.argtypes = [C.c_int, _dp]
        L.ref_radon_mask.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.ref_calibrate_scale.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                          C.POINTER(C.c_double)]
        L.ref_ct_metric_mask.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_double, C.c_int, C.c_uint64, C.c_int, _dp]
        L.ref_metric_mask.argtypes = [C.c_int, _dp, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_make_phantom.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.ref_simulate_ct.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_double, C.c_uint64,
                                      _dp]
        L.ref_rng_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _dp]
        L.ref_problem_sizes.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_int64)]
        L.ref_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.c_int, _dp, C.c_double, _vp, C.c_int, C.c_int,
                                C.c_int, _vp, _vp, C.c_int, _dp, _dp, _dp, C.c_int,
                                C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_ncs_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_int, _dp, C.c_double, _vp, _dp, _dp, C.c_int]
        L.ref_set_fan.argtypes = [C.c_double, C.c_double]
        L.ref_fan_defaults.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_fanbeam_triplets.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_int64, C.POINTER(C.c_int64), _vp, _vp, _vp]
        L.ref_fanbeam_apply.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_int, _dp, _dp]
        L.ref_fanbeam_empirical_mask.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                                 C.c_double, C.c_int, C.c_uint64, _dp,
                                                 C.POINTER(C.c_int)]
        L.ref_admm_cg_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_double, C.c_double, C.c_int, _dp, C.c_double,
                                        C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int,
                                        C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_objective.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_int, _dp, _dp, C.POINTER(C.c_double)]

    def _chk(self, rc, what):
        if rc != 0:
            raise OracleError(f"{what}: {self.lib.ref_last_error().decode()} (status {rc})")

    def radon_forward(self, x, angles, det):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros((angles, det))
        self._chk(self.lib.ref_radon_forward(x.shape[-1], angles, det, x.ravel(), out.ravel()),
                  "radon_forward")
        return out

    def radon_adjoint(self, u, n):
        u = np.ascontiguousarray(u, np.float64)
        out = np.zeros((n, n))
        self._chk(self.lib.ref_radon_adjoint(n, u.shape[0], u.shape[1], u.ravel(), out.ravel()),
                  "radon_adjoint")
        return out

    def grad_forward(self, x):
        x = np.ascontiguousarray(x, np.float64)
        n = x.shape[-1]
        out = np.zeros(2 * n * (n - 1))
        self._chk(self.lib.ref_grad_forward(n, x.ravel(), out), "grad_forward")
        return out

    def grad_adjoint(self, g, n):
        out = np.zeros((n, n))
        self._chk(self.lib.ref_grad_adjoint(n, np.ascontiguousarray(g, np.float64).ravel(),
                                            out.ravel()), "grad_adjoint")
        return out

    def mask_apply(self, mask, x):
        x = np.ascontiguousarray(x, np.float64)
        h = np.ascontiguousarray(np.asarray(mask, np.complex128)).view(np.float64).ravel()
        out = np.zeros_like(x)
        self._chk(self.lib.ref_mask_apply(x.shape[-1], h, x.ravel(), out.ravel()), "mask_apply")
        return out

    def pinv_mask(self, mask, rel_tol=1e-12):
        mask = np.ascontiguousarray(np.asarray(mask, np.complex128))
        out = np.zeros_like(mask)
        self._chk(self.lib.ref_pinv_mask(mask.shape[0], mask.view(np.float64).ravel(), rel_tol,
                                         out.view(np.float64).ravel()), "pinv_mask")
        return out

    def laplacian_mask(self, n):
        out = np.zeros((n, n), np.complex128)
        self._chk(self.lib.ref_laplacian_mask(n, out.view(np.float64).ravel()), "laplacian")
        return out

    def radon_mask(self, n, scale, dc):
        out = np.zeros((n, n), np.complex128)
        self._chk(self.lib.ref_radon_mask(n, scale, dc, out.view(np.float64).ravel()),
                  "radon_mask")
        return out

    def calibrate_scale(self, n, angles, det, samples=8, seed=0):
        r = C.c_double()
        self._chk(self.lib.ref_calibrate_scale(n, angles, det, samples, seed, C.byref(r)),
                  "calibrate_scale")
        return r.value

    def ct_metric_mask(self, n, angles, det, alpha, beta, dc, samples=8, seed=0,
                       positivity=False):
        out = np.zeros((n, n), np.complex128)
        self._chk(self.lib.ref_ct_metric_mask(n, angles, det, alpha, beta, dc, samples, seed,
                                              int(positivity), out.view(np.float64).ravel()),
                  "ct_metric_mask")
        return out

    def metric_mask(self, meas, alpha, beta, positivity=False):
        meas = np.ascontiguousarray(np.asarray(meas, np.complex128))
        out = np.zeros_like(meas)
        self._chk(self.lib.ref_metric_mask(meas.shape[0], meas.view(np.float64).ravel(), alpha,
                                           beta, int(positivity), out.view(np.float64).ravel()),
                  "metric_mask")
        return out

    def make_phantom(self, n, ellipses):
        e = np.ascontiguousarray(np.asarray(ellipses, np.float64).reshape(-1, 6))
        out = np.zeros((n, n))
        self._chk(self.lib.ref_make_phantom(n, len(e), e.ravel(), out.ravel()), "make_phantom")
        return out

    def simulate_ct(self, x, angles, det, sigma, seed):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros((angles, det))
        self._chk(self.lib.ref_simulate_ct(x.shape[-1], angles, det, x.ravel(), sigma, seed,
                                           out.ravel()), "simulate_ct")
        return out

    def rng_normals(self, seed, stream, count):
        out = np.zeros(count)
        self._chk(self.lib.ref_rng_normals(seed, stream, count, out), "rng")
        return out

    def solve(self, prob, gamma, mask, max_iters, record_every=None, x0=None, u0=None,
              check_step=False, pdhg=False):
        p = prob
        if pdhg:
            mask = None
        record_every = record_every or max(1, max_iters)
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        h = None if mask is None else np.ascontiguousarray(
            np.asarray(mask, np.complex128)).view(np.float64).ravel()
        x = np.zeros(p.n * p.n)
        u = np.zeros(p.range_size)
        max_rows = max_iters // record_every + 3
        rows = np.zeros((max_rows, 5))
        nr = C.c_int()
        obj = C.c_double()
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64).ravel()
        u0a = None if u0 is None else np.ascontiguousarray(u0, np.float64).ravel()
        self._chk(self.lib.ref_solve(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                                     int(p.positivity), b, gamma, _ptr(h), max_iters,
                                     record_every, int(check_step), _ptr(x0a), _ptr(u0a),
                                     int(pdhg), x, u, rows.ravel(), max_rows, C.byref(nr),
                                     C.byref(obj)), "solve")
        return SolveOut(x.reshape(p.n, p.n), u, rows[: nr.value].copy(), obj.value)

    def set_fan(self, radius, fan_angle):
        self.lib.ref_set_fan(radius, fan_angle)

    def fan_defaults(self, n):
        r, f = C.c_double(), C.c_double()
        self.lib.ref_fan_defaults(n, C.byref(r), C.byref(f))
        return r.value, f.value

    def fanbeam_triplets(self, n, views, rays, radius, fan_angle):
        nnz = C.c_int64()
        self._chk(self.lib.ref_fanbeam_triplets(n, views, rays, radius, fan_angle, 0,
                                                C.byref(nnz), None, None, None), "fanbeam")
        k = nnz.value
        row, col, val = np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k)
        self._chk(self.lib.ref_fanbeam_triplets(n, views, rays, radius, fan_angle, k,
                                                C.byref(nnz), row.ctypes.data, col.ctypes.data,
                                                val.ctypes.data), "fanbeam")
        return row, col, val

    def fanbeam_empirical_mask(self, n, views, rays, radius, fan_angle, samples=8, seed=0):
        out = np.zeros((n, n), np.complex128)
        dead = C.c_int()
        self._chk(self.lib.ref_fanbeam_empirical_mask(n, views, rays, radius, fan_angle,
                                                      samples, seed,
                                                      out.view(np.float64).ravel(),
                                                      C.byref(dead)), "empirical_mask")
        return out, dead.value

    def fanbeam_apply(self, n, views, rays, radius, fan_angle, v, adjoint=False):
        v = np.ascontiguousarray(v, np.float64).ravel()
        out = np.zeros(n * n if adjoint else views * rays)
        self._chk(self.lib.ref_fanbeam_apply(n, views, rays, radius, fan_angle, int(adjoint), v,
                                             out), "fanbeam_apply")
        return out

    def admm_cg_solve(self, prob, gamma, n_cg, max_iters, record_every=None):
        """admm_cg_solve (solvers.cpp:435-440) of the reference build."""
        p = prob
        record_every = record_every or max(1, max_iters)
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        x = np.zeros(p.n * p.n)
        u = np.zeros(p.range_size)
        max_rows = max_iters // record_every + 3
        rows = np.zeros((max_rows, 5))
        nr = C.c_int()
        obj = C.c_double()
        self._chk(self.lib.ref_admm_cg_solve(p.kind, p.n, p.angles, p.det, p.alpha, p.beta,
                                             p.lam, int(p.positivity), b, gamma, n_cg,
                                             max_iters, record_every, x, u, rows.ravel(),
                                             max_rows, C.byref(nr), C.byref(obj)),
                  "admm_cg_solve")
        return SolveOut(x.reshape(p.n, p.n), u, rows[: nr.value].copy(), obj.value)

    def ncs_step(self, prob, gamma, mask, x, u, steps=1):
        p = prob
        b = np.ascontiguousarray(p.b, np.float64).ravel()
        h = None if mask is None else np.ascontiguousarray(
            np.asarray(mask, np.complex128)).view(np.float64).ravel()
        x = np.ascontiguousarray(x, np.float64).ravel().copy()
        u = np.ascontiguousarray(u, np.float64).ravel().copy()
        self._chk(self.lib.ref_ncs_step(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                                        int(p.positivity), b, gamma, _ptr(h), x, u, steps),
                  "ncs_step")
        return x.reshape(p.n, p.n), u

    def objective(self, prob, x):
        p = prob
        f = C.c_double()
        self._chk(self.lib.ref_objective(p.kind, p.n, p.angles, p.det, p.alpha, p.beta, p.lam,
                                         int(p.positivity),
                                         np.ascontiguousarray(p.b, np.float64).ravel(),
                                         np.ascontiguousarray(x, np.float64).ravel(),
                                         C.byref(f)), "objective")
        return f.value


@dataclass
class Prob:
    """Problem description shared by oracle calls (kind 0 CT-TV, 1 TV-denoise)."""
    kind: int
    n: int
    angles: int
    det: int
    alpha: float
    beta: float
    lam: float
    b: np.ndarray
    positivity: bool = False

    @property
    def m0(self):
        return self.angles * self.det if self.kind != 1 else self.n * self.n

    @property
    def g(self):
        return 2 * self.n * (self.n - 1)

    @property
    def range_size(self):
        return self.m0 + self.g + (self.n * self.n if self.positivity else 0)
