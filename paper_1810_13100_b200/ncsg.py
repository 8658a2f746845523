"""Python view of the C ABI (include/ncsg.h) with the reference's names.

Mirrors the operator / solver surface of the reference's pybind module and C++
API (proj/python/bindings.cpp, proj/include/ncstomo/*.hpp) for the NCS hot
path: ``RadonMap``, ``GradMap``, ``mask_apply`` (MaskApplier::apply),
``SplitProblem`` + ``ncs_solve`` / ``pdhg_solve`` / ``ncs_step``.  Every call
goes through ``libncsg.so``; there is no CPU fallback -- on a machine without
a CUDA device the compute calls raise ``NcsgError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _build

_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class NcsgError(RuntimeError):
    """Failure reported by libncsg (status != NCSG_OK)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class DivergenceError(NcsgError):
    """Mirrors ncstomo::DivergenceError (solvers.hpp:101-105)."""

    def __init__(self, status, msg, iter_=None):
        super().__init__(status, msg)
        self.iter = iter_


class PlanInfo(C.Structure):
    """ncsg_plan_info: the live plan of a problem (include/ncsg.h)."""
    _fields_ = [("orbit_forward", C.c_int), ("gather_adjoint", C.c_int), ("fp_slots", C.c_int),
                ("bp_partials", C.c_int), ("n_orbits", C.c_int), ("transposed_copy", C.c_int),
                ("samples", C.c_int64), ("m0", C.c_int64), ("g", C.c_int64),
                ("range", C.c_int64), ("batch", C.c_int64), ("dual_fused", C.c_int),
                ("adjoint_table_bytes", C.c_int64)]


XCHG_ALLREDUCE, XCHG_SLAB, XCHG_P2P = 0, 1, 2
F32, F64, I32 = 0, 1, 2
SUM, MIN, MAX = 0, 1, 2
_AllReduceFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int,
                           C.c_void_p)
_XferFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class CommOps(C.Structure):
    """ncsg_comm_ops: the callback transport (include/ncsg.h)."""
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int), ("nranks", C.c_int),
                ("all_reduce", _AllReduceFn), ("reduce_scatter", _XferFn),
                ("all_gather", _XferFn), ("all_to_all", _XferFn)]


class ProblemDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n", C.c_int), ("n_angles", C.c_int), ("n_det", C.c_int),
        ("batch", C.c_int), ("positivity", C.c_int), ("alpha", C.c_double),
        ("beta", C.c_double), ("lambda_", C.c_double), ("gamma", C.c_double),
        ("pinv_rel_tol", C.c_double), ("mask", C.c_void_p), ("b", C.c_void_p),
        ("angle_begin", C.c_int), ("angle_end", C.c_int), ("device", C.c_int),
        ("sparse", C.c_void_p), ("shard_rank", C.c_int), ("shard_count", C.c_int),
        ("m_pinv", C.c_void_p), ("m_symbol", C.c_void_p),
    ]


class RecordRow(C.Structure):
    _fields_ = [("iter", C.c_int64), ("objective", C.c_double), ("rel_subopt", C.c_double),
                ("seminorm_step", C.c_double), ("wall_ms", C.c_double)]


SYMBOLS = [
    "ncsg_last_error", "ncsg_version", "ncsg_device_count", "ncsg_default_detector_count",
    "ncsg_radon_create", "ncsg_radon_destroy", "ncsg_radon_domain_size",
    "ncsg_radon_range_size", "ncsg_radon_sample_count", "ncsg_radon_forward",
    "ncsg_radon_adjoint", "ncsg_radon_forward_host", "ncsg_radon_adjoint_host",
    "ncsg_grad_forward", "ncsg_grad_adjoint", "ncsg_grad_forward_host",
    "ncsg_grad_adjoint_host", "ncsg_mask_apply_host", "ncsg_problem_create",
    "ncsg_problem_destroy", "ncsg_problem_domain_size", "ncsg_problem_range_size",
    "ncsg_problem_stream", "ncsg_set_state", "ncsg_get_state", "ncsg_state_x", "ncsg_state_u",
    "ncsg_step", "ncsg_step_graph", "ncsg_sync", "ncsg_objective", "ncsg_last_seminorm",
    "ncsg_solve", "ncsg_step_phase_a", "ncsg_atu_buffer", "ncsg_step_phase_b",
    "ncsg_profile_begin", "ncsg_profile_end", "ncsg_launch_count", "ncsg_set_atu_buffer",
    "ncsg_calibrate_scale", "ncsg_radon_dc_response", "ncsg_screen_step_condition",
    "ncsg_set_cg", "ncsg_fanbeam_create", "ncsg_fan_defaults", "ncsg_sparse_create",
    "ncsg_sparse_destroy", "ncsg_sparse_nnz", "ncsg_sparse_forward", "ncsg_sparse_adjoint",
    "ncsg_sparse_forward_host", "ncsg_sparse_adjoint_host", "ncsg_sparse_empirical_mask",
]
PHASES = ["adjoint", "fft_rows_r2c", "fft_cols", "fft_rows_c2r", "make_quad", "forward",
          "dual_update"]


def lib():
    """Load libncsg.so (building it in-tree if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("NCSG_LIB")  # experiment builds (scripts/build_variant.py)
    if not path:
        path = _build.LIB
        if not os.path.exists(path):
            _build.build()
    L = C.CDLL(path)
    L.ncsg_last_error.restype = C.c_char_p
    L.ncsg_version.restype = C.c_char_p
    for name in ("ncsg_radon_domain_size", "ncsg_radon_range_size", "ncsg_problem_domain_size",
                 "ncsg_problem_range_size"):
        getattr(L, name).restype = C.c_size_t
        getattr(L, name).argtypes = [C.c_void_p]
    L.ncsg_radon_sample_count.restype = C.c_int64
    L.ncsg_radon_sample_count.argtypes = [C.c_void_p]
    L.ncsg_radon_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.ncsg_radon_destroy.argtypes = [C.c_void_p]
    for name in ("ncsg_radon_forward", "ncsg_radon_adjoint"):
        getattr(L, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    for name in ("ncsg_radon_forward_host", "ncsg_radon_adjoint_host"):
        getattr(L, name).argtypes = [C.c_void_p, _dp, _dp, C.c_int]
    for name in ("ncsg_grad_forward", "ncsg_grad_adjoint"):
        getattr(L, name).argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    for name in ("ncsg_grad_forward_host", "ncsg_grad_adjoint_host"):
        getattr(L, name).argtypes = [C.c_int, _dp, _dp, C.c_int]
    L.ncsg_mask_apply_host.argtypes = [C.c_int, _dp, _dp, _dp, C.c_int, C.c_int]
    L.ncsg_problem_create.argtypes = [C.POINTER(ProblemDesc), C.POINTER(C.c_void_p)]
    L.ncsg_problem_destroy.argtypes = [C.c_void_p]
    L.ncsg_problem_stream.restype = C.c_void_p
    L.ncsg_problem_stream.argtypes = [C.c_void_p]
    L.ncsg_set_state.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
    L.ncsg_get_state.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    for name in ("ncsg_state_x", "ncsg_state_u", "ncsg_atu_buffer"):
        getattr(L, name).restype = C.c_void_p
        getattr(L, name).argtypes = [C.c_void_p]
    for name in ("ncsg_step", "ncsg_step_graph"):
        getattr(L, name).argtypes = [C.c_void_p, C.c_int]
    L.ncsg_sync.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.ncsg_objective.argtypes = [C.c_void_p, _dp]
    L.ncsg_last_seminorm.argtypes = [C.c_void_p, _dp]
    L.ncsg_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p,
                             C.POINTER(RecordRow), C.c_int, C.POINTER(C.c_int),
                             C.POINTER(C.c_double)]
    L.ncsg_set_cg.argtypes = [C.c_void_p, C.c_int]
    L.ncsg_fanbeam_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                      C.POINTER(C.c_void_p)]
    L.ncsg_fan_defaults.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ncsg_sparse_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
    L.ncsg_sparse_destroy.argtypes = [C.c_void_p]
    L.ncsg_sparse_empirical_mask.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _dp,
                                             C.POINTER(C.c_int)]
    L.ncsg_sparse_nnz.restype = C.c_int64
    L.ncsg_sparse_nnz.argtypes = [C.c_void_p]
    for name in ("ncsg_sparse_forward", "ncsg_sparse_adjoint"):
        getattr(L, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    for name in ("ncsg_sparse_forward_host", "ncsg_sparse_adjoint_host"):
        getattr(L, name).argtypes = [C.c_void_p, _dp, _dp, C.c_int]
    L.ncsg_calibrate_scale.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.POINTER(C.c_double)]
    L.ncsg_radon_dc_response.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.ncsg_screen_step_condition.argtypes = [C.c_void_p, C.c_uint64, C.c_int,
                                             C.POINTER(C.c_double), C.POINTER(C.c_double)]
    for name in ("ncsg_step_phase_a", "ncsg_step_phase_b", "ncsg_profile_begin"):
        getattr(L, name).argtypes = [C.c_void_p]
    L.ncsg_set_atu_buffer.argtypes = [C.c_void_p, C.c_void_p]
    L.ncsg_profile_end.argtypes = [C.c_void_p, _dp, C.c_int, C.POINTER(C.c_int)]
    L.ncsg_launch_count.restype = C.c_int64
    L.ncsg_problem_plan.argtypes = [C.c_void_p, C.POINTER(PlanInfo)]
    L.ncsg_nccl_unique_id.argtypes = [C.c_char_p]
    L.ncsg_comm_create_nccl.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]
    L.ncsg_comm_create_callbacks.argtypes = [C.POINTER(CommOps), C.POINTER(C.c_void_p)]
    L.ncsg_comm_create_local.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.ncsg_comm_destroy.argtypes = [C.c_void_p]
    L.ncsg_comm_create_null.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.ncsg_problem_set_comm.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    _lib = L
    return L


def _check(status: int, what: str = ""):
    if status == 0:
        return
    msg = lib().ncsg_last_error().decode()
    if status == 4:
        raise DivergenceError(status, msg)
    if status == 2:
        raise ValueError(msg)
    raise NcsgError(status, f"{what}: {msg}" if what else msg)


def launch_count() -> int:
    return lib().ncsg_launch_count()


def device_count() -> int:
    return lib().ncsg_device_count()


def default_detector_count(n: int) -> int:
    return lib().ncsg_default_detector_count(n)


class RadonMap:
    """RadonMap(n, n_angles, n_det) (radon.hpp:16-36) on the GPU."""

    def __init__(self, n: int, n_angles: int, n_det: int | None = None, device: int = 0):
        if n_det is None:
            n_det = default_detector_count(n)
        h = C.c_void_p()
        _check(lib().ncsg_radon_create(n, n_angles, n_det, device, C.byref(h)), "RadonMap")
        self._h = h
        self.n, self.n_angles, self.n_det = n, n_angles, n_det

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ncsg_radon_destroy(self._h)
            self._h = None

    def domain_size(self):
        return lib().ncsg_radon_domain_size(self._h)

    def range_size(self):
        return lib().ncsg_radon_range_size(self._h)

    def sample_count(self):
        return lib().ncsg_radon_sample_count(self._h)

    def forward(self, x) -> np.ndarray:
        """fp64 host in/out (RadonMap::forward, radon.cpp:82-102)."""
        x = np.ascontiguousarray(x, np.float64)
        batch = x.size // (self.n * self.n)
        out = np.zeros((batch, self.n_angles, self.n_det))
        _check(lib().ncsg_radon_forward_host(self._h, x.ravel(), out.ravel(), batch), "forward")
        return out.reshape(x.shape[:-2] + (self.n_angles, self.n_det))

    def adjoint(self, u) -> np.ndarray:
        """fp64 host in/out (RadonMap::adjoint, radon.cpp:104-127)."""
        u = np.ascontiguousarray(u, np.float64)
        batch = u.size // (self.n_angles * self.n_det)
        out = np.zeros((batch, self.n, self.n))
        _check(lib().ncsg_radon_adjoint_host(self._h, u.ravel(), out.ravel(), batch), "adjoint")
        return out.reshape(u.shape[:-2] + (self.n, self.n))

    def calibrate_scale(self, n_samples: int = 8, seed: int = 0) -> float:
        """calibrate_scale(NormalMap(R), radon_mask(n, 1, 1), n_samples, seed)
        (circulant.cpp:142-169) on the GPU."""
        out = C.c_double()
        _check(lib().ncsg_calibrate_scale(self._h, n_samples, seed, C.byref(out)),
               "calibrate_scale")
        return out.value

    def dc_response(self) -> float:
        """<1, R^T R 1> / n^2 (the dc rule of the pinned configs)."""
        out = C.c_double()
        _check(lib().ncsg_radon_dc_response(self._h, C.byref(out)), "dc_response")
        return out.value

    def measurement_mask(self, samples: int = 8, seed: int = 0, dc: float | None = None):
        """measurement_mask for parallel-beam geometry (pipeline.cpp:100-110):
        radon_mask(n, calibrate_scale(...), dc) as an (n, n) complex array."""
        from .instances import radon_mask

        scale = self.calibrate_scale(samples, seed)
        if dc is None:
            dc = self.dc_response()
        return radon_mask(self.n, scale, dc)

    def forward_device(self, x_ptr: int, out_ptr: int, batch: int = 1, stream=None):
        _check(lib().ncsg_radon_forward(self._h, x_ptr, out_ptr, batch, stream), "forward")

    def adjoint_device(self, u_ptr: int, out_ptr: int, batch: int = 1, stream=None):
        _check(lib().ncsg_radon_adjoint(self._h, u_ptr, out_ptr, batch, stream), "adjoint")


class GradMap:
    """GradMap(n) (grad.hpp:17-28): flat range = h block then v block."""

    def __init__(self, n: int):
        if n < 2:
            raise ValueError("grad needs N >= 2")
        self.n = n

    def domain_size(self):
        return self.n * self.n

    def range_size(self):
        return 2 * self.n * (self.n - 1)

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float64)
        batch = x.size // (self.n * self.n)
        out = np.zeros((batch, self.range_size()))
        _check(lib().ncsg_grad_forward_host(self.n, x.ravel(), out.ravel(), batch),
               "grad forward")
        return out[0] if batch == 1 else out

    def adjoint(self, g):
        g = np.ascontiguousarray(g, np.float64)
        batch = g.size // self.range_size()
        out = np.zeros((batch, self.n, self.n))
        _check(lib().ncsg_grad_adjoint_host(self.n, g.ravel(), out.ravel(), batch), "grad adjoint")
        return out[0] if batch == 1 else out


def mask_apply(mask, x, device: int = 0) -> np.ndarray:
    """MaskApplier::apply (circulant.cpp:27-37): Re(F^-1(h .* F x)), fp64 host I/O."""
    x = np.ascontiguousarray(x, np.float64)
    n = x.shape[-1]
    h = np.ascontiguousarray(np.asarray(mask, np.complex128)).view(np.float64).ravel()
    batch = x.size // (n * n)
    out = np.zeros_like(x)
    _check(lib().ncsg_mask_apply_host(n, h, x.ravel(), out.ravel(), batch, device), "mask_apply")
    return out


CT, DENOISE, PET = 0, 1, 2


@dataclass
class SolveResult:
    x: np.ndarray
    u: np.ndarray
    rows: np.ndarray  # (batch, k, 5): iter, objective, rel_subopt, seminorm, wall_ms
    objective: np.ndarray
    screen_est: float = float("nan")  # step-condition screen estimate (check_step_condition)


def fan_defaults(n: int) -> tuple[float, float]:
    """FanBeamGeometry::defaults (fanbeam.cpp:10-17): (source_radius, fan_angle)."""
    r, f = C.c_double(), C.c_double()
    _check(lib().ncsg_fan_defaults(n, C.byref(r), C.byref(f)), "fan_defaults")
    return r.value, f.value


class SparseMap:
    """SparseMap (sparse.hpp:21-43) on the GPU: CSR + stored transpose.
    FanBeam(...) builds build_fanbeam's matrix (fanbeam.cpp:43-111)."""

    def __init__(self, handle, n, views, rays):
        self._h = handle
        self.n, self.n_angles, self.n_det = n, views, rays

    @classmethod
    def from_triplets(cls, n, views, rays, rows, cols, vals, device: int = 0):
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        h = C.c_void_p()
        _check(lib().ncsg_sparse_create(n, views, rays, rows.size, rows.ctypes.data,
                                        cols.ctypes.data, vals.ctypes.data, device, C.byref(h)),
               "SparseMap")
        return cls(h, n, views, rays)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ncsg_sparse_destroy(self._h)
            self._h = None

    def nnz(self) -> int:
        return lib().ncsg_sparse_nnz(self._h)

    def forward(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        batch = x.size // (self.n * self.n)
        out = np.zeros((batch, self.n_angles, self.n_det))
        _check(lib().ncsg_sparse_forward_host(self._h, x.ravel(), out.ravel(), batch), "forward")
        return out.reshape(x.shape[:-2] + (self.n_angles, self.n_det))

    def adjoint(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        batch = u.size // (self.n_angles * self.n_det)
        out = np.zeros((batch, self.n, self.n))
        _check(lib().ncsg_sparse_adjoint_host(self._h, u.ravel(), out.ravel(), batch), "adjoint")
        return out.reshape(u.shape[:-2] + (self.n, self.n))


def _sparse_empirical_mask(self, samples: int = 8, seed: int = 0):
    """measurement_mask for this (non-parallel) geometry: empirical_mask(NormalMap(A),
    n, samples, seed) (circulant.cpp:98-140) -> ((n, n) complex mask, dead bins)."""
    out = np.zeros((self.n, self.n), np.complex128)
    dead = C.c_int()
    _check(lib().ncsg_sparse_empirical_mask(self._h, samples, seed, out.view(np.float64).ravel(),
                                            C.byref(dead)), "empirical_mask")
    return out, dead.value


SparseMap.empirical_mask = _sparse_empirical_mask


class FanBeam(SparseMap):
    """build_fanbeam(n, FanBeamGeometry{views, rays, source_radius, fan_angle})."""

    def __init__(self, n: int, views: int, rays: int, source_radius: float | None = None,
                 fan_angle: float | None = None, device: int = 0):
        r0, f0 = fan_defaults(n)
        self.source_radius = r0 if source_radius is None else source_radius
        self.fan_angle = f0 if fan_angle is None else fan_angle
        h = C.c_void_p()
        _check(lib().ncsg_fanbeam_create(n, views, rays, self.source_radius, self.fan_angle,
                                         device, C.byref(h)), "FanBeam")
        super().__init__(h, n, views, rays)


class Problem:
    """SplitProblem + SolverConfig + device Engine (solvers.hpp:24-78).

    kind CT: blocks {1, R, Quadratic, b}, {beta/alpha, D, ScaledL1(lambda alpha/beta)}
    kind DENOISE: blocks {1, I, Quadratic, b}, {beta/alpha, D, ...}
    positivity appends {1, I, Nonneg}.  mask=None selects PDHG (M = gamma I).
    """

    def __init__(self, kind: int, n: int, alpha: float, beta: float, lam: float, gamma: float,
                 b, mask=None, n_angles: int = 0, n_det: int = 0, batch: int = 1,
                 positivity: bool = False, pinv_rel_tol: float = 1e-12,
                 angle_range: tuple[int, int] = (0, 0), device: int = 0,
                 sparse: SparseMap | None = None, orbit_shard: tuple[int, int] = (0, 0)):
        self.kind, self.n, self.batch = kind, n, batch
        self._sparse = sparse  # keep the projector alive for the problem's lifetime
        if sparse is not None:
            n_angles, n_det = sparse.n_angles, sparse.n_det
        self.n_angles, self.n_det = n_angles, n_det
        self.alpha, self.beta, self.lam, self.gamma = alpha, beta, lam, gamma
        self.positivity = positivity
        b = np.ascontiguousarray(b, np.float64).ravel()
        m = n_angles * n_det if kind != DENOISE else n * n
        if b.size != batch * m:  # the C ABI reads batch * m offsets from b
            raise ValueError(f"offset size mismatch: got {b.size}, need batch*m = {batch * m}")
        if mask is not None and np.asarray(mask).size != n * n:
            raise ValueError(f"mask must have N*N = {n * n} entries")
        self._b = b
        d = ProblemDesc()
        d.kind, d.n, d.n_angles, d.n_det = kind, n, n_angles, n_det
        d.batch, d.positivity = batch, int(positivity)
        d.alpha, d.beta, d.lambda_, d.gamma = alpha, beta, lam, gamma
        d.pinv_rel_tol = pinv_rel_tol
        if mask is not None:
            self._mask = np.ascontiguousarray(np.asarray(mask, np.complex128)).view(np.float64)
            d.mask = self._mask.ctypes.data
        else:
            self._mask = None
            d.mask = None
        d.b = b.ctypes.data
        d.angle_begin, d.angle_end = angle_range
        d.device = device
        d.sparse = sparse._h if sparse is not None else None
        d.shard_rank, d.shard_count = orbit_shard
        h = C.c_void_p()
        _check(lib().ncsg_problem_create(C.byref(d), C.byref(h)), "problem_create")
        self._h = h
        self.range_size = lib().ncsg_problem_range_size(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ncsg_problem_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def stream(self):
        return lib().ncsg_problem_stream(self._h)

    def set_state(self, x=None, u=None, iter_: int = 0):
        xa = None if x is None else np.ascontiguousarray(x, np.float64).ravel()
        ua = None if u is None else np.ascontiguousarray(u, np.float64).ravel()
        _check(lib().ncsg_set_state(self._h, None if xa is None else xa.ctypes.data,
                                    None if ua is None else ua.ctypes.data, iter_), "set_state")

    def get_state(self):
        x = np.zeros((self.batch, self.n, self.n))
        u = np.zeros((self.batch, self.range_size))
        it = C.c_int64()
        _check(lib().ncsg_get_state(self._h, x.ctypes.data, u.ctypes.data, C.byref(it)),
               "get_state")
        return x, u, it.value

    def step(self, iters: int = 1, graph: bool = False):
        fn = lib().ncsg_step_graph if graph else lib().ncsg_step
        _check(fn(self._h, iters), "step")

    def sync(self):
        it = C.c_int64(-1)
        st = lib().ncsg_sync(self._h, C.byref(it))
        if st == 4:
            raise DivergenceError(st, lib().ncsg_last_error().decode(), it.value)
        _check(st, "sync")

    # -- angle-sharded step (multi-GPU): phase A, exchange A^T u, phase B --
    def bind_atu(self, tensor):
        """Use a caller-owned CUDA tensor (batch*N*N fp32) as the A^T u buffer."""
        self._atu = tensor
        _check(lib().ncsg_set_atu_buffer(self._h, C.c_void_p(tensor.data_ptr())), "bind_atu")

    def phase_a(self):
        _check(lib().ncsg_step_phase_a(self._h), "phase_a")

    def phase_b(self):
        _check(lib().ncsg_step_phase_b(self._h), "phase_b")

    def profile_begin(self):
        _check(lib().ncsg_profile_begin(self._h), "profile_begin")

    def profile_end(self) -> tuple[dict, int]:
        out = np.zeros(len(PHASES))
        steps = C.c_int()
        _check(lib().ncsg_profile_end(self._h, out, len(PHASES), C.byref(steps)), "profile_end")
        return dict(zip(PHASES, out.tolist())), steps.value

    def set_comm(self, comm: "Comm | None", exchange: int = XCHG_SLAB) -> None:
        """Attach a communicator: ncsg_step / solve then run the whole sharded
        iteration (ncsg_problem_set_comm)."""
        self._comm = comm
        _check(lib().ncsg_problem_set_comm(self._h, comm._h if comm else None, exchange),
               "set_comm")

    def plan(self) -> dict:
        """The live plan (partial-slot / partial-image counts, orbit mode,
        sample count) -- ncsg_problem_plan."""
        info = PlanInfo()
        _check(lib().ncsg_problem_plan(self._h, C.byref(info)), "plan")
        return {k: getattr(info, k) for k, _ in PlanInfo._fields_}

    def objective(self) -> np.ndarray:
        out = np.zeros(self.batch)
        _check(lib().ncsg_objective(self._h, out), "objective")
        return out

    def set_cg(self, n_cg: int) -> None:
        """admm_cg_solve mode (solvers.cpp:435-440): x-update by n_cg CG steps
        on A^T A (no mask, batch 1); n_cg = 0 restores the circulant solve."""
        _check(lib().ncsg_set_cg(self._h, n_cg), "set_cg")

    def screen(self, seed: int = 0, iters: int = 40) -> tuple[float, float]:
        """Engine::screen_step_condition (solvers.cpp:206-245): (estimate of the
        largest eigenvalue of alpha A^T A - M, shift)."""
        est, shift = C.c_double(), C.c_double()
        _check(lib().ncsg_screen_step_condition(self._h, seed, iters, C.byref(est),
                                                C.byref(shift)), "screen")
        return est.value, shift.value

    def solve(self, max_iters: int, record_every: int | None = None, f_star=None,
              check_step_condition: bool = False, seed: int = 0) -> SolveResult:
        if record_every is None:
            record_every = max(1, max_iters)
        max_rows = max_iters // max(1, record_every) + 3
        rows = (RecordRow * (max_rows * self.batch))()
        nr = C.c_int()
        est = C.c_double()
        fs = None
        if f_star is not None:
            fs = np.ascontiguousarray(np.broadcast_to(np.asarray(f_star, np.float64),
                                                      (self.batch,)))
        _check(lib().ncsg_solve(self._h, max_iters, record_every, int(check_step_condition),
                                seed, None if fs is None else fs.ctypes.data, rows, max_rows,
                                C.byref(nr), C.byref(est)), "solve")
        arr = np.array([[r.iter, r.objective, r.rel_subopt, r.seminorm_step, r.wall_ms]
                        for r in rows]).reshape(self.batch, max_rows, 5)[:, : nr.value]
        x, u, _ = self.get_state()
        return SolveResult(x, u, arr, arr[:, -1, 1].copy(), est.value)


class Comm:
    """A communicator of the sharded NCS step (ncsg_comm): NCCL, caller
    callbacks, or one rank of an in-process group."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep  # callback objects the C side points to

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().ncsg_nccl_unique_id(buf), "nccl_unique_id")
        return buf.raw

    @classmethod
    def nccl(cls, unique_id: bytes, rank: int, nranks: int, device: int = 0) -> "Comm":
        h = C.c_void_p()
        _check(lib().ncsg_comm_create_nccl(unique_id, rank, nranks, device, C.byref(h)),
               "comm_create_nccl")
        return cls(h)

    @classmethod
    def null(cls, rank: int, nranks: int) -> "Comm":
        """A rank whose collectives do nothing (timing one rank's kernels)."""
        h = C.c_void_p()
        _check(lib().ncsg_comm_create_null(rank, nranks, C.byref(h)), "comm_create_null")
        return cls(h)

    @classmethod
    def local_group(cls, nranks: int) -> list:
        hs = (C.c_void_p * nranks)()
        _check(lib().ncsg_comm_create_local(nranks, hs), "comm_create_local")
        return [cls(C.c_void_p(hs[r])) for r in range(nranks)]

    @classmethod
    def callbacks(cls, rank: int, nranks: int, all_reduce, reduce_scatter, all_gather,
                  all_to_all) -> "Comm":
        """Python callbacks (device pointers as ints; the stream is already
        synchronised; write results before returning)."""
        def safe(f, *a):
            try:
                f(*a)
                return 0
            except Exception:  # reported as NCSG_CUDA by the library
                import traceback

                traceback.print_exc()
                return -1

        fns = (_AllReduceFn(lambda ctx, buf, cnt, dt, op, st: safe(all_reduce, buf, cnt, dt, op)),
               _XferFn(lambda ctx, snd, rcv, cnt, st: safe(reduce_scatter, snd, rcv, cnt)),
               _XferFn(lambda ctx, snd, rcv, cnt, st: safe(all_gather, snd, rcv, cnt)),
               _XferFn(lambda ctx, snd, rcv, cnt, st: safe(all_to_all, snd, rcv, cnt)))
        ops = CommOps(None, rank, nranks, *fns)
        h = C.c_void_p()
        _check(lib().ncsg_comm_create_callbacks(C.byref(ops), C.byref(h)), "comm_create_callbacks")
        return cls(h, keep=(fns, ops))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ncsg_comm_destroy(self._h)
            self._h = None


def ct_problem(cfg, b, mask=None, batch=None, **kw) -> Problem:
    """Problem for a pinned CT config (paper_1810_13100_b200.configs)."""
    return Problem(CT, cfg.n, cfg.alpha, cfg.beta, cfg.lam, cfg.gamma, b, mask=mask,
                   n_angles=cfg.angles, n_det=cfg.det, batch=batch or cfg.batch, **kw)


def denoise_problem(cfg, b, mask=None, **kw) -> Problem:
    return Problem(DENOISE, cfg.n, cfg.alpha, cfg.beta, cfg.lam, cfg.gamma, b, mask=mask,
                   batch=cfg.batch, **kw)


def write_record_csv(path: str, rows) -> None:
    """write_record_csv (io.cpp:203-215) for one problem's record rows
    (iter, objective, rel_subopt, seminorm_step, wall_ms): same header and
    %.17g formatting as the reference."""
    with open(path, "w") as f:
        f.write("iter,objective,rel_subopt,seminorm_step,wall_ms\n")
        for r in np.asarray(rows).reshape(-1, 5):
            f.write("%d,%.17g,%.17g,%.17g,%.17g\n" % (int(r[0]), r[1], r[2], r[3], r[4]))
