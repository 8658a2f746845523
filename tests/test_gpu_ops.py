"""Per-operator parity of the CUDA path against the oracle (north_star: relative
L2 error <= 1e-5 for R, R^T, D and the FFT solve), through the C ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / max(1e-300, np.linalg.norm(b)))


GEOMS = [
    (16, 12, 25),    # python smoke geometry (test_smoke.py:36-49)
    (32, 30, 47),
    (64, 48, 93),    # impulse geometry (test_ops.cpp:37-47)
    (64, 60, 93),    # adjoint-probe geometry (test_ops.cpp:32-35)
    (100, 37, 143),  # non power of two, odd angle count
    (17, 9, 27),     # odd N (half-integer centre is integer)
    (64, 1, 93),     # single angle
    (64, 4, 95),     # angles exactly 0, 45, 90, 135 degrees
    (200, 8, 301),   # wide detector, N not a multiple of the tile sizes
    (33, 8, 49),     # odd N in orbit mode: theta = 0 samples on the image edge
    (65, 12, 93),    # odd N, orbit mode, N not a multiple of the gather tile
    (48, 4, 71),     # orbits of 0 and 45 degrees only (absent members)
]


@pytest.mark.parametrize("n,A,D", GEOMS)
def test_radon_forward_adjoint_small(ncsg, port, n, A, D):
    rng = np.random.default_rng(n * 1000 + A)
    x = rng.standard_normal((n, n))
    u = rng.standard_normal((A, D))
    R = ncsg.RadonMap(n, A, D)
    assert R.sample_count() == port.radon_valid_counts(n, A, D).sum()
    assert rel(R.forward(x), port.radon_forward(x, A, D)) <= TOL
    assert rel(R.adjoint(u), port.radon_adjoint(u, n)) <= TOL


@pytest.mark.parametrize("n,A,D", [(33, 8, 49), (65, 12, 93), (64, 60, 93), (128, 180, 185)])
def test_gather_adjoint_border_pixels(ncsg, port, n, A, D):
    """The orbit gather's exact-validity path: the image's border rows and
    columns (the only pixels a sample outside the square can reach) agree
    with the oracle element-wise, and the gather agrees with the per-angle
    scatter kernel (NCSG_NO_GATHER)."""
    import os
    rng = np.random.default_rng(n + A)
    u = rng.standard_normal((A, D))
    ref = port.radon_adjoint(u, n)
    got = ncsg.RadonMap(n, A, D).adjoint(u)
    border = np.zeros((n, n), bool)
    border[0, :] = border[-1, :] = border[:, 0] = border[:, -1] = True
    scale = np.abs(ref).max()
    assert np.abs(got - ref)[border].max() <= 1e-5 * scale
    os.environ["NCSG_NO_GATHER"] = "1"
    try:
        scat = ncsg.RadonMap(n, A, D).adjoint(u)
    finally:
        del os.environ["NCSG_NO_GATHER"]
    assert rel(got, scat) <= TOL


@pytest.mark.parametrize("knob,values", [("NCSG_ORB_SEG_ROWS", ["32", "64", "96"]),
                                         ("NCSG_GA_CHUNKS", ["1", "3", "7", "12"])])
def test_projector_sizing_knobs(ncsg, port, knob, values):
    """The launch-shape choices (forward segment height, adjoint orbit
    chunks) only change the partial-sum grouping: every setting matches the
    oracle."""
    import os
    n, A, D = 160, 48, 229
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, n))
    u = rng.standard_normal((A, D))
    ref_f, ref_a = port.radon_forward(x, A, D), port.radon_adjoint(u, n)
    for v in values:
        os.environ[knob] = v
        try:
            R = ncsg.RadonMap(n, A, D)
            assert rel(R.forward(x), ref_f) <= TOL, (knob, v)
            assert rel(R.adjoint(u), ref_a) <= TOL, (knob, v)
        finally:
            del os.environ[knob]


def test_radon_batched_multi_chunk(ncsg, port):
    """Batched operators with several orbit chunks per problem (the gather's
    partial images and tile bookkeeping are per batch element)."""
    n, A, D = 96, 40, 137
    rng = np.random.default_rng(9)
    x = rng.standard_normal((3, n, n))
    u = rng.standard_normal((3, A, D))
    R = ncsg.RadonMap(n, A, D)
    fx, au = R.forward(x), R.adjoint(u)
    for q in range(3):
        assert rel(fx[q], port.radon_forward(x[q], A, D)) <= TOL
        assert rel(au[q], port.radon_adjoint(u[q], n)) <= TOL


@pytest.mark.parametrize("name", ["c1", "c3", "c5"])
def test_radon_config_sizes(ncsg, port, name):
    from paper_1810_13100_b200 import configs

    cfg = configs.get(name)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((cfg.n, cfg.n))
    u = rng.standard_normal((cfg.angles, cfg.det))
    R = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det)
    assert R.sample_count() == port.radon_valid_counts(cfg.n, cfg.angles, cfg.det).sum()
    assert rel(R.forward(x), port.radon_forward(x, cfg.angles, cfg.det)) <= TOL
    assert rel(R.adjoint(u), port.radon_adjoint(u, cfg.n)) <= TOL


@pytest.mark.slow
def test_radon_c4_size(ncsg, port):
    """C4 (2048^2, 2048 x 2897): forward on a ray sample, adjoint in full."""
    from paper_1810_13100_b200 import configs

    cfg = configs.base("c4")
    rng = np.random.default_rng(11)
    x = rng.standard_normal((cfg.n, cfg.n))
    R = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det)
    y = R.forward(x).ravel()
    rays = rng.choice(cfg.angles * cfg.det, 20000, replace=False)
    assert rel(y[rays], port.radon_forward_rays(x, cfg.angles, cfg.det, rays)) <= TOL
    u = rng.standard_normal((cfg.angles, cfg.det))
    assert rel(R.adjoint(u), port.radon_adjoint(u, cfg.n)) <= TOL
    assert R.sample_count() == 8581547248  # SURVEY.md §8 sizes table


def test_gather_adjoint_table_and_direct_modes(ncsg, port, monkeypatch):
    # the gather adjoint with its window-weight table (built per plan, 21-bit
    # fixed-point weights) and with the windows evaluated every step
    # (NCSG_GA_WTAB=0; also the fallback above NCSG_GA_WTAB_MAX_GB) agree with
    # each other and with radon.cpp:104-127
    n, A = 96, 64  # not a multiple of the 32 x 32 tile: padded edge tiles
    D = ncsg.default_detector_count(n)
    u = np.random.default_rng(3).standard_normal((A, D))
    want = port.radon_adjoint(u, n)
    got = {}
    for mode, env in (("table", {}), ("direct", {"NCSG_GA_WTAB": "0"}),
                      ("capped", {"NCSG_GA_WTAB_MAX_GB": "0.000001"})):
        for k in ("NCSG_GA_WTAB", "NCSG_GA_WTAB_MAX_GB"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        got[mode] = ncsg.RadonMap(n, A, D).adjoint(u)
        assert rel(got[mode], want) <= TOL
    assert np.array_equal(got["direct"], got["capped"])
    assert rel(got["table"], got["direct"]) <= 4e-6
    for k in ("NCSG_GA_WTAB", "NCSG_GA_WTAB_MAX_GB"):
        monkeypatch.delenv(k, raising=False)
    b = np.zeros((A, D))
    p = ncsg.Problem(ncsg.CT, n, 0.1, 0.1, 0.01, 1.0, b, n_angles=A, n_det=D)
    plan = p.plan()  # 8 bytes per (pixel of the 3 x 3 whole tiles, orbit)
    assert plan["adjoint_table_bytes"] == 8 * plan["n_orbits"] * 9 * 1024
    monkeypatch.setenv("NCSG_GA_WTAB", "0")
    q = ncsg.Problem(ncsg.CT, n, 0.1, 0.1, 0.01, 1.0, b, n_angles=A, n_det=D)
    assert q.plan()["adjoint_table_bytes"] == 0


def test_adjoint_identity_and_determinism(ncsg):
    n, A, D = 128, 180, 185
    rng = np.random.default_rng(3)
    x, u = rng.standard_normal((n, n)), rng.standard_normal((A, D))
    R = ncsg.RadonMap(n, A, D)
    y1, y2 = R.forward(x), R.forward(x)
    z1, z2 = R.adjoint(u), R.adjoint(u)
    np.testing.assert_array_equal(y1, y2)  # bitwise reproducible (test_ops.cpp:49-58)
    np.testing.assert_array_equal(z1, z2)
    lhs, rhs = np.vdot(y1, u), np.vdot(x, z1)
    assert abs(lhs - rhs) / abs(lhs) <= 1e-5


def test_batched_projector_equals_single(ncsg):
    n, A, D = 64, 48, 93
    rng = np.random.default_rng(4)
    xs = rng.standard_normal((3, n, n))
    us = rng.standard_normal((3, A, D))
    R = ncsg.RadonMap(n, A, D)
    yb, zb = R.forward(xs), R.adjoint(us)
    for k in range(3):
        np.testing.assert_array_equal(yb[k], R.forward(xs[k]))
        np.testing.assert_array_equal(zb[k], R.adjoint(us[k]))


def test_impulse_projects_to_one_per_angle(ncsg):
    # test_ops.cpp:37-47
    n = 64
    x = np.zeros((n, n))
    x[32, 32] = 1.0
    s = ncsg.RadonMap(n, 48).forward(x)
    np.testing.assert_allclose(s.sum(axis=1), 1.0, rtol=0.05)


def test_zero_in_zero_out(ncsg):
    R = ncsg.RadonMap(32, 30)
    assert not R.forward(np.zeros((32, 32))).any()
    assert not R.adjoint(np.zeros((30, 47))).any()


def test_grad_parity(ncsg, port):
    for n in (2, 3, 17, 64):
        rng = np.random.default_rng(n)
        x = rng.standard_normal((n, n))
        g = rng.standard_normal(2 * n * (n - 1))
        G = ncsg.GradMap(n)
        assert rel(G.forward(x), port.grad_forward(x)) <= TOL
        assert rel(G.adjoint(g), port.grad_adjoint(g, n)) <= TOL
    # 3x3 hand values (test_ops.cpp:60-79)
    x = np.array([1, 2, 4, 8, 16, 32, 64, 128, 256], float).reshape(3, 3)
    g = ncsg.GradMap(3).forward(x)
    assert g[0] == -1 and g[2] == -8 and g[6] == 1 - 8 and g[11] == 32 - 256


# 8-32: shared-memory Stockham passes; 64-4096: the register-resident
# power-of-two engine (fft_pow2.cuh), every last-stage radix (64: 16x4,
# 128: 16x8, 256: 16x16, 512: 16x16x2, 2048: 16x16x8, 4096: 16x16x16)
@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_mask_apply_parity(ncsg, port, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, n))
    h = port.radon_mask(n, 3.0, 7.0) + port.laplacian_mask(n)
    assert rel(ncsg.mask_apply(h, x), port.mask_apply(h, x)) <= TOL
    if n <= 512:  # a general complex mask (Hermitian part taken, circulant.cpp:36)
        hc = h + 0.5j * rng.standard_normal((n, n))
        assert rel(ncsg.mask_apply(hc, x), port.mask_apply(hc, x)) <= TOL


def test_mask_apply_identity_and_constants(ncsg):
    # SPEC.md apply_circulant examples: h == 1 -> x; Laplacian kills constants
    n = 16
    x = np.random.default_rng(1).standard_normal((n, n))
    np.testing.assert_allclose(ncsg.mask_apply(np.ones((n, n)), x), x, atol=1e-6)
    from paper_1810_13100_b200.instances import laplacian_mask

    assert np.abs(ncsg.mask_apply(laplacian_mask(n), np.full((n, n), 3.0))).max() < 1e-5


@pytest.mark.parametrize("n", [9, 12, 15, 30, 100, 105, 126, 96])
def test_mask_apply_mixed_radix_sizes(ncsg, port, n):
    # MaskApplier::apply for sizes the reference's FFTW handles and the
    # radix-8 fast path does not: mixed-radix (2, 3, 4, 5, 7, 8) Stockham
    # stages, odd sizes included (the half spectrum then has no Nyquist column)
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, n))
    h = (port.laplacian_mask(n) + port.radon_mask(n, 3.0, 5.0)
         + 0.3j * rng.standard_normal((n, n)))
    want = port.mask_apply(h, x)
    assert rel(ncsg.mask_apply(h, x), want) <= 1e-5


@pytest.mark.parametrize("n", [11, 22, 26, 33, 97, 121, 143, 187, 251, 442, 509])
def test_mask_apply_other_prime_factors(ncsg, port, n):
    # FFTW takes any N (fft.cpp:18-29): prime factors above 7 (11, 13, 17, ...,
    # prime N itself) run the one-output-per-thread generic Stockham stage
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, n))
    h = (port.laplacian_mask(n) + port.radon_mask(n, 3.0, 5.0)
         + 0.3j * rng.standard_normal((n, n)))
    assert rel(ncsg.mask_apply(h, x), port.mask_apply(h, x)) <= 1e-5


@pytest.mark.parametrize("n,views,rays", [(16, 12, 21), (32, 24, 45), (64, 40, 91)])
def test_fanbeam_sparse_map(ncsg, port, n, views, rays):
    # build_fanbeam + SparseMap::forward/adjoint (fanbeam.cpp, sparse.cpp:55-71)
    R, fan = port.fan_defaults(n)
    assert (R, fan) == ncsg.fan_defaults(n)
    A = ncsg.FanBeam(n, views, rays)
    rows, cols, vals = port.fanbeam_triplets(n, views, rays, R, fan)
    assert A.nnz() == rows.size
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, n))
    u = rng.standard_normal((views, rays))
    fx = port.fanbeam_apply(n, views, rays, R, fan, x)
    au = port.fanbeam_apply(n, views, rays, R, fan, u, adjoint=True)
    assert rel(A.forward(x), fx) <= 1e-5
    assert rel(A.adjoint(u), au) <= 1e-5
    # the same matrix from triplets
    B = ncsg.SparseMap.from_triplets(n, views, rays, rows, cols, vals)
    np.testing.assert_array_equal(B.forward(x), A.forward(x))
