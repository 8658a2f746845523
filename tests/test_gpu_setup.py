"""GPU setup path against the oracle and, where it is
built, the reference itself: calibrate_scale (circulant.cpp:142-169), the DC
response of R^T R, measurement_mask (pipeline.cpp:100-110) and the
step-condition power-method screen (solvers.cpp:206-245, 466-484).

Tolerances: the GPU applies R, R^T and the FFT in fp32 and accumulates the
sums in fp64, so scalar results agree to ~1e-6 relative; the screen estimate
is lambda - shift, a difference of two numbers of size `shift`, so it is
compared with an absolute tolerance of 1e-4 * shift."""
import numpy as np
import pytest

from oracle.oracle import Prob
from test_gpu_solver import gpu_problem, small_ct

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,A,samples,seed", [(32, 30, 8, 0), (64, 48, 3, 7), (128, 180, 8, 0)])
def test_calibrate_scale_matches_oracle(ncsg, port, n, A, samples, seed):
    D = port.default_detector_count(n)
    want = port.calibrate_scale(n, A, D, samples, seed)
    got = ncsg.RadonMap(n, A, D).calibrate_scale(samples, seed)
    assert abs(got - want) <= 1e-5 * abs(want), (got, want)


def test_calibrate_scale_matches_reference(ncsg, ref):
    n, A = 32, 30
    D = ncsg.default_detector_count(n)
    want = ref.calibrate_scale(n, A, D, 8, 0)
    got = ncsg.RadonMap(n, A, D).calibrate_scale(8, 0)
    assert abs(got - want) <= 1e-5 * abs(want), (got, want)


def test_calibrate_scale_rejects_bad_samples(ncsg):
    with pytest.raises(ValueError):
        ncsg.RadonMap(32, 30).calibrate_scale(0, 0)


@pytest.mark.parametrize("n,A", [(32, 30), (64, 48)])
def test_dc_response(ncsg, port, n, A):
    D = port.default_detector_count(n)
    want = float((port.radon_forward(np.ones((n, n)), A, D) ** 2).sum() / n ** 2)
    got = ncsg.RadonMap(n, A, D).dc_response()
    assert abs(got - want) <= 1e-6 * want, (got, want)


def test_measurement_mask(ncsg, port):
    n, A = 64, 48
    D = port.default_detector_count(n)
    dc = float((port.radon_forward(np.ones((n, n)), A, D) ** 2).sum() / n ** 2)
    want = port.radon_mask(n, port.calibrate_scale(n, A, D, 8, 0), dc)
    got = ncsg.RadonMap(n, A, D).measurement_mask(8, 0)
    assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


def _check_screen(got, shift, want):
    assert abs(got - want) <= 1e-4 * shift, (got, want, shift)


@pytest.mark.parametrize("gamma_scale", [0.0, 1.2])
def test_screen_ct(ncsg, port, gamma_scale):
    prob, mask, gamma = small_ct(port)
    g = gamma_scale * gamma
    want = port.screen(prob, g, mask, iters=40, seed=0)
    est, shift = gpu_problem(ncsg, prob, g, mask).screen(0, 40)
    _check_screen(est, shift, want)
    if gamma_scale == 0.0:
        assert est > 0.0  # gamma = 0 violates the step condition
    else:
        assert est < 0.0


def test_screen_seed_and_iters(ncsg, port):
    prob, mask, gamma = small_ct(port, n=32, A=24)
    for seed, iters in [(3, 15), (11, 40)]:
        want = port.screen(prob, 0.0, mask, iters=iters, seed=seed)
        est, shift = gpu_problem(ncsg, prob, 0.0, mask).screen(seed, iters)
        _check_screen(est, shift, want)


def test_screen_pdhg_and_positivity(ncsg, port):
    prob, mask, gamma = small_ct(port, n=32, A=24)
    gp = 1.2 * port.screen(prob, 0.0, None, iters=40) + 1.0
    want = port.screen(prob, gp, None, iters=40)
    est, shift = gpu_problem(ncsg, prob, gp, None).screen(0, 40)
    assert shift == pytest.approx(gp)
    _check_screen(est, shift, want)
    prob.positivity = True
    mask = mask + 1.0
    want = port.screen(prob, 0.0, mask, iters=40)
    est, shift = gpu_problem(ncsg, prob, 0.0, mask).screen(0, 40)
    _check_screen(est, shift, want)


def test_screen_denoise(ncsg, port):
    from paper_1810_13100_b200 import datagen

    n = 64
    x = datagen.phantom(n, 5, 3)
    b = x + 0.1 * datagen.stream_noise(x.shape, 4)
    prob = Prob(1, n, 0, 0, 1.0, 1.0, 0.05, b)
    mask = np.ones((n, n)) + port.laplacian_mask(n)
    for g in (0.0, 1e-3):
        want = port.screen(prob, g, mask, iters=40)
        est, shift = gpu_problem(ncsg, prob, g, mask).screen(0, 40)
        _check_screen(est, shift, want)


def test_solve_runs_screen(ncsg, port):
    # solve_template (solvers.cpp:278): check_step_condition screens before
    # the loop; the iterates are unaffected.
    prob, mask, gamma = small_ct(port, n=32, A=24)
    want = port.screen(prob, gamma, mask, iters=40, seed=5)
    a = gpu_problem(ncsg, prob, gamma, mask).solve(10, check_step_condition=True, seed=5)
    b = gpu_problem(ncsg, prob, gamma, mask).solve(10)
    _check_screen(a.screen_est, gamma + prob.alpha * np.max(np.abs(mask)), want)
    assert np.isnan(b.screen_est)
    np.testing.assert_array_equal(a.x, b.x)


def test_screen_gamma_rule(ncsg, port):
    # The configs' gamma rule (gamma = 1.05 * screen at gamma = 0) needs the
    # gamma = 0 estimate itself to ~1e-5 relative.
    prob, mask, gamma = small_ct(port, n=32, A=24)
    est, _ = gpu_problem(ncsg, prob, 0.0, mask).screen(0, 40)
    want = port.screen(prob, 0.0, mask, iters=40)
    assert abs(est - want) <= 1e-5 * abs(want)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c3", "c5", "c4", "c2"])
def test_pinned_setup_values_full_size(ncsg, name):
    # oracle/pin_configs.py computed dc, the mask scale and the gamma = 0
    # screen estimate of every BASELINE config with the oracle (fp64, CPU);
    # the GPU setup path reproduces them at full size.
    from paper_1810_13100_b200 import configs, instances

    cfg = configs.get(name)
    if cfg.kind == "ct":
        r = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det)
        assert abs(r.dc_response() - cfg.dc) <= 1e-5 * cfg.dc
        scale = r.calibrate_scale(cfg.pinned["mask_samples"], cfg.pinned["mask_seed"])
        assert abs(scale - cfg.mask_scale) <= 1e-5 * cfg.mask_scale, (scale, cfg.mask_scale)
        del r
    mask = instances.metric_mask(cfg)
    kind = ncsg.CT if cfg.kind == "ct" else ncsg.DENOISE
    p = ncsg.Problem(kind, cfg.n, cfg.alpha, cfg.beta, cfg.lam, 0.0, np.zeros(cfg.m), mask=mask,
                     n_angles=cfg.angles, n_det=cfg.det)
    est, shift = p.screen(0, 40)
    _check_screen(est, shift, cfg.pinned["screen_lmax"])


@pytest.mark.parametrize("n,views,rays,samples", [(16, 12, 23, 4), (32, 24, 45, 8)])
def test_fanbeam_empirical_mask(ncsg, port, ref, n, views, rays, samples):
    # measurement_mask for fan beam = empirical_mask (circulant.cpp:98-140):
    # fp32 spectra on the GPU against the fp64 oracle (itself pinned to the
    # reference at 1e-12); per-bin ratios of F(A^T A v)/F(v), so bins where
    # a probe's |F v| is small carry larger relative error.
    R, fan = port.fan_defaults(n)
    want, dead_o = port.fanbeam_empirical_mask(n, views, rays, R, fan, samples, 3)
    got, dead_g = ncsg.FanBeam(n, views, rays).empirical_mask(samples, 3)
    assert dead_g == dead_o
    scale = np.max(np.abs(want))
    assert np.max(np.abs(got - want)) <= 1e-4 * scale
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c3", "c5"])
def test_converged_power_method_full_size(ncsg, name):
    # the 300-step estimate gamma is pinned to (oracle/pin_configs.py) -- the
    # GPU reproduces the oracle's converged lambda_max at full size
    from paper_1810_13100_b200 import configs, instances

    cfg = configs.get(name)
    assert cfg.pinned["lmax_source"] == "oracle"
    mask = instances.metric_mask(cfg)
    p = ncsg.Problem(ncsg.CT, cfg.n, cfg.alpha, cfg.beta, cfg.lam, 0.0, np.zeros(cfg.m), mask=mask,
                     n_angles=cfg.angles, n_det=cfg.det)
    est, shift = p.screen(0, cfg.pinned["lmax_iters"])
    _check_screen(est, shift, cfg.pinned["lmax"])

