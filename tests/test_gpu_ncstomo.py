"""The GPU drop-in for the reference's Python module (paper_1810_13100_b200.ncstomo,
bindings.cpp:180-336) against the reference build: reconstruct with the ncs
(explicit and "auto" mask), pdhg and admm solvers, Geometry forward/adjoint,
simulate_ct, default_params and the argument errors of bindings.cpp."""
import numpy as np
import pytest

from oracle.oracle import Prob

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(1e-300, np.linalg.norm(np.ravel(b))))


@pytest.fixture(scope="module")
def nt(ncsg):
    from paper_1810_13100_b200 import ncstomo

    return ncstomo


def case(nt, port, n=32, angles=24):
    g = nt.Geometry("parallel", n, angles)
    x = nt.make_phantom(n, [nt.Ellipse(1.0, 0.1, -0.05, 0.7, 0.5, 0.0),
                            nt.Ellipse(-0.4, 0.2, 0.3, 0.35, 0.25, 10.0)])
    sino = port.radon_forward(x, angles, g.n_detectors)
    sino = sino + 0.01 * sino.max() * np.random.default_rng(3).standard_normal(sino.shape)
    return g, x, sino


def test_geometry_and_simulate(nt, port):
    g = nt.Geometry("parallel", 32, 24)
    assert (g.n_angles, g.n_detectors) == (24, port.default_detector_count(32))
    x = np.random.default_rng(1).standard_normal((32, 32))
    assert rel(g.forward(x), port.radon_forward(x, 24, g.n_detectors)) <= 1e-5
    s = nt.simulate_ct(x, g, 0.5, 7)
    noise = s - g.forward(x)
    assert abs(np.std(noise) - 0.5) < 0.05
    with pytest.raises(ValueError):
        g.forward(np.zeros((16, 16)))
    with pytest.raises(ValueError):
        nt.Geometry("cone", 32, 24)
    f = nt.Geometry("fan", 32, 24)
    R, fan = port.fan_defaults(32)
    assert rel(f.forward(x), port.fanbeam_apply(32, 24, f.n_detectors, R, fan, x)) <= 1e-5


def test_reconstruct_ncs_matches_reference(nt, port, ref):
    g, x, sino = case(nt, port)
    p = nt.default_params("ct")
    alpha = beta = 0.1
    dc = 300.0
    meas = nt.measurement_mask(g, dc, 8, 0)
    want_mask = ref.ct_metric_mask(32, 24, g.n_detectors, alpha, beta, dc)
    mask = meas + (beta / alpha) ** 2 * port.laplacian_mask(32)
    assert np.max(np.abs(mask - want_mask)) <= 1e-5 * np.max(np.abs(want_mask))
    prob = Prob(0, 32, 24, g.n_detectors, alpha, beta, 0.01, sino)
    gamma = 1.2 * port.screen(prob, 0.0, want_mask, iters=300)
    r = ref.solve(prob, gamma, want_mask, 40, record_every=10)
    out = nt.reconstruct(sino, g, solver="ncs", iters=40, alpha=alpha, beta=beta, gamma=gamma,
                         lambda_=0.01, dc=dc, mask="auto", record_every=10)
    assert rel(out.image, r.x) <= 1e-4
    assert out.records.shape == (5, 5) and out.iters == 40
    assert abs(out.objective - r.objective) <= 1e-4 * abs(r.objective)
    assert out.warnings == []
    # gamma far too small: the screen warns (solvers.cpp:238-244)
    bad = nt.reconstruct(sino, g, iters=2, alpha=alpha, beta=beta, gamma=1e-3, lambda_=0.01,
                         dc=dc, mask="auto")
    assert bad.warnings and "step condition" in bad.warnings[0]


def test_reconstruct_pdhg_and_admm(nt, port, ref):
    g, x, sino = case(nt, port)
    prob = Prob(0, 32, 24, g.n_detectors, 0.1, 0.1, 0.01, sino)
    gp = 1.2 * port.screen(prob, 0.0, None, iters=300) + 1.0
    r = ref.solve(prob, gp, None, 40, record_every=10, pdhg=True)
    out = nt.reconstruct(sino, g, solver="pdhg", iters=40, alpha=0.1, beta=0.1, gamma=gp,
                         lambda_=0.01, record_every=10)
    assert rel(out.image, r.x) <= 1e-4
    ra = ref.admm_cg_solve(prob, 0.0, 2, 10, record_every=5)
    oa = nt.reconstruct(sino, g, solver="admm", iters=10, alpha=0.1, beta=0.1, gamma=0.0,
                        lambda_=0.01, cg_iters=2, record_every=5)
    assert rel(oa.image, ra.x) <= 1e-4
    assert oa.records[-1, 0] == 20


def test_reconstruct_argument_errors(nt, port):
    g, x, sino = case(nt, port, n=16, angles=12)
    with pytest.raises(ValueError):
        nt.reconstruct(sino, g, solver="pdhg", mask="auto")
    with pytest.raises(ValueError):
        nt.reconstruct(sino, g, mask="bogus")
    with pytest.raises(ValueError):
        nt.reconstruct(sino, g, solver="sgd")
    with pytest.raises(ValueError):
        nt.reconstruct(sino[:, :-1], g)
    with pytest.raises(ValueError):
        nt.reconstruct(sino, g, iters=-1)
