"""Quick GPU-vs-oracle sanity check (development helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Port, Prob
from paper_1810_13100_b200 import ncsg, configs, instances

P = Port()
rng = np.random.default_rng(0)

def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(1e-300, np.linalg.norm(np.ravel(b))))

for (n, A) in [(16, 12), (32, 30), (64, 48), (128, 180), (100, 37), (256, 360), (512, 720)]:
    D = P.default_detector_count(n) if n != 128 else 185
    if n == 256: D = 363
    if n == 512: D = 725
    x = rng.standard_normal((n, n)); u = rng.standard_normal((A, D))
    R = ncsg.RadonMap(n, A, D)
    t = time.time(); y = R.forward(x); t1 = time.time() - t
    yo = P.radon_forward(x, A, D)
    t = time.time(); z = R.adjoint(u); t2 = time.time() - t
    zo = P.radon_adjoint(u, n)
    cnt = P.radon_valid_counts(n, A, D).sum()
    print(f"n={n} A={A} D={D}: fwd rel {rel(y, yo):.2e} adj rel {rel(z, zo):.2e} samples gpu {R.sample_count()} oracle {cnt}  ({t1:.3f}s,{t2:.3f}s)", flush=True)
    lhs = np.vdot(y, u); rhs = np.vdot(x, z); print("   adjoint identity", abs(lhs - rhs) / abs(lhs))

n = 64
x = rng.standard_normal((n, n)); G = ncsg.GradMap(n)
print("grad", rel(G.forward(x), P.grad_forward(x)), rel(G.adjoint(P.grad_forward(x)), P.grad_adjoint(P.grad_forward(x), n)))
for n in (8, 16, 64, 256):
    x = rng.standard_normal((n, n))
    h = P.radon_mask(n, 3.0, 7.0) + P.laplacian_mask(n)
    h2 = h + 0.3j * rng.standard_normal((n, n))
    print("mask", n, rel(ncsg.mask_apply(h, x), P.mask_apply(h, x)), rel(ncsg.mask_apply(h2, x), P.mask_apply(h2, x)))

# NCS parity at C1
cfg = configs.get("c1")
x_true, b = instances.make_instance(cfg, lambda im: P.radon_forward(im, cfg.angles, cfg.det))
mask = instances.metric_mask(cfg)
prob = Prob(0, cfg.n, cfg.angles, cfg.det, cfg.alpha, cfg.beta, cfg.lam, b)
for iters in (1, 10, 100, 500):
    t = time.time(); ro = P.solve(prob, cfg.gamma, mask, iters); to = time.time() - t
    pg = ncsg.ct_problem(cfg, b, mask=mask)
    pg.set_state()
    t = time.time(); rg = pg.solve(iters); tg = time.time() - t
    print(f"C1 iters={iters}: x rel {rel(rg.x[0], ro.x):.2e} u rel {rel(rg.u[0], ro.u):.2e} obj {rg.objective[0]:.8e} vs {ro.objective:.8e} rel {abs(rg.objective[0]-ro.objective)/abs(ro.objective):.2e} sem {rg.rows[0,-1,3]:.6e} vs {ro.rows[-1,3]:.6e}  oracle {to:.2f}s gpu {tg:.3f}s", flush=True)
