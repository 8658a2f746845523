"""Generates the small reference golden fixtures tests/golden/ref_*.npz from
the reference's own sources compiled unchanged (oracle/_ref/libncsref.so):
R / R^T of seeded inputs and a short ncs_solve per case, all computed by the
reference itself.  tests/test_oracle_pin.py checks the oracle against them
bitwise (one thread) and tests/test_gpu_solver.py checks the CUDA path
within the parity bar.  Run here (the reference is only present in this
container): `python oracle/gen_golden.py`."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Prob, Ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ct_case(ref, port, name, n, A, iters, record_every, lam=0.01, positivity=False, seed=3):
    D = port.default_detector_count(n)
    rng = np.random.default_rng(seed)
    x = ref.make_phantom(n, [[1.0, 0.1, -0.05, 0.7, 0.5, 0.0],   # intensity, x0, y0, a, b, rot
                             [-0.4, 0.2, 0.3, 0.35, 0.25, 0.1]])
    clean = ref.radon_forward(x, A, D)
    b = clean + 0.01 * np.max(clean) * ref.rng_normals(seed, 1, A * D).reshape(A, D)
    radon_x = rng.standard_normal((n, n))
    radon_u = rng.standard_normal((A, D))
    alpha = 0.1
    dc = float((ref.radon_forward(np.ones((n, n)), A, D) ** 2).sum() / n ** 2)
    mask = ref.ct_metric_mask(n, A, D, alpha, alpha, dc, samples=8, seed=0,
                              positivity=positivity)
    prob = Prob(0, n, A, D, alpha, alpha, lam, b, positivity=positivity)
    gamma = 1.2 * port.screen(prob, 0.0, mask, iters=40)
    r = ref.solve(prob, gamma, mask, iters, record_every=record_every)
    np.savez_compressed(os.path.join(OUT, f"ref_{name}.npz"), kind=0, n=n, angles=A, det=D,
                        alpha=alpha, beta=alpha, lam=lam, gamma=gamma, positivity=int(positivity),
                        b=b, mask=mask, iters=iters, record_every=record_every,
                        x=r.x, u=r.u, rows=r.rows, radon_x=radon_x,
                        radon_fwd=ref.radon_forward(radon_x, A, D), radon_u=radon_u,
                        radon_adj=ref.radon_adjoint(radon_u, n))
    print(name, "gamma", gamma, "objective", r.rows[-1, 1])


def tv_case(ref, port, name, n, iters, record_every, lam=0.05, seed=4):
    x = ref.make_phantom(n, [[1.0, 0.0, 0.1, 0.6, 0.4, 0.2]])
    b = x + 0.1 * ref.rng_normals(seed, 2, n * n).reshape(n, n)
    mask = ref.metric_mask(np.ones((n, n)), 1.0, 1.0)
    prob = Prob(1, n, 0, 0, 1.0, 1.0, lam, b)
    gamma = 1e-3
    r = ref.solve(prob, gamma, mask, iters, record_every=record_every)
    np.savez_compressed(os.path.join(OUT, f"ref_{name}.npz"), kind=1, n=n, angles=0, det=0,
                        alpha=1.0, beta=1.0, lam=lam, gamma=gamma, positivity=0, b=b, mask=mask,
                        iters=iters, record_every=record_every, x=r.x, u=r.u, rows=r.rows)
    print(name, "objective", r.rows[-1, 1])


def main():
    os.makedirs(OUT, exist_ok=True)
    ref, port = Ref(), Port()
    ct_case(ref, port, "ct16", 16, 12, 30, 10)
    ct_case(ref, port, "ct32", 32, 30, 60, 20)
    ct_case(ref, port, "ct32_pos", 32, 24, 40, 10, positivity=True)
    tv_case(ref, port, "tv32", 32, 60, 20)


if __name__ == "__main__":
    main()
