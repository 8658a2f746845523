"""Generates tests/golden/c3_full.npz: the oracle's C3 NCS solve (512^2, 720 x
725, the BASELINE iteration count) from the pinned parameters, for
test_gpu_solver.test_c3_full_against_golden.  Run once on a CPU host
(`python tests/golden/make_c3_golden.py`, ~10-20 min with OpenMP); the GPU
box never runs the oracle at this size.  Stores x (fp32), a seeded sample of
u, the record rows and the head of b (to check the instance is the same)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Prob  # noqa: E402
from paper_1810_13100_b200 import configs, instances  # noqa: E402


def main():
    P = Port()
    cfg = configs.get("c3")
    _, b = instances.make_instance(cfg, lambda im: P.radon_forward(im, cfg.angles, cfg.det))
    mask = instances.metric_mask(cfg)
    prob = Prob(cfg.kind_id, cfg.n, cfg.angles, cfg.det, cfg.alpha, cfg.beta, cfg.lam, b)
    t0 = time.time()
    o = P.solve(prob, cfg.gamma, mask, cfg.iters, record_every=cfg.iters // 4)
    dt = time.time() - t0
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(o.u.size, 20000, replace=False))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_full.npz")
    np.savez_compressed(out, x=o.x.astype(np.float32), u_idx=idx, u_sample=o.u.ravel()[idx],
                        rows=o.rows, b_head=np.ravel(b)[:4096], seconds=dt)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB) after {dt:.0f} s")


if __name__ == "__main__":
    main()
