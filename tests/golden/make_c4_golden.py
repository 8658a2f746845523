"""Generates tests/golden/c4_full.npz: the oracle's C4 NCS solve (2048^2,
2048 x 2897, the BASELINE 300 iterations) from the pinned parameters, for
test_gpu_solver.test_c4_full_against_golden.  Run once on a CPU host
(`python tests/golden/make_c4_golden.py [threads]`: 11 287 s with 7 OpenMP
threads, ~10 s per iteration with the 16 host threads of a GPU box --
scripts/gpu/c4_golden.sh); the GPU box never runs the oracle solve at this
size, only the one oracle forward that rebuilds b.  Stores x (fp32), a seeded
sample of u, the record rows (record_every = 75, solve_template's rows) and the
head of b (to check the instance is the same).  Follows solve_template
(solvers.cpp:267-337) through the C restatement (ncs_oracle.c), which is
pinned bitwise to the reference build at C1/C3 (tests/test_oracle_pin.py)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Prob  # noqa: E402
from paper_1810_13100_b200 import configs, instances  # noqa: E402


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else None
    P = Port()
    cfg = configs.get("c4")
    _, b = instances.make_instance(
        cfg, lambda im: P.radon_forward(im, cfg.angles, cfg.det, threads=threads))
    mask = instances.metric_mask(cfg)
    prob = Prob(cfg.kind_id, cfg.n, cfg.angles, cfg.det, cfg.alpha, cfg.beta, cfg.lam, b)
    t0 = time.time()
    # NCS_GOLDEN_ITERS: a shorter pin of the same instance (c4_<iters>.npz)
    iters = int(os.environ.get("NCS_GOLDEN_ITERS", cfg.iters))
    o = P.solve(prob, cfg.gamma, mask, iters, record_every=max(1, iters // 4), threads=threads)
    dt = time.time() - t0
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(o.u.size, 100000, replace=False))
    out = os.environ.get("NCS_GOLDEN_OUT") or os.path.join(
        os.path.dirname(os.path.abspath(__file__)), "c4_full.npz")
    np.savez_compressed(out, x=o.x.astype(np.float32), u_idx=idx, u_sample=o.u.ravel()[idx],
                        rows=o.rows, b_head=np.ravel(b)[:4096], seconds=dt)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB) after {dt:.0f} s")


if __name__ == "__main__":
    main()
