"""Generates tests/golden/c5_full.npz: the oracle's C5 NCS solve (64
independent 256^2 problems, 360 x 363, the BASELINE 500 iterations each) for
test_gpu_solver.test_c5_all_problems_against_golden.  Run once on a CPU host
(`python tests/golden/make_c5_golden.py [processes]`, one single-threaded
oracle solve per problem, ~3 min each, the problems spread over processes);
the GPU box never runs the oracle at this size.  Stores per problem the
record rows (record_every = 250: iterations 250 and 500), x and u at a seeded
sample of 4096 pixels / 4096 dual entries (the same indices for every
problem) and the head of b (to check the instance is the same).  Follows
solve_template (solvers.cpp:267-337) through the C restatement
(ncs_oracle.c), pinned bitwise to the reference build (tests/test_oracle_pin.py)."""
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

N_SAMPLE = 4096


def solve_one(q):
    from oracle.oracle import Port, Prob
    from paper_1810_13100_b200 import configs, instances

    P = Port()
    cfg = configs.get("c5")
    _, b = instances.make_instance(
        cfg, lambda im: P.radon_forward(im, cfg.angles, cfg.det, threads=1), problem=q)
    mask = instances.metric_mask(cfg)
    prob = Prob(cfg.kind_id, cfg.n, cfg.angles, cfg.det, cfg.alpha, cfg.beta, cfg.lam, b)
    o = P.solve(prob, cfg.gamma, mask, cfg.iters, record_every=cfg.iters // 2, threads=1)
    return q, o.x.astype(np.float64).ravel(), o.u.ravel(), o.rows, np.ravel(b)[:256]


def main():
    from paper_1810_13100_b200 import configs

    procs = int(sys.argv[1]) if len(sys.argv) > 1 else max(1, os.cpu_count() - 1)
    cfg = configs.get("c5")
    t0 = time.time()
    with mp.get_context("spawn").Pool(procs) as pool:
        res = sorted(pool.map(solve_one, range(cfg.batch)), key=lambda r: r[0])
    dt = time.time() - t0
    rng = np.random.default_rng(0)
    x_idx = np.sort(rng.choice(res[0][1].size, N_SAMPLE, replace=False))
    u_idx = np.sort(rng.choice(res[0][2].size, N_SAMPLE, replace=False))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c5_full.npz")
    np.savez_compressed(
        out, x_idx=x_idx, u_idx=u_idx,
        x_sample=np.stack([r[1][x_idx] for r in res]).astype(np.float32),
        u_sample=np.stack([r[2][u_idx] for r in res]),
        x_norm=np.array([np.linalg.norm(r[1]) for r in res]),
        rows=np.stack([r[3] for r in res]), b_head=np.stack([r[4] for r in res]), seconds=dt)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB) after {dt:.0f} s")


if __name__ == "__main__":
    main()
