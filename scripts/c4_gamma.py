"""Power-method estimate of alpha*lambda_max(A^T A - C) for a pinned config
with more iterations than the 40-step screen (GPU), to check the pinned gamma
margin: python scripts/c4_gamma.py c4 40 100 200 400"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1810_13100_b200 import configs, instances, ncsg  # noqa: E402

cfg = configs.get(sys.argv[1])
mask = instances.metric_mask(cfg)
kind = ncsg.CT if cfg.kind == "ct" else ncsg.DENOISE
p = ncsg.Problem(kind, cfg.n, cfg.alpha, cfg.beta, cfg.lam, 0.0, np.zeros(cfg.m), mask=mask,
                 n_angles=cfg.angles, n_det=cfg.det)
print("pinned gamma", cfg.gamma, "pinned 40-step estimate", cfg.pinned["screen_lmax"])
for it in map(int, sys.argv[2:]):
    for seed in (0, 1):
        est, shift = p.screen(seed, it)
        print(f"iters {it} seed {seed}: estimate {est:.6g} (gamma/estimate {cfg.gamma / est:.4f})")
