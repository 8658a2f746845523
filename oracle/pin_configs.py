"""ORACLE / TEST INFRASTRUCTURE ONLY.

Pins alpha, beta, gamma, dc and the calibrated mask scale of every
BASELINE.json config with the oracle (see paper_1810_13100_b200/configs.py for
the rules) and writes paper_1810_13100_b200/pinned.json.  Run once:

    python oracle/pin_configs.py c1 c2 c3 c5      # minutes
    python scripts/pin_gamma_gpu.py c4            # C4's converged lambda_max on the GPU
                                                  # (300 oracle power steps at C4 ~ 4 h)
"""
import json
import os
import sys
import time

import numpy as np

sys.path[0] = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
from oracle.oracle import Port, Prob  # noqa: E402
from paper_1810_13100_b200 import configs, instances  # noqa: E402

ALPHA = {"ct": 0.1, "denoise": 1.0}
MARGIN = 1.2


LMAX_ITERS = 300  # power-method steps for gamma; the reference's screen uses 40


def pin(name, P, old=None):
    """dc, mask scale (skipped when `old` has them), the 40-step screen
    estimate (the reference's screen, kept for the setup-parity test) and the
    converged estimate lambda_max(alpha (A^T A - C)) that gamma is pinned to:
    40 power steps underestimate it badly (C3: 4543 vs 6797, C4: 14903 vs
    76153), and NCS with gamma below it diverges (C4 at iteration 107)."""
    cfg = configs.base(name)
    a = ALPHA[cfg.kind]
    rec = {"alpha": a, "beta": a, "mask_samples": 8, "mask_seed": 0}
    t0 = time.time()
    if cfg.kind == "ct":
        if old and "dc" in old and "mask_scale" in old:
            rec["dc"], rec["mask_scale"] = old["dc"], old["mask_scale"]
        else:
            one = np.ones((cfg.n, cfg.n))
            r1 = P.radon_forward(one, cfg.angles, cfg.det)
            rec["dc"] = float((r1 * r1).sum() / (cfg.n * cfg.n))
            rec["mask_scale"] = P.calibrate_scale(cfg.n, cfg.angles, cfg.det, 8, 0)
    c = configs.Config(**{**cfg.__dict__, "pinned": rec})
    mask = instances.metric_mask(c)
    b = np.zeros(c.m)
    prob = Prob(c.kind_id, c.n, c.angles, c.det, a, a, c.lam, b)
    if old and "screen_lmax" in old:
        rec["screen_lmax"] = old["screen_lmax"]
    else:
        rec["screen_lmax"] = P.screen(prob, 0.0, mask, iters=40, seed=0)
    est = P.screen(prob, 0.0, mask, iters=LMAX_ITERS, seed=0)
    rec["lmax"] = est
    rec["lmax_iters"] = LMAX_ITERS
    rec["lmax_source"] = "oracle"
    # A^T A - C == 0 up to roundoff (TV denoise: C = 1 + (beta/alpha)^2 Laplacian
    # is exactly A^T A) -> the PDHG-like floor gamma = 1e-3 alpha
    rec["gamma"] = MARGIN * est if est > 1e-9 else 1e-3 * a
    rec["pin_seconds"] = time.time() - t0
    return rec


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c5"]
    P = Port()
    pins = {}
    if os.path.exists(configs.PINNED):
        pins = json.load(open(configs.PINNED))
    for name in names:
        rec = pin(name, P, pins.get(name))
        print(name, rec, flush=True)
        pins = json.load(open(configs.PINNED)) if os.path.exists(configs.PINNED) else {}
        pins[name] = rec
        with open(configs.PINNED + ".tmp", "w") as f:
            json.dump(pins, f, indent=1, sort_keys=True)
        os.replace(configs.PINNED + ".tmp", configs.PINNED)


if __name__ == "__main__":
    main()
