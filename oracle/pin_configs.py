"""ORACLE / TEST INFRASTRUCTURE ONLY.

Pins alpha, beta, gamma, dc and the calibrated mask scale of every
BASELINE.json config with the oracle (see paper_1810_13100_b200/configs.py for
the rules) and writes paper_1810_13100_b200/pinned.json.  Run once:

    python oracle/pin_configs.py c1 c2 c3 c5      # minutes
    python oracle/pin_configs.py c4               # ~1 h on 8 cores
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


def pin(name, P):
    cfg = configs.base(name)
    a = ALPHA[cfg.kind]
    rec = {"alpha": a, "beta": a, "mask_samples": 8, "mask_seed": 0}
    t0 = time.time()
    if cfg.kind == "ct":
        one = np.ones((cfg.n, cfg.n))
        r1 = P.radon_forward(one, cfg.angles, cfg.det)
        rec["dc"] = float((r1 * r1).sum() / (cfg.n * cfg.n))
        rec["mask_scale"] = P.calibrate_scale(cfg.n, cfg.angles, cfg.det, 8, 0)
    c = configs.Config(**{**cfg.__dict__, "pinned": rec})
    mask = instances.metric_mask(c)
    b = np.zeros(c.m)
    prob = Prob(c.kind_id, c.n, c.angles, c.det, a, a, c.lam, b)
    est = P.screen(prob, 0.0, mask, iters=40, seed=0)
    rec["screen_lmax"] = est
    rec["gamma"] = MARGIN * est if est > 0 else 1e-3 * a
    rec["pin_seconds"] = time.time() - t0
    return rec


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c5"]
    P = Port()
    pins = {}
    if os.path.exists(configs.PINNED):
        pins = json.load(open(configs.PINNED))
    for name in names:
        rec = pin(name, P)
        print(name, rec, flush=True)
        pins = json.load(open(configs.PINNED)) if os.path.exists(configs.PINNED) else {}
        pins[name] = rec
        with open(configs.PINNED + ".tmp", "w") as f:
            json.dump(pins, f, indent=1, sort_keys=True)
        os.replace(configs.PINNED + ".tmp", configs.PINNED)


if __name__ == "__main__":
    main()
