"""Breakdown of bench.py's e2e call for a config: problem creation (with the
library's NCSG_SETUP_TIMES stages on stderr), set_state, solve, download."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(name="c3"):
    import torch

    import bench
    from paper_1810_13100_b200 import configs, ncsg

    cfg = configs.get(name)
    torch.cuda.set_device(0)
    _, _, b, mask = bench.setup_problem(cfg, None)
    make = ncsg.ct_problem if cfg.kind == "ct" else ncsg.denoise_problem
    for k in range(3):
        t0 = time.perf_counter()
        p = make(cfg, b, mask=mask)
        t1 = time.perf_counter()
        p.set_state()
        t2 = time.perf_counter()
        r = p.solve(cfg.iters, record_every=cfg.iters)
        t3 = time.perf_counter()
        print(f"{name} run {k}: create {1e3 * (t1 - t0):.1f} ms, set_state {1e3 * (t2 - t1):.1f} ms, "
              f"solve+download {1e3 * (t3 - t2):.1f} ms ({cfg.iters} its)", flush=True)
        del p


if __name__ == "__main__":
    main(*sys.argv[1:])
