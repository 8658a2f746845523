"""One NCS step of a config under the CUDA profiler range, for ncu captures
(`ncu --profile-from-start off ... python scripts/ncu_step.py --config c3`):
problem set up from the seeded instance, a few warm steps, then exactly one
step between cudaProfilerStart/Stop."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--warm", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    from paper_1810_13100_b200 import configs, ncsg

    cfg = configs.get(args.config)
    torch.cuda.set_device(0)
    _, _, b, mask = bench.setup_problem(cfg, None)
    prob = ncsg.ct_problem(cfg, b, mask=mask) if cfg.kind == "ct" else ncsg.denoise_problem(
        cfg, b, mask=mask)
    prob.set_state()
    prob.step(args.warm)
    prob.sync()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    prob.step(1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    prob.sync()
    print("ok", args.config, prob.plan())


if __name__ == "__main__":
    main()
