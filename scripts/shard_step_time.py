"""Per-rank step time of the sharded C3 problem on ONE GPU (phase A + phase B
of a single shard, no collective): what each of N GPUs computes per step,
for contiguous-angle vs orbit sharding.  Projects strong scaling; the NCCL
all-reduce of N^2 floats per step comes on top.
    python scripts/shard_step_time.py"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1810_13100_b200 import configs, instances, multigpu, ncsg  # noqa: E402

cfg = configs.get("c3")
R = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det)
_, b = instances.make_instance(cfg, R.forward)
mask = instances.metric_mask(cfg)
out = {}
for world in (1, 2, 4, 8):
    for mode in ("orbit", "contiguous"):
        if world == 1 and mode == "contiguous":
            continue
        if mode == "orbit" and world > 1:
            p = ncsg.ct_problem(cfg, b, mask=mask, orbit_shard=(0, world))
        else:
            r = multigpu.shard_angles(cfg.angles, world, 0)
            p = ncsg.ct_problem(cfg, b, mask=mask, angle_range=r if world > 1 else (0, 0))
        atu = torch.zeros(cfg.n * cfg.n, device="cuda")
        p.bind_atu(atu)
        p.set_state()
        s = torch.cuda.ExternalStream(p.stream)
        for _ in range(3):
            p.phase_a()
            p.phase_b()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            ev[0].record(s)
            for _ in range(20):
                p.phase_a()
                p.phase_b()
            ev[1].record(s)
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 20
        out[f"{mode}_{world}"] = ms
        print(mode, world, f"{ms:.4f} ms/step per rank", flush=True)
print(json.dumps(out))
