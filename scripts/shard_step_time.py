"""Per-rank compute time of the sharded step on ONE GPU, for a scaling
projection (only one GPU is available to this build; no measured multi-GPU
number exists).  Rank 0 of a P-rank orbit-sharded problem steps with a
communicator whose collectives are no-ops (ncsg_comm_create_null), so the
timed stream holds exactly
rank 0's kernels of the real sharded step (its adjoint and forward over 1/P
of the orbits, the slab or replicated FFT, the dual update); the values are
meaningless, the work is the real work.  The exchange is then added from its
message sizes at the measured NVLink peer bandwidth (770 GB/s per direction,
B200_PROFILING.md) plus a per-collective latency, both stated in the output.

    python scripts/shard_step_time.py [c3 c4 ...]   ->  profiles/r2_shard_projection.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NVLINK_GBS = 770.0      # measured peer copy per direction (B200_PROFILING.md)
COLL_LAT_US = 8.0       # assumed per-collective launch + sync latency on NVSwitch


def main(names):
    import torch

    import bench
    from paper_1810_13100_b200 import configs, multigpu, ncsg

    out = {"method": __doc__.split("\n\n")[0], "nvlink_gbs": NVLINK_GBS,
           "collective_latency_us": COLL_LAT_US, "configs": {}}
    for name in names:
        cfg = configs.get(name)
        torch.cuda.set_device(0)
        _, _, b, mask = bench.setup_problem(cfg, None)
        rows = {}
        for world in (1, 2, 4, 8):
            xchg = multigpu.default_exchange(cfg.n, world) if world > 1 else "none"
            if cfg.batch > 1:  # replicas: batch / P independent problems per rank
                xchg = "replicas" if world > 1 else "none"
                share = cfg.batch // world
                p = ncsg.ct_problem(cfg, b[:share], mask=mask, batch=share)
            elif world == 1:
                p = ncsg.ct_problem(cfg, b, mask=mask)
            else:
                p = ncsg.ct_problem(cfg, b, mask=mask, orbit_shard=(0, world))
                comm = ncsg.Comm.null(0, world)
                p.set_comm(comm, ncsg.XCHG_ALLREDUCE if xchg == "allreduce" else ncsg.XCHG_SLAB)
            p.set_state()
            s = torch.cuda.ExternalStream(p.stream)
            p.step(3)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            k = 10 if cfg.n <= 1024 else 3
            with torch.cuda.stream(s):
                ev[0].record(s)
                p.step(k)
                ev[1].record(s)
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / k
            n2 = cfg.n * cfg.n
            units = cfg.batch // world if cfg.batch > 1 else 1  # problems per rank-step
            if world == 1 or cfg.batch > 1:
                comm_us = 0.0
            elif xchg == "allreduce":  # ring all-reduce: 2 (P-1)/P of 4 n^2 bytes
                comm_us = COLL_LAT_US + 2 * (world - 1) / world * 4 * n2 / (NVLINK_GBS * 1e3)
            else:  # reduce-scatter + 2 all-to-all + all-gather (slab design)
                rs = (world - 1) / world * 4 * n2
                a2a = 2 * (world - 1) / world ** 2 * 8 * cfg.n * (cfg.n // 2 + 1)
                ag = (world - 1) / world * 4 * n2
                comm_us = 4 * COLL_LAT_US + (rs + a2a + ag) / (NVLINK_GBS * 1e3)
            step_ms = ms + comm_us * 1e-3
            rate = 1000.0 / step_ms * (units * world if cfg.batch > 1 else 1)
            rows[world] = {"exchange": xchg, "rank_compute_ms": ms, "exchange_us_model": comm_us,
                           "projected_ms_per_step": step_ms, "projected_it_s": rate}
            print(name, world, xchg, f"compute {ms:.4f} ms + exchange {comm_us:.1f} us "
                  f"-> {rate:.0f} it/s (projected)", flush=True)
            del p
        out["configs"][name] = rows
    dst = os.environ.get("NCSG_OUT", "profiles/r2_shard_projection.json")
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c4"])
