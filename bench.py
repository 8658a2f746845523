#!/usr/bin/env python
"""NCS iterations/s on the BASELINE.json metric config (C3: 512^2 CT-TV, 720
angles x 725 detectors), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...     # the reference's own CPU NCS

A "step" is one NCS iteration (Engine::step, solvers.cpp:124-161) of the
config's problem with its state resident in HBM.  Each timed step is
bracketed by CUDA events on the solver's stream; L2 is flushed (a 256 MiB
write) between timed steps, outside the events.  `value` = K / sum(step
times).  `e2e` times the public API end to end (problem upload from host
memory, K steps, objective + state download).  Multi-GPU (torchrun): the
problem is sharded by projection angle; one NCCL all-reduce of the partial
A^T u per step, replicated circulant solve,
device time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NCS iters/s on 512² CT-TV (720 angles), 1/2/4/8 B200; % of HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def peaks():
    if os.path.exists(PEAKS):
        with open(PEAKS) as f:
            p = json.load(f)
        return p, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        mask = 0
        for r in self.rows:
            mask |= r[2]
        reasons = [name for bit, name in THROTTLE_BITS.items() if mask & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(sm)}


def kernels_per_step(prob):
    """Kernels of one eager step (counted by the library), the same set a
    graph replay of one step launches."""
    from paper_1810_13100_b200 import ncsg

    n0 = ncsg.launch_count()
    prob.step(1, graph=False)
    prob.sync()
    return ncsg.launch_count() - n0


def kernel_bytes(cfg, plan):
    """Per-launch algorithmic bytes of every phase of the step AS PLANNED
    (partial-slot and partial-image counts from the live plan,
    ncsg_problem_plan), whole batch, fp32, and the bound each is measured
    against:

      * projectors (forward R, adjoint R^T): on-chip gather, 16 B of texel
        traffic per bilinear sample (4 texels x 4 B), S samples
        per application -> shared-memory roofline;
      * streaming passes: HBM bytes their inputs and outputs must cross once.
    """
    N = cfg.n
    n = N * N
    spec = 8 * N * (N // 2 + 1)  # half spectrum, complex64
    B = max(1, int(plan["batch"]))
    m, g, P, F = plan["m0"], plan["g"], plan["bp_partials"], plan["fp_slots"]
    S = plan["samples"]
    ct = cfg.kind == "ct"
    out = {}
    if ct:
        out["adjoint"] = ("smem", 16 * S)
        out["forward"] = ("smem", 16 * S)
        if plan["orbit_forward"]:
            out["make_quad"] = ("hbm", 4 * n + 16 * n)  # x in, member cells out
    # r2c: A^T u assembly (partial images or the identity dual, D^T u_g) in,
    # half spectrum out
    r2c_in = 4 * (P * n if ct else n) + 4 * g
    out["fft_rows_r2c"] = ("hbm", r2c_in + spec)
    out["fft_cols"] = ("hbm", 3 * spec)  # spectrum r/w + filter
    out["fft_rows_c2r"] = ("hbm", spec + 4 * n * (3 + plan["transposed_copy"]))
    # dual: data block (CT: F partial slots + u r/w + ax r/w + b; denoise:
    # u r/w + b), gradient block u_g r/w, x and x_old
    data = 4 * (F * m + 5 * m) if ct else 4 * 3 * n
    dual = data + 4 * 2 * g + 4 * 2 * n
    if plan.get("dual_fused"):
        # DENOISE: the whole dual update runs inside the inverse row pass
        # (x and x_old are already on chip there)
        out["fft_rows_c2r"] = ("hbm", out["fft_rows_c2r"][1] + dual - 4 * 2 * n)
    else:
        out["dual_update"] = ("hbm", dual)
    return {k: (bound, B * v) for k, (bound, v) in out.items()}


def load_ncu(cfg_name):
    """Per-kernel ncu figures of this config's committed capture
    (profiles/ncu_<cfg>.json, written by scripts/ncu_summary.py), or {}."""
    path = os.path.join(ROOT, "profiles", f"ncu_{cfg_name}.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        d["_path"] = os.path.relpath(path, ROOT)
        return d
    except (OSError, ValueError):
        return {}


def setup_problem(cfg, nc, dev=0, angle_range=(0, 0)):
    """Seeded instances for every problem of the config (C5: 64 problems, one
    phantom/noise seed each), the GPU forward synthesising the sinograms."""
    from paper_1810_13100_b200 import instances, ncsg

    R = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det, device=dev) if cfg.kind == "ct" else None
    fwd = R.forward if R is not None else None
    xs, bs = zip(*[instances.make_instance(cfg, fwd, problem=q) for q in range(cfg.batch)])
    mask = instances.metric_mask(cfg)
    return R, np.stack(xs), np.stack(bs), mask


def _ref_problem_rate(args):
    """One process of the batched CPU baseline: per-iteration time of the
    reference's ncs_solve on problem `q` of the batch (module level so that
    multiprocessing can pickle it)."""
    name, q, b, mask, iters_hi, iters_lo = args
    from oracle.oracle import Prob, Ref
    from paper_1810_13100_b200 import configs

    cfg = configs.get(name)
    prob = Prob(cfg.kind_id, cfg.n, cfg.angles, cfg.det, cfg.alpha, cfg.beta, cfg.lam, b)
    impl = Ref()
    t = time.perf_counter()
    impl.solve(prob, cfg.gamma, mask, iters_lo)
    t_lo = time.perf_counter() - t
    t = time.perf_counter()
    impl.solve(prob, cfg.gamma, mask, iters_hi)
    t_hi = time.perf_counter() - t
    return max(1e-9, (t_hi - t_lo) / (iters_hi - iters_lo)), t_hi, t_lo


def cpu_reference_rate(cfg, b, mask, iters_hi=3, iters_lo=1):
    """The reference's own ncs_solve (oracle/_ref, compiled unchanged) timed on
    host cores: per-iteration time = (t(hi) - t(lo)) / (hi - lo), so solver
    setup, Engine::init and the final recorded seminorm cancel. The reference
    is serial, so one problem runs on one core; a batched config (C5) runs P
    of its problems as P processes on the host cores at once
    and reports the aggregate problem-iterations/s."""
    from oracle.oracle import REF_SO, Port, Prob, Ref

    if cfg.batch > 1 and os.path.exists(REF_SO):
        import multiprocessing as mp

        P = max(1, min(cfg.batch, len(os.sched_getaffinity(0))))
        m = cfg.angles * cfg.det if cfg.kind == "ct" else cfg.n * cfg.n
        bb = np.asarray(b).reshape(-1, m)  # the batch, or one instance (reference arm)
        jobs = [(cfg.name, q, bb[q % len(bb)], mask, iters_hi, iters_lo) for q in range(P)]
        with mp.get_context("spawn").Pool(P) as pool:
            res = pool.map(_ref_problem_rate, jobs)
        rate = sum(1.0 / r[0] for r in res)
        return {"value": rate, "unit": "it/s", "cores": P, "kind": "reference",
                "sample": f"{cfg.name}: problems 0..{P - 1} of the batch as {P} concurrent "
                          f"processes, each ncs_solve {iters_hi} vs {iters_lo} iterations "
                          f"(difference of wall times); aggregate problem-iterations/s"}

    b0 = np.asarray(b).reshape(cfg.batch, -1)[0]  # one problem
    prob = Prob(cfg.kind_id, cfg.n, cfg.angles, cfg.det, cfg.alpha, cfg.beta, cfg.lam, b0)
    if os.path.exists(REF_SO):
        impl, kind, cores = Ref(), "reference", 1
        run = lambda k: impl.solve(prob, cfg.gamma, mask, k)
    else:
        impl, kind = Port(), "port"
        cores = max(1, len(os.sched_getaffinity(0)))
        run = lambda k: impl.solve(prob, cfg.gamma, mask, k, threads=cores)
    t = time.perf_counter()
    run(iters_lo)
    t_lo = time.perf_counter() - t
    t = time.perf_counter()
    run(iters_hi)
    t_hi = time.perf_counter() - t
    per = max(1e-9, (t_hi - t_lo) / (iters_hi - iters_lo))
    out = {"value": 1.0 / per, "unit": "it/s", "cores": cores, "kind": kind,
           "sample": f"{cfg.name} ncs_solve {iters_hi} vs {iters_lo} iterations, "
                     f"difference of wall times ({t_hi:.1f}s, {t_lo:.1f}s), same b and mask"}
    if kind == "reference":
        # beside the serial reference: the OpenMP restatement (oracle/ncs_oracle.c,
        # ray- and angle-parallel projectors) on every host core, same sample
        try:
            port, nt = Port(), max(1, len(os.sched_getaffinity(0)))
            tp = []
            for k in (iters_lo, iters_hi):
                t = time.perf_counter()
                port.solve(prob, cfg.gamma, mask, k, threads=nt)
                tp.append(time.perf_counter() - t)
            out["openmp_port"] = {"value": 1.0 / max(1e-9, (tp[1] - tp[0]) / (iters_hi - iters_lo)),
                                  "unit": "it/s", "cores": nt, "kind": "port"}
        except Exception as e:  # noqa: BLE001 - extra information only
            out["openmp_port"] = {"value": None, "error": str(e)}
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1810_13100_b200 import instances
    from oracle.oracle import Port

    P = Port()
    x_true, b = instances.make_instance(cfg, lambda im: P.radon_forward(im, cfg.angles, cfg.det))
    mask = instances.metric_mask(cfg)
    k = max(2, min(args.steps, 4))
    cb = cpu_reference_rate(cfg, b, mask, iters_hi=k, iters_lo=1)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "it/s",
            "n_gpus": args.gpus, "steps": k - 1, "warmup": 0, "ms_per_step": 1000.0 / cb["value"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(cfg), "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload(cfg):
    return {"workload": f"{cfg.name}: {cfg.description}", "n": cfg.n, "angles": cfg.angles,
            "detectors": cfg.det, "lambda": cfg.lam, "alpha": cfg.alpha, "beta": cfg.beta,
            "gamma": cfg.gamma, "dc": cfg.dc, "mask_scale": cfg.mask_scale, "batch": cfg.batch,
            "l2": "flushed (256 MiB write) between timed steps, outside the events",
            "launch": "eager" if os.environ.get("NCSG_EAGER") == "1" else "CUDA graph per step",
            "parallelism": "angle-sharded" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "1 GPU"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_1810_13100_b200 import configs

    cfg = configs.get(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        bench_multi(args, cfg)
        return
    bench_single(args, cfg)


def roofline_of(cfg, plan, phase_avg, clocks):
    """Per-kernel roofline table and the headline entry (the dominant phase).

    achieved = algorithmic bytes per launch (kernel_bytes) / the phase's mean
    CUDA-event time on the solver stream; peak = measured HBM copy bandwidth
    (MEASURED_PEAKS.json) for streaming passes, 148 SM x 128 B/clk at the
    clock sampled during the timed region for the shared-memory gathers of
    the projectors; traffic / L2 hit rate = this config's ncu
    capture (dram__bytes_read + write, lts__t_sector_hit_rate) when committed."""
    pk, pk_kind = peaks()
    sm_mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    peaks_gbs = {"hbm": pk["hbm_gbs"], "smem": 148 * 128 * sm_mhz * 1e6 / 1e9}
    kinds = {"hbm": f"{pk_kind} (MEASURED_PEAKS.json hbm_gbs)",
             "smem": f"148 SM x 128 B/clk x {sm_mhz:.0f} MHz (sampled SM clock under load)"}
    prof = load_ncu(cfg.name)
    table = {}
    for k, (bound, nbytes) in kernel_bytes(cfg, plan).items():
        ms = phase_avg.get(k)
        if not ms:
            continue
        ach = nbytes / (ms * 1e-3) / 1e9
        row = {"bound": bound, "launch_ms": ms, "bytes_per_launch": nbytes, "achieved": ach,
               "peak": peaks_gbs[bound], "unit": "GB/s", "frac": ach / peaks_gbs[bound]}
        if k == "adjoint" and plan.get("adjoint_table_bytes"):
            # table mode: the window weights (geometry only, built per plan)
            # stream from HBM once per launch (from L2 when the table fits, C1/C5)
            tb = int(plan["adjoint_table_bytes"])
            row["table_bytes_per_launch"] = tb
            row["table_hbm_gbs"] = tb / (ms * 1e-3) / 1e9
            row["table_hbm_frac"] = row["table_hbm_gbs"] / peaks_gbs["hbm"]
        kp = prof.get("kernels", {}).get(k)
        if kp:
            row["traffic"] = kp.get("dram_bytes")
            row["l2_hit_rate"] = kp.get("l2_hit_rate")
            row["ncu_us"] = kp.get("duration_us")
        table[k] = row
    dom = max(table, key=lambda k: table[k]["launch_ms"])
    h = table[dom]
    return {"bound": h["bound"], "kernel": dom, "achieved": h["achieved"], "peak": h["peak"],
            "peak_kind": kinds[h["bound"]], "unit": "GB/s", "frac": h["frac"],
            "traffic": h.get("traffic"), "l2_hit_rate": h.get("l2_hit_rate"),
            "traffic_source": prof.get("_path"), "bytes_per_launch": h["bytes_per_launch"],
            "launch_ms": h["launch_ms"], "kernels": table,
            "note": "projectors: on-chip gather bound (16 B per bilinear sample, SURVEY §8d) "
                    "against shared-memory bandwidth; streaming passes: algorithmic HBM bytes "
                    "against the measured HBM copy peak"}


def bench_multi(args, cfg):
    """N > 1 (torchrun, one rank per GPU).  A single problem (C1-C4) is
    sharded by angle and steps inside libncsg with an NCCL communicator
    (slab FFT or all-reduce exchange, multigpu.default_exchange); a batched
    config (C5) runs replicas -- rank r solves its share of the independent
    problems.  Each rank times its own steps with CUDA events on its solver
    stream between barriers; the reported time is the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1810_13100_b200 import instances, multigpu, ncsg

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # NCSG_BENCH_GLOO=1: gloo process group and host-staged callback
    # collectives, all ranks on cuda:0 -- a functional run of this path on a
    # one-GPU box (the timing is then meaningless); default NCCL, one GPU per rank
    gloo = os.environ.get("NCSG_BENCH_GLOO") == "1"
    if gloo:
        local = 0
    torch.cuda.set_device(local)
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    R = ncsg.RadonMap(cfg.n, cfg.angles, cfg.det, device=local)
    mask = instances.metric_mask(cfg)
    if cfg.batch > 1:  # replicas: this rank's problems of the batch
        lo, hi = multigpu.replica_share(cfg.batch, world, rank)
        bs = np.stack([instances.make_instance(cfg, R.forward, problem=q)[1]
                       for q in range(lo, hi)])

        def make():
            p = ncsg.ct_problem(cfg, bs, mask=mask, batch=hi - lo, device=local)
            p.set_state()
            return p

        prob = make()
        units = hi - lo  # problems per step on this rank
        mode = f"replicas: problems {lo}..{hi - 1} of {cfg.batch} on this rank, no collective"
    else:
        x_true, b = instances.make_instance(cfg, R.forward)
        comm0 = multigpu.gloo_comm(rank, world) if gloo else None
        s = multigpu.ShardedSolver(cfg, b, mask, rank, world, local, comm=comm0)
        prob = s.prob
        units = 1
        mode = (f"{'orbit' if s.range == (0, 0) else 'angle'}-sharded, "
                + ("gloo host-staged callbacks (functional run, one GPU) " if gloo else "NCCL ")
                + {"slab": "reduce-scatter + slab FFT (2 all-to-all) + all-gather of x",
                   "p2p": "slab FFT with the reduce-scatter, both all-to-alls and the "
                          "all-gather fused into the producing kernels over NVLink peer "
                          "memory (CUDA IPC), stream-ordered barriers",
                   "allreduce": "all-reduce of A^T u + replicated FFT solve"}[s.exchange])

        def make():
            q = multigpu.ShardedSolver(cfg, b, mask, rank, world, local, comm=s.comm,
                                       exchange=s.exchange)
            return q.prob

    stream = torch.cuda.ExternalStream(prob.stream, device=f"cuda:{local}")
    prob.step(args.warmup)
    prob.sync()
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = ncsg.launch_count()
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                flush.fill_(float(k))
                starts[k].record(stream)
                prob.step(1)
                ends[k].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    launches = ncsg.launch_count() - launches0
    ms_local = sum(a.elapsed_time(e) for a, e in zip(starts, ends)) / args.steps
    dev = "cpu" if gloo else "cuda"
    t = torch.tensor([ms_local, float(units)], device=dev)
    tm = t.clone()
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm[0].item())
    tu = t.clone()
    dist.all_reduce(tu, op=dist.ReduceOp.SUM)
    total_units = float(tu[1].item())  # problems per step over all ranks
    prob.profile_begin()
    with torch.cuda.stream(stream):
        for k in range(min(args.steps, 10)):
            flush.fill_(float(k))
            prob.step(1)
    phase_ms, nprof = prob.profile_end()
    phase_avg = {k: v / max(1, nprof) for k, v in phase_ms.items()}
    torch.cuda.synchronize()
    # e2e: the public API on every rank -- problem creation from host arrays
    # (its shard or its replicas), solve of the config's iteration count with
    # the cross-rank records, state back to host; wall clock, max over ranks
    dist.barrier()
    t0 = time.perf_counter()
    p2 = make()
    res = p2.solve(cfg.iters, record_every=cfg.iters)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    e2e_s = float(dt.item())
    plan = prob.plan()
    if rank == 0:
        clocks = clk.summary()
        value = 1000.0 / ms * total_units
        m_own = plan["m0"]  # rays of the offsets uploaded per problem (sinogram size)
        line = {"metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True,
                "scaling": "weak" if cfg.batch > 1 else "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": workload(cfg),
                "roofline": roofline_of(cfg, plan, phase_avg, clocks),
                "phases_ms_rank0": phase_avg, "gpu_launches": launches, "clocks": clocks,
                "exchange": mode,
                "e2e": {"value": cfg.iters * total_units / e2e_s, "unit": "it/s",
                        "h2d_bytes_per_step": (8 * m_own * units
                                               + 2 * 8 * (cfg.n // 2 + 1) * cfg.n) / cfg.iters,
                        "d2h_bytes_per_step": 8 * (res.x.size + res.u.size) / cfg.iters,
                        "iters": cfg.iters, "seconds": e2e_s,
                        "note": "per rank: problem create + solve(iters) with cross-rank "
                                "records + state download; max over ranks"}}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def bench_single(args, cfg):
    import torch

    from paper_1810_13100_b200 import instances, ncsg

    torch.cuda.set_device(0)
    R, x_true, b, mask = setup_problem(cfg, None)
    prob = ncsg.ct_problem(cfg, b, mask=mask) if cfg.kind == "ct" else ncsg.denoise_problem(
        cfg, b, mask=mask)
    prob.set_state()
    # the step as a captured CUDA graph (ncsg_step_graph: one graph launch per
    # step, its kernels chained by programmatic dependent launch); NCSG_EAGER=1
    # times the eager per-kernel launches instead
    graph = os.environ.get("NCSG_EAGER") != "1"
    prob.step(args.warmup, graph=False)
    prob.step(1, graph=graph)  # capture outside the timed region
    prob.sync()
    stream = torch.cuda.ExternalStream(prob.stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    launches0 = ncsg.launch_count()
    with ClockSampler(0) as clk:
        time.sleep(0.3)
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                flush.fill_(float(k))
                starts[k].record(stream)
                prob.step(1, graph=graph)
                ends[k].record(stream)
        torch.cuda.synchronize()
    launches = ncsg.launch_count() - launches0
    if graph:  # graph replays do not pass through the counted launch calls
        launches = args.steps * kernels_per_step(prob)
    prob.sync()
    # per-phase CUDA events in a separate pass, so they do not perturb `value`
    prob.profile_begin()
    with torch.cuda.stream(stream):
        for k in range(min(args.steps, 10)):
            flush.fill_(float(k))
            prob.step(1)
    phase_ms, nprof = prob.profile_end()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = sum(step_ms) / len(step_ms)
    value = 1000.0 / ms * cfg.batch if cfg.batch > 1 else 1000.0 / ms
    phase_avg = {k: v / max(1, nprof) for k, v in phase_ms.items()}

    clocks = clk.summary()
    plan = prob.plan()
    S = plan["samples"]
    roofline = roofline_of(cfg, plan, phase_avg, clocks)

    line = {"metric": METRIC, "value": value, "unit": "it/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload(cfg), "roofline": roofline,
            "phases_ms": phase_avg, "gpu_launches": launches, "clocks": clocks,
            "samples_per_projection": S}
    # the timed problem, its events and the flush buffer are released before the
    # end-to-end calls (each creates its own problem, as a user's call would)
    del prob, stream, starts, ends, flush, R
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if not args.no_e2e:
        line["e2e"] = e2e_rate(cfg, b, mask, args.steps)
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_reference_rate(cfg, b, mask)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)


def e2e_rate(cfg, b, mask, steps):
    """Public API end to end, the call a user makes for this config: host b +
    mask -> ncsg.Problem (geometry replay, pinv filter, H2D uploads), one
    ncs_solve of the config's iteration count (record_every = max_iters, the
    reference's bench protocol), objective + x/u back to host
    (D2H).  Wall clock around all of it."""
    from paper_1810_13100_b200 import ncsg

    iters = cfg.iters
    make = ncsg.ct_problem if cfg.kind == "ct" else ncsg.denoise_problem
    runs = []
    for k in range(6):  # one untimed warm-up call, then the median of five
        t = time.perf_counter()
        prob = make(cfg, b, mask=mask)
        prob.set_state()
        res = prob.solve(iters, record_every=iters)
        if k:
            runs.append(time.perf_counter() - t)
        del prob
    dt = statistics.median(runs)
    nk = cfg.n // 2 + 1
    m = cfg.angles * cfg.det
    h2d = 4 * b.size + 2 * 8 * nk * cfg.n + 8 * m  # b, two half-spectrum filters, ray table
    d2h = 4 * (res.x.size + res.u.size) + res.rows.size * 8
    assert np.all(np.isfinite(res.objective))
    return {"value": iters * cfg.batch / dt, "unit": "it/s", "h2d_bytes_per_step": h2d / iters,
            "d2h_bytes_per_step": d2h / iters, "iters": iters, "seconds": dt,
            "seconds_runs": runs,
            "note": f"ncsg.Problem create + set_state + solve({iters}) + state/records download, "
                    "wall clock, median of 5 calls after one untimed warm-up call"}


if __name__ == "__main__":
    main()
