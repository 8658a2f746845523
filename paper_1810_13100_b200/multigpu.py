"""Angle-sharded NCS over several GPUs of one node.

Each rank owns a contiguous block of projection angles: its rows of R, of the
sinogram dual u_s, of b and of the cached R x.  One step is

    phase A   partial A^T u = R_r^T u_s,r (+ w D^T u_g on rank 0)      [local]
    exchange  all-reduce of the N x N partial over NVLink (NCCL)
    phase B   replicated circulant solve + x update (identical on every rank),
              R_r x for the own angles, dual update of the own rays and of the
              replicated u_g                                            [local]

The gradient dual u_g and x are replicated and updated identically on every
rank, so they never need to move; the only collective per step is one
all-reduce of N^2 floats (1 MiB at 512^2) -- the "one all-reduce + replicated
FFT solve" variant of SURVEY.md §8f rank 3, which at 512^2 costs less than
reduce-scatter + 2 all-to-all + all-gather latencies.
"""
from __future__ import annotations

import json
import os
import time


def orbit_rep(t: int, n_angles: int) -> int:
    """Representative (in [0, A/4]) of angle t's dihedral orbit {t, t+A/2,
    A-t, A/2-t} (ncsg_internal.cuh orbit_rep)."""
    q = n_angles // 4
    if t <= q:
        return t
    if t < 2 * q:
        return 2 * q - t
    if t <= 3 * q:
        return t - 2 * q
    return n_angles - t


def orbit_owner(t: int, n_angles: int, world: int) -> int:
    """Rank owning angle t under orbit sharding (orbits round-robin by rep)."""
    return orbit_rep(t, n_angles) % world


def shard_angles(n_angles: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced angle block [begin, end) of `rank`."""
    base, rem = divmod(n_angles, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


class ShardedSolver:
    """One rank's share of an angle-sharded CT problem."""

    def __init__(self, cfg, b, mask, rank, world, device):
        import torch

        from . import ncsg

        self.rank, self.world = rank, world
        if cfg.angles % 4 == 0 and world > 1:
            # orbit sharding: every rank keeps the dihedral orbit forward
            self.range = (0, 0)
            self.prob = ncsg.ct_problem(cfg, b, mask=mask, orbit_shard=(rank, world),
                                        device=device)
        else:
            self.range = shard_angles(cfg.angles, world, rank)
            self.prob = ncsg.ct_problem(cfg, b, mask=mask, angle_range=self.range, device=device)
        self.prob.set_state()
        self.atu = torch.zeros(cfg.batch * cfg.n * cfg.n, dtype=torch.float32,
                               device=f"cuda:{device}")
        self.prob.bind_atu(self.atu)
        self.stream = torch.cuda.ExternalStream(self.prob.stream, device=f"cuda:{device}")

    def step(self, iters: int = 1):
        import torch
        import torch.distributed as dist

        with torch.cuda.stream(self.stream):
            for _ in range(iters):
                self.prob.phase_a()
                if self.world > 1:
                    dist.all_reduce(self.atu)
                self.prob.phase_b()

    def profile(self, steps: int):
        """Per-phase CUDA-event times (ms) of this rank over `steps` steps; the
        all-reduce falls between the adjoint and FFT phases."""
        self.prob.profile_begin()
        self.step(steps)
        return self.prob.profile_end()

    def objective(self):
        import torch
        import torch.distributed as dist

        f = torch.tensor(self.prob.objective(), dtype=torch.float64)
        if self.world > 1:
            f = f.cuda()
            dist.all_reduce(f)
            f = f.cpu()
        return f.numpy()
