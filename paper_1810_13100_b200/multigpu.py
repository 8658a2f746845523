"""Sharded NCS over the GPUs of one node.

One process per GPU.  A single large problem is sharded by projection angle
(whole dihedral orbits per rank when the angle count is a multiple of 4, so
every shard keeps the orbit forward; contiguous angle blocks otherwise): each
rank owns its rows of R, of the sinogram dual u_s, of b and of the cached
R x.  The step runs inside libncsg with an NCCL communicator
(ncsg_problem_set_comm), in one of two exchange modes:

  p2p        the slab decomposition below with every exchange fused into its
             producing kernel over NVLink peer memory (CUDA IPC mappings):
             the A^T u assembly stores rows into their owners' slots, the row
             FFT stores bin blocks into their column owners, the column pass
             stores back, the x update stores its rows into every rank's
             image; a stream-ordered NCCL barrier between the kernels
             (default for large N; falls back to slab if peer mappings fail);
  slab       partial A^T u -> NCCL reduce-scatter into N/P-row slabs -> row
             FFT of the own slab -> all-to-all -> column FFT . filter .
             inverse -> all-to-all -> inverse rows + x update of the own rows
             -> all-gather of x (north_star's design with NCCL collectives);
  allreduce  one all-reduce of the N^2 partial, replicated circulant solve
             (latency-bound sizes such as 512^2).

Batched configs (C5) run as replicas: rank r solves its share of the
independent problems, no collective in the step.
"""
from __future__ import annotations

import os


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


def replica_share(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Problems [begin, end) of a batched config solved by `rank` (C5)."""
    return shard_angles(batch, world, rank)


def default_exchange(n: int, world: int) -> str:
    """p2p (the fused slab exchange) where the image splits into power-of-two
    slabs, at most 8 ranks and large enough for the slab FFT to pay
    (N >= 1024), else the all-reduce; NCSG_XCHG=slab|p2p|allreduce overrides."""
    env = os.environ.get("NCSG_XCHG")
    if env in ("slab", "allreduce", "p2p"):
        return env
    r = n // world
    ok = n % world == 0 and r % 2 == 0 and (r & (r - 1)) == 0
    return "p2p" if ok and n >= 1024 and world <= 8 else "allreduce"


def nccl_comm(rank: int, world: int, device: int):
    """An ncsg NCCL communicator; the unique id travels over the already
    initialised torch.distributed process group."""
    import torch.distributed as dist

    from . import ncsg

    obj = [ncsg.Comm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return ncsg.Comm.nccl(obj[0], rank, world, device)


class ShardedSolver:
    """One rank's share of an angle-sharded CT problem, stepping inside
    libncsg with a communicator (NCCL by default)."""

    def __init__(self, cfg, b, mask, rank, world, device, comm=None, exchange=None):
        import torch

        from . import ncsg

        self.rank, self.world = rank, world
        if cfg.angles % 4 == 0 and world > 1:
            # orbit sharding: every rank keeps the dihedral orbit forward
            self.range = (0, 0)
            self.prob = ncsg.ct_problem(cfg, b, mask=mask, orbit_shard=(rank, world),
                                        device=device)
        else:
            self.range = shard_angles(cfg.angles, world, rank) if world > 1 else (0, 0)
            self.prob = ncsg.ct_problem(cfg, b, mask=mask, angle_range=self.range, device=device)
        self.prob.set_state()
        self.exchange = exchange or default_exchange(cfg.n, world)
        if world > 1:
            self.comm = comm if comm is not None else nccl_comm(rank, world, device)
            modes = {"slab": ncsg.XCHG_SLAB, "p2p": ncsg.XCHG_P2P,
                     "allreduce": ncsg.XCHG_ALLREDUCE}
            try:
                self.prob.set_comm(self.comm, modes[self.exchange])
            except (ncsg.NcsgError, ValueError):
                if self.exchange != "p2p":
                    raise
                self.exchange = "slab"  # no peer mappings on this node: NCCL collectives
                self.prob.set_comm(self.comm, ncsg.XCHG_SLAB)
        self.stream = torch.cuda.ExternalStream(self.prob.stream, device=f"cuda:{device}")

    def step(self, iters: int = 1, graph: bool = False):
        self.prob.step(iters, graph=graph)

    def profile(self, steps: int):
        """Per-phase CUDA-event times (ms) of this rank over `steps` steps; the
        collectives fall inside the FFT phases (slab) or between the adjoint
        and the FFT rows (all-reduce)."""
        self.prob.profile_begin()
        self.step(steps)
        return self.prob.profile_end()

    def objective(self):
        """The whole problem's objective (cross-rank sums inside the library)."""
        return self.prob.objective()

    def solve(self, max_iters: int, record_every: int | None = None):
        return self.prob.solve(max_iters, record_every=record_every)


def gloo_comm(rank: int, world: int):
    """An ncsg communicator whose collectives are host-staged torch.distributed
    (gloo) calls: functional multi-process runs with several ranks on one GPU
    (tests, the bench's NCSG_BENCH_GLOO mode)."""
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    from . import ncsg

    import nvidia.cuda_runtime

    lib = os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib", "libcudart.so.12")
    rt = C.CDLL(lib)
    rt.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    types = {ncsg.F32: (np.float32, 4), ncsg.F64: (np.float64, 8), ncsg.I32: (np.int32, 4)}

    def down(ptr, count, dt=np.float32, es=4):
        h = np.empty(count, dt)
        assert rt.cudaMemcpy(h.ctypes.data, ptr, count * es, 2) == 0
        return h

    def up(ptr, h):
        h = np.ascontiguousarray(h)
        assert rt.cudaMemcpy(ptr, h.ctypes.data, h.nbytes, 1) == 0
        assert rt.cudaDeviceSynchronize() == 0

    def all_reduce(buf, count, dt, op):
        npt, es = types[dt]
        t = torch.from_numpy(down(buf, count, npt, es))
        dist.all_reduce(t, op={ncsg.SUM: dist.ReduceOp.SUM, ncsg.MIN: dist.ReduceOp.MIN,
                               ncsg.MAX: dist.ReduceOp.MAX}[op])
        up(buf, t.numpy())

    def gather_all(snd, count):
        t = torch.from_numpy(down(snd, count))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [q.numpy() for q in parts]

    def reduce_scatter(snd, rcv, count):
        t = torch.from_numpy(down(snd, count * world))
        dist.all_reduce(t)
        up(rcv, t.numpy()[rank * count:(rank + 1) * count])

    def all_gather(snd, rcv, count):
        up(rcv, np.concatenate(gather_all(snd, count)))

    def all_to_all(snd, rcv, count):
        parts = gather_all(snd, count * world)
        up(rcv, np.concatenate([parts[r][rank * count:(rank + 1) * count] for r in range(world)]))

    return ncsg.Comm.callbacks(rank, world, all_reduce, reduce_scatter, all_gather, all_to_all)
