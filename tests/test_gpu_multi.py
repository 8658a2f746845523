"""The sharded NCS iteration inside libncsg (ncsg_problem_set_comm) on one GPU:
P ranks as an in-process group (one host thread per rank, exchanging through
host memory -- the ranks' kernels never wait on each other), each rank a
problem holding its angle or orbit shard.  Slab mode runs the reduce-scatter
of the partial A^T u into N/P-row slabs, the slab FFT with its two
all-to-all transposes and the all-gather of x (north_star's design); the
all-reduce mode the replicated solve.  Both must reproduce the unsharded
engine (validated against the oracle in test_gpu_solver.py): Engine::step,
solvers.cpp:124-161, with StackedMap::adjoint's sum (linear_map.cpp:47-55)
taken across ranks."""
import os
import threading

import numpy as np
import pytest

from test_gpu_solver import check_run, gpu_problem, rel, small_ct

pytestmark = pytest.mark.gpu


def shard_angles(n_angles, world, rank):
    base, rem = divmod(n_angles, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def run_ranks(fns):
    out = [None] * len(fns)
    err = []

    def go(r):
        try:
            out[r] = fns[r]()
        except Exception as e:  # surfaced after the join
            err.append(e)

    th = [threading.Thread(target=go, args=(r,)) for r in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def sharded_problems(ncsg, prob, gamma, mask, P, shard, mode):
    comms = ncsg.Comm.local_group(P)
    probs = []
    for r in range(P):
        kw = {"orbit_shard": (r, P)} if shard == "orbit" else {
            "angle_range": shard_angles(prob.angles, P, r)}
        p = ncsg.Problem(ncsg.CT, prob.n, prob.alpha, prob.beta, prob.lam, gamma, prob.b,
                         mask=mask, n_angles=prob.angles, n_det=prob.det, **kw)
        p.set_state()
        probs.append(p)
    # attaching is collective for the P2P mode (the ranks exchange their
    # buffers' peer views): every rank on its own thread
    x = {"slab": ncsg.XCHG_SLAB, "p2p": ncsg.XCHG_P2P, "allreduce": ncsg.XCHG_ALLREDUCE}[mode]
    run_ranks([lambda p=p, c=c: p.set_comm(c, x) for p, c in zip(probs, comms)])
    return probs, comms


@pytest.mark.parametrize("P,shard,mode", [(2, "orbit", "slab"), (4, "orbit", "slab"),
                                          (2, "orbit", "allreduce"), (2, "contig", "slab"),
                                          (4, "contig", "allreduce"), (8, "orbit", "slab"),
                                          (2, "orbit", "p2p"), (4, "orbit", "p2p"),
                                          (8, "orbit", "p2p"), (4, "contig", "p2p")])
def test_sharded_solve_matches_unsharded(ncsg, port, P, shard, mode):
    prob, mask, gamma = small_ct(port, n=64, A=48)
    ref = gpu_problem(ncsg, prob, gamma, mask).solve(40, record_every=10)
    probs, comms = sharded_problems(ncsg, prob, gamma, mask, P, shard, mode)
    res = run_ranks([lambda p=p: p.solve(40, record_every=10) for p in probs])
    for r in range(P):
        assert rel(res[r].x[0], ref.x[0]) <= 1e-5, (r, rel(res[r].x[0], ref.x[0]))
        np.testing.assert_array_equal(res[r].rows[0][:, 0], ref.rows[0][:, 0])
        f, fr = res[r].rows[0][:, 1], ref.rows[0][:, 1]
        assert np.max(np.abs(f - fr) / np.abs(fr)) <= 1e-5
        s, sr = res[r].rows[0][1:, 3], ref.rows[0][1:, 3]
        assert np.max(np.abs(s - sr) / np.abs(sr)) <= 1e-4
    # every rank holds the same replicated x
    for r in range(1, P):
        np.testing.assert_array_equal(res[r].x, res[0].x)


def test_sharded_solve_against_oracle(ncsg, port):
    # the slab-sharded engine against the fp64 oracle at the configured bar
    prob, mask, gamma = small_ct(port, n=64, A=48)
    o = port.solve(prob, gamma, mask, 60, record_every=20)
    probs, comms = sharded_problems(ncsg, prob, gamma, mask, 4, "orbit", "p2p")
    res = run_ranks([lambda p=p: p.solve(60, record_every=20) for p in probs])
    assert rel(res[0].x[0], o.x) <= 1e-4
    oo = o.rows[:, 1]
    assert np.max(np.abs(res[0].rows[0][:, 1] - oo) / np.abs(oo)) <= 1e-4


def test_sharded_steps_and_divergence_flags(ncsg, port):
    # ncsg_step on a sharded problem with a communicator == unsharded steps,
    # and a NaN in one rank's own rays is reported by every rank (flags are
    # reduced across ranks), with the absolute iteration
    prob, mask, gamma = small_ct(port, n=64, A=48)
    ref = gpu_problem(ncsg, prob, gamma, mask)
    ref.step(7)
    xr, _, _ = ref.get_state()
    probs, comms = sharded_problems(ncsg, prob, gamma, mask, 2, "orbit", "slab")

    def steps(p):
        p.step(7)
        p.sync()
        return p.get_state()[0]

    xs = run_ranks([lambda p=p: steps(p) for p in probs])
    for x in xs:
        assert rel(x, xr) <= 1e-5
    b = np.array(prob.b, dtype=np.float64, copy=True)
    b.ravel()[5] = np.nan  # angle 0: owned by rank 0 under orbit sharding
    from oracle.oracle import Prob

    bad = Prob(prob.kind, prob.n, prob.angles, prob.det, prob.alpha, prob.beta, prob.lam, b)
    probs, comms = sharded_problems(ncsg, bad, gamma, mask, 2, "orbit", "slab")

    def diverge(p):
        p.set_state(iter_=3)
        p.step(2)
        try:
            p.sync()
        except ncsg.DivergenceError as e:
            return e.iter, str(e)
        return None

    out = run_ranks([lambda p=p: diverge(p) for p in probs])
    for r in range(2):
        assert out[r] is not None and out[r][0] == 4 and "dual iterate became NaN" in out[r][1]


def test_slab_mode_validation(ncsg, port):
    prob, mask, gamma = small_ct(port, n=32, A=24)
    comms = ncsg.Comm.local_group(3)  # 32 rows do not split into 3 even power-of-two slabs
    p = ncsg.Problem(ncsg.CT, prob.n, prob.alpha, prob.beta, prob.lam, gamma, prob.b, mask=mask,
                     n_angles=prob.angles, n_det=prob.det, angle_range=(0, 8))
    with pytest.raises(ValueError, match="slab FFT"):
        p.set_comm(comms[0], ncsg.XCHG_SLAB)
    q = ncsg.Problem(ncsg.CT, prob.n, prob.alpha, prob.beta, prob.lam, gamma, prob.b, mask=mask,
                     n_angles=prob.angles, n_det=prob.det, orbit_shard=(1, 2))
    with pytest.raises(ValueError, match="rank / size"):
        q.set_comm(comms[0], ncsg.XCHG_ALLREDUCE)


@pytest.mark.parametrize("mode", ["slab", "p2p"])
def test_two_process_gloo_callbacks(ncsg, port, tmp_path, mode):
    # two processes (one CUDA context each on cuda:0), the library's
    # collectives through Python callbacks over torch.distributed gloo on
    # host-staged buffers: the real CUDA phases of the slab-sharded step
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    free = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    procs = [subprocess.Popen([sys.executable, os.path.join(here, "gloo_rank_worker.py"), str(r),
                               "2", str(free), str(tmp_path), mode]) for r in range(2)]
    for q in procs:
        assert q.wait(timeout=600) == 0
    prob, mask, gamma = small_ct(port, n=64, A=48)
    ref = gpu_problem(ncsg, prob, gamma, mask).solve(30, record_every=10)
    for r in range(2):
        d = np.load(os.path.join(str(tmp_path), f"rank{r}.npz"))
        assert rel(d["x"][0], ref.x[0]) <= 1e-5
        f, fr = d["rows"][0][:, 1], ref.rows[0][:, 1]
        assert np.max(np.abs(f - fr) / np.abs(fr)) <= 1e-5


@pytest.mark.parametrize("mode", ["nccl-slab", "nccl-p2p", "nccl-allreduce"])
def test_two_gpu_nccl_matches_unsharded(ncsg, port, tmp_path, mode):
    # one process per GPU, the library's NCCL transport (and the fused P2P
    # exchange over CUDA IPC peer memory) across two real devices; skipped on
    # one-GPU boxes, where the gloo test above runs the same phases
    if ncsg.device_count() < 2:
        pytest.skip("needs two GPUs")
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    free = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    procs = [subprocess.Popen([sys.executable, os.path.join(here, "gloo_rank_worker.py"), str(r),
                               "2", str(free), str(tmp_path), mode]) for r in range(2)]
    for q in procs:
        assert q.wait(timeout=600) == 0
    prob, mask, gamma = small_ct(port, n=64, A=48)
    ref = gpu_problem(ncsg, prob, gamma, mask).solve(30, record_every=10)
    for r in range(2):
        d = np.load(os.path.join(str(tmp_path), f"rank{r}.npz"))
        assert rel(d["x"][0], ref.x[0]) <= 1e-5


@pytest.mark.parametrize("mode", ["slab", "allreduce"])
def test_nccl_transport_single_rank(ncsg, port, mode):
    # the NCCL transport itself (dlopen'd libnccl, ncclCommInitRank, reduce-
    # scatter, grouped send/recv all-to-all, in-place all-gather, all-reduce)
    # on a one-rank communicator: the sharded step with P = 1 must equal the
    # plain engine, and it is graph-capturable
    import torch  # noqa: F401  (loads the process's NCCL first)

    prob, mask, gamma = small_ct(port, n=64, A=48)
    ref = gpu_problem(ncsg, prob, gamma, mask).solve(20, record_every=10)
    comm = ncsg.Comm.nccl(ncsg.Comm.nccl_unique_id(), 0, 1, 0)
    p = gpu_problem(ncsg, prob, gamma, mask)
    p.set_comm(comm, ncsg.XCHG_SLAB if mode == "slab" else ncsg.XCHG_ALLREDUCE)
    g = p.solve(20, record_every=10)
    assert rel(g.x[0], ref.x[0]) <= 1e-6
    q = gpu_problem(ncsg, prob, gamma, mask)
    q.set_comm(comm, ncsg.XCHG_SLAB if mode == "slab" else ncsg.XCHG_ALLREDUCE)
    q.step(5, graph=True)
    q.step(5, graph=True)
    r = gpu_problem(ncsg, prob, gamma, mask)
    r.step(10)
    assert rel(q.get_state()[0], r.get_state()[0]) <= 1e-6
