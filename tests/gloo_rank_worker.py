"""One rank of the two-process sharded-NCS test (tests/test_gpu_multi.py::
test_two_process_gloo_callbacks): both processes share cuda:0, each owns an
orbit shard, and the library's collectives go through Python callbacks that
stage the device buffers on the host and exchange them with torch.distributed
(gloo over 127.0.0.1); in the "p2p" mode the fused exchange stores straight
into the other process's buffers through CUDA IPC mappings.  Writes rank r's
final x and record rows to <out>/rank<r>.npz."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(rank, world, port, out, mode="slab"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from oracle.oracle import Port
    from paper_1810_13100_b200 import ncsg
    from test_gpu_solver import small_ct

    # "nccl-<exchange>": one GPU per rank and the library's NCCL transport
    # (test_two_gpu_nccl_matches_unsharded; needs >= `world` GPUs)
    nccl = mode.startswith("nccl-")
    mode = mode[5:] if nccl else mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1810_13100_b200 import multigpu

    port_ = Port()
    prob, mask, gamma = small_ct(port_, n=64, A=48)
    dev = rank if nccl else 0
    torch.cuda.set_device(dev)
    p = ncsg.Problem(ncsg.CT, prob.n, prob.alpha, prob.beta, prob.lam, gamma, prob.b, mask=mask,
                     n_angles=prob.angles, n_det=prob.det, orbit_shard=(rank, world), device=dev)
    # NCCL over NVLink, or host-staged gloo collectives on a shared GPU
    comm = multigpu.nccl_comm(rank, world, dev) if nccl else multigpu.gloo_comm(rank, world)
    p.set_state()
    p.set_comm(comm, {"p2p": ncsg.XCHG_P2P, "slab": ncsg.XCHG_SLAB,
                      "allreduce": ncsg.XCHG_ALLREDUCE}[mode])
    res = p.solve(30, record_every=10)
    np.savez(os.path.join(out, f"rank{rank}.npz"), x=res.x, rows=res.rows)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4],
         sys.argv[5] if len(sys.argv) > 5 else "slab")
