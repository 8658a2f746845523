"""One rank of the two-process sharded-NCS test (tests/test_gpu_multi.py::
test_two_process_gloo_callbacks): both processes share cuda:0, each owns an
orbit shard, and the library's collectives go through Python callbacks that
stage the device buffers on the host and exchange them with torch.distributed
(gloo over 127.0.0.1).  Writes rank r's final x and record rows to
<out>/rank<r>.npz."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def cudart():
    import nvidia.cuda_runtime

    d = os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib")
    rt = C.CDLL(os.path.join(d, "libcudart.so.12"))
    rt.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    return rt


def main(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from oracle.oracle import Port
    from paper_1810_13100_b200 import ncsg
    from test_gpu_solver import small_ct

    dist.init_process_group("gloo", rank=rank, world_size=world)
    rt = cudart()
    H2D, D2H = 1, 2
    dtypes = {ncsg.F32: (np.float32, 4), ncsg.F64: (np.float64, 8), ncsg.I32: (np.int32, 4)}

    def down(ptr, count, dt=np.float32, es=4):
        h = np.empty(count, dt)
        assert rt.cudaMemcpy(h.ctypes.data, ptr, count * es, D2H) == 0
        return h

    def up(ptr, h):
        # a pageable H2D cudaMemcpy may return before the DMA lands: wait for
        # it, the library's next kernel runs on its own non-blocking stream
        h = np.ascontiguousarray(h)
        assert rt.cudaMemcpy(ptr, h.ctypes.data, h.nbytes, H2D) == 0
        assert rt.cudaDeviceSynchronize() == 0

    def all_reduce(buf, count, dt, op):
        npt, es = dtypes[dt]
        t = torch.from_numpy(down(buf, count, npt, es))
        o = {ncsg.SUM: dist.ReduceOp.SUM, ncsg.MIN: dist.ReduceOp.MIN,
             ncsg.MAX: dist.ReduceOp.MAX}[op]
        dist.all_reduce(t, op=o)
        up(buf, t.numpy())

    def gather_all(snd, count):
        t = torch.from_numpy(down(snd, count))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [q.numpy() for q in parts]

    def reduce_scatter(snd, rcv, count):
        t = torch.from_numpy(down(snd, count * world))
        dist.all_reduce(t)  # gloo: reduce_scatter as all-reduce + own slice
        up(rcv, t.numpy()[rank * count:(rank + 1) * count])

    def all_gather(snd, rcv, count):
        up(rcv, np.concatenate(gather_all(snd, count)))

    def all_to_all(snd, rcv, count):
        parts = gather_all(snd, count * world)
        up(rcv, np.concatenate([parts[r][rank * count:(rank + 1) * count] for r in range(world)]))

    port_ = Port()
    prob, mask, gamma = small_ct(port_, n=64, A=48)
    torch.cuda.set_device(0)
    p = ncsg.Problem(ncsg.CT, prob.n, prob.alpha, prob.beta, prob.lam, gamma, prob.b, mask=mask,
                     n_angles=prob.angles, n_det=prob.det, orbit_shard=(rank, world))
    comm = ncsg.Comm.callbacks(rank, world, all_reduce, reduce_scatter, all_gather, all_to_all)
    p.set_state()
    p.set_comm(comm, ncsg.XCHG_SLAB)
    res = p.solve(30, record_every=10)
    np.savez(os.path.join(out, f"rank{rank}.npz"), x=res.x, rows=res.rows)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
