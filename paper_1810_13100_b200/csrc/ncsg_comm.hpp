// Internal communicator interface of the sharded NCS step (comm.cpp).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "ncsg_internal.cuh"

namespace ncsg {

// Collectives on device buffers, stream-ordered (NCCL) or completed before
// return (callbacks, local group).  All float sums are of fp32 data.
class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  virtual void all_reduce(void* buf, size_t count, ncsg_dtype t, ncsg_redop op, cudaStream_t s) = 0;
  // recv[count] = sum over ranks r of send_r[rank * count .. + count]
  virtual void reduce_scatter(const float* send, float* recv, size_t count, cudaStream_t s) = 0;
  // recv[r * count ..] = send_r[0 .. count]
  virtual void all_gather(const float* send, float* recv, size_t count, cudaStream_t s) = 0;
  // recv[r * count ..] = send_r[rank * count ..]
  virtual void all_to_all(const float* send, float* recv, size_t count, cudaStream_t s) = 0;
  virtual const char* name() const = 0;
  // stream-ordered collectives that a CUDA graph can capture (NCCL)
  virtual bool capturable() const { return false; }
  // Peer memory (the fused P2P exchange): every rank's `mine` (the base of a
  // cudaMalloc allocation of the same size on every rank) as pointers this
  // rank's kernels can store to -- NVLink peers through CUDA IPC (NCCL
  // transport), plain pointers within one process (local group).  Empty when
  // the transport has no peer memory.
  virtual std::vector<void*> share_pointers(void* mine) { (void)mine; return {}; }
  // All ranks' work on their streams so far is complete and visible to the
  // peers' later work (stream-ordered for NCCL).
  virtual void barrier(cudaStream_t s) = 0;

 protected:
  int rank_ = 0, nranks_ = 1;
};

Comm* make_nccl_comm(const unsigned char* id, int rank, int nranks, int device);
void nccl_unique_id(unsigned char* out);
Comm* make_callback_comm(const ncsg_comm_ops& ops);
Comm* make_null_comm(int rank, int nranks);
std::vector<Comm*> make_local_group(int nranks);

}  // namespace ncsg
