// Communicators for the sharded NCS step: the exchange of a
// sharded problem's partial A^T u, its slab-decomposed FFT and its x slabs.
//
// Three transports behind one interface (ncsg_comm, include/ncsg.h):
//   * NCCL over NVLink / NVSwitch -- libnccl.so.2 opened at run time (the
//     process's already-loaded copy when torch brought one), so libncsg has
//     no link-time NCCL dependency; one communicator per rank/GPU;
//   * caller callbacks (ncsg_comm_ops) -- e.g. gloo on host-staged buffers in
//     the CPU multi-process tests;
//   * an in-process group of ranks driven by host threads, exchanging through
//     host memory (the one-GPU emulation of the multi-rank path: the ranks'
//     kernels never wait on each other, only their host threads do).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ncsg_comm.hpp"

namespace ncsg {

namespace {

// ---------------------------------------------------------------- NCCL
// Minimal mirror of nccl.h (2.x ABI): opaque communicator, 128-byte id, the
// enums' values.
using nccl_comm_t = void*;
struct NcclId {
  char internal[128];
};
enum { kNcclInt32 = 2, kNcclFloat32 = 7, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };

struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(nccl_comm_t*, int, NcclId, int) = nullptr;
  int (*CommDestroy)(nccl_comm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*ReduceScatter)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // an already-loaded NCCL (torch's) first, then the loader's search path
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) return a;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(a.h, name)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.ReduceScatter, "ncclReduceScatter");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.h || !api.CommInitRank || !api.Send)
    throw Error{NCSG_CUDA, "NCCL (libnccl.so.2) is not available in this process"};
  return api;
}

void nccl_check(int r, const char* what) {
  if (r != 0)
    throw Error{NCSG_CUDA, std::string(what) + ": " +
                               (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error")};
}

int nccl_type(ncsg_dtype t) {
  return t == NCSG_F64 ? kNcclFloat64 : (t == NCSG_I32 ? kNcclInt32 : kNcclFloat32);
}
int nccl_op(ncsg_redop o) { return o == NCSG_MIN ? kNcclMin : (o == NCSG_MAX ? kNcclMax : kNcclSum); }

// Peer views of every rank's allocation for multi-process transports: the
// CUDA IPC handles (64 bytes = 16 floats) all-gathered through the
// transport itself, the peers' handles opened in this process (NVLink /
// NVSwitch peer mappings across GPUs; plain mappings between processes that
// share a GPU).  Opened mappings are appended to `opened` for closing.
std::vector<void*> ipc_share(Comm& c, void* mine, std::vector<void*>& opened) {
  cudaIpcMemHandle_t h;
  NCSG_CUDA_CHECK(cudaIpcGetMemHandle(&h, mine));
  static_assert(sizeof(h) % 4 == 0, "handle size");
  const size_t nf = sizeof(h) / 4;
  const int P = c.nranks();
  float* d = nullptr;
  NCSG_CUDA_CHECK(cudaMalloc(&d, nf * 4 * (P + 1)));
  cudaStream_t s = nullptr;
  NCSG_CUDA_CHECK(cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice));
  c.all_gather(d, d + nf, nf, s);
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<cudaIpcMemHandle_t> all(P);
  NCSG_CUDA_CHECK(cudaMemcpy(all.data(), d + nf, sizeof(h) * P, cudaMemcpyDeviceToHost));
  cudaFree(d);
  std::vector<void*> out(P);
  for (int r = 0; r < P; ++r) {
    if (r == c.rank()) {
      out[r] = mine;
      continue;
    }
    NCSG_CUDA_CHECK(cudaIpcOpenMemHandle(&out[r], all[r], cudaIpcMemLazyEnablePeerAccess));
    opened.push_back(out[r]);
  }
  return out;
}

class NcclComm final : public Comm {
 public:
  NcclComm(const unsigned char* id, int rank, int nranks, int device) {
    rank_ = rank;
    nranks_ = nranks;
    NCSG_CUDA_CHECK(cudaSetDevice(device));
    NcclId uid;
    std::memcpy(uid.internal, id, sizeof uid.internal);
    nccl_check(nccl().CommInitRank(&c_, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (scratch_) cudaFree(scratch_);
    if (c_) nccl().CommDestroy(c_);
  }
  std::vector<void*> share_pointers(void* mine) override { return ipc_share(*this, mine, opened_); }
  void barrier(cudaStream_t s) override {
    if (!scratch_) NCSG_CUDA_CHECK(cudaMalloc(&scratch_, 4));
    nccl_check(nccl().AllReduce(scratch_, scratch_, 1, kNcclInt32, kNcclSum, c_, s),
               "ncclAllReduce (barrier)");
  }
  void all_reduce(void* buf, size_t count, ncsg_dtype t, ncsg_redop op, cudaStream_t s) override {
    nccl_check(nccl().AllReduce(buf, buf, count, nccl_type(t), nccl_op(op), c_, s), "ncclAllReduce");
  }
  void reduce_scatter(const float* send, float* recv, size_t count, cudaStream_t s) override {
    nccl_check(nccl().ReduceScatter(send, recv, count, kNcclFloat32, kNcclSum, c_, s),
               "ncclReduceScatter");
  }
  void all_gather(const float* send, float* recv, size_t count, cudaStream_t s) override {
    nccl_check(nccl().AllGather(send, recv, count, kNcclFloat32, c_, s), "ncclAllGather");
  }
  void all_to_all(const float* send, float* recv, size_t count, cudaStream_t s) override {
    // grouped point-to-point: chunk r of send goes to rank r, chunk r of recv
    // comes from rank r (NCCL has no all-to-all primitive)
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < nranks_; ++r) {
      nccl_check(nccl().Send(send + r * count, count, kNcclFloat32, r, c_, s), "ncclSend");
      nccl_check(nccl().Recv(recv + r * count, count, kNcclFloat32, r, c_, s), "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  const char* name() const override { return "nccl"; }
  bool capturable() const override { return true; }

 private:
  nccl_comm_t c_ = nullptr;
  void* scratch_ = nullptr;
  std::vector<void*> opened_;
};

// ----------------------------------------------------------- callbacks
class CallbackComm final : public Comm {
 public:
  explicit CallbackComm(const ncsg_comm_ops& ops) : ops_(ops) {
    rank_ = ops.rank;
    nranks_ = ops.nranks;
  }
  void all_reduce(void* buf, size_t count, ncsg_dtype t, ncsg_redop op, cudaStream_t s) override {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    call(ops_.all_reduce ? ops_.all_reduce(ops_.ctx, buf, count, t, op, s) : -1, "all_reduce");
  }
  void reduce_scatter(const float* send, float* recv, size_t count, cudaStream_t s) override {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    call(ops_.reduce_scatter ? ops_.reduce_scatter(ops_.ctx, send, recv, count, s) : -1,
         "reduce_scatter");
  }
  void all_gather(const float* send, float* recv, size_t count, cudaStream_t s) override {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    call(ops_.all_gather ? ops_.all_gather(ops_.ctx, send, recv, count, s) : -1, "all_gather");
  }
  void all_to_all(const float* send, float* recv, size_t count, cudaStream_t s) override {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    call(ops_.all_to_all ? ops_.all_to_all(ops_.ctx, send, recv, count, s) : -1, "all_to_all");
  }
  const char* name() const override { return "callbacks"; }
  void barrier(cudaStream_t s) override {
    if (!scratch_) NCSG_CUDA_CHECK(cudaMalloc(&scratch_, 4));
    all_reduce(scratch_, 1, NCSG_I32, NCSG_SUM, s);
  }
  std::vector<void*> share_pointers(void* mine) override { return ipc_share(*this, mine, opened_); }
  ~CallbackComm() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (scratch_) cudaFree(scratch_);
  }

 private:
  void* scratch_ = nullptr;
  std::vector<void*> opened_;
  static void call(int rc, const char* what) {
    if (rc != 0)
      throw Error{NCSG_CUDA, std::string("communicator callback ") + what + " failed (" +
                                 std::to_string(rc) + ")"};
  }
  ncsg_comm_ops ops_;
};

// ------------------------------------------------- in-process rank group
// Every collective: each rank's thread syncs its stream, copies its send
// data to host, meets the others at a barrier, computes its own result from
// all ranks' host copies (fixed rank order) and uploads it.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<std::vector<char>> host;  // per-rank staged send data
  std::vector<void*> ptrs;              // share_pointers exchange
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)) {
    rank_ = rank;
    nranks_ = g_->n;
  }
  void all_reduce(void* buf, size_t count, ncsg_dtype t, ncsg_redop op, cudaStream_t s) override {
    const size_t es = t == NCSG_F64 ? 8 : 4;
    stage(buf, count * es, s);
    std::vector<char> out(count * es);
    for (size_t i = 0; i < count; ++i) {
      if (t == NCSG_F64)
        reinterpret_cast<double*>(out.data())[i] = reduce<double>(i, op);
      else if (t == NCSG_I32)
        reinterpret_cast<int*>(out.data())[i] = reduce<int>(i, op);
      else
        reinterpret_cast<float*>(out.data())[i] = reduce<float>(i, op);
    }
    finish(buf, out.data(), out.size(), s);
  }
  void reduce_scatter(const float* send, float* recv, size_t count, cudaStream_t s) override {
    stage(send, count * nranks_ * 4, s);
    std::vector<float> out(count, 0.f);
    for (int r = 0; r < nranks_; ++r) {
      const float* src = reinterpret_cast<const float*>(g_->host[r].data()) + rank_ * count;
      for (size_t i = 0; i < count; ++i) out[i] += src[i];
    }
    finish(recv, out.data(), count * 4, s);
  }
  void all_gather(const float* send, float* recv, size_t count, cudaStream_t s) override {
    stage(send, count * 4, s);
    std::vector<float> out(count * nranks_);
    for (int r = 0; r < nranks_; ++r)
      std::memcpy(out.data() + r * count, g_->host[r].data(), count * 4);
    finish(recv, out.data(), out.size() * 4, s);
  }
  void all_to_all(const float* send, float* recv, size_t count, cudaStream_t s) override {
    stage(send, count * nranks_ * 4, s);
    std::vector<float> out(count * nranks_);
    for (int r = 0; r < nranks_; ++r)
      std::memcpy(out.data() + r * count,
                  reinterpret_cast<const float*>(g_->host[r].data()) + rank_ * count, count * 4);
    finish(recv, out.data(), out.size() * 4, s);
  }
  const char* name() const override { return "local"; }
  std::vector<void*> share_pointers(void* mine) override {
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->ptrs.resize(nranks_);
      g_->ptrs[rank_] = mine;
    }
    g_->barrier();
    std::vector<void*> out = g_->ptrs;
    g_->barrier();
    return out;
  }
  void barrier(cudaStream_t s) override {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    g_->barrier();
  }

 private:
  template <class T>
  T reduce(size_t i, ncsg_redop op) const {
    T acc = reinterpret_cast<const T*>(g_->host[0].data())[i];
    for (int r = 1; r < nranks_; ++r) {
      const T v = reinterpret_cast<const T*>(g_->host[r].data())[i];
      acc = op == NCSG_SUM ? acc + v : (op == NCSG_MIN ? (v < acc ? v : acc) : (v > acc ? v : acc));
    }
    return acc;
  }
  void stage(const void* dev, size_t bytes, cudaStream_t s) {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    g_->host[rank_].resize(bytes);
    NCSG_CUDA_CHECK(cudaMemcpy(g_->host[rank_].data(), dev, bytes, cudaMemcpyDeviceToHost));
    g_->barrier();  // everyone's send data is staged
  }
  void finish(void* dev, const void* data, size_t bytes, cudaStream_t s) {
    g_->barrier();  // everyone has read the staged data
    NCSG_CUDA_CHECK(cudaMemcpyAsync(dev, data, bytes, cudaMemcpyHostToDevice, s));
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  std::shared_ptr<LocalGroup> g_;
};

// No exchange at all: every collective returns at once.  A timing tool --
// one rank's kernels of the sharded step, stream-ordered and uninterrupted,
// for projecting multi-GPU step times on one GPU (scripts/shard_step_time.py).
class NullComm final : public Comm {
 public:
  NullComm(int rank, int nranks) {
    rank_ = rank;
    nranks_ = nranks;
  }
  void all_reduce(void*, size_t, ncsg_dtype, ncsg_redop, cudaStream_t) override {}
  void reduce_scatter(const float*, float*, size_t, cudaStream_t) override {}
  void all_gather(const float*, float*, size_t, cudaStream_t) override {}
  void all_to_all(const float*, float*, size_t, cudaStream_t) override {}
  void barrier(cudaStream_t) override {}
  const char* name() const override { return "null"; }
  bool capturable() const override { return true; }
};

}  // namespace

Comm* make_null_comm(int rank, int nranks) { return new NullComm(rank, nranks); }

Comm* make_nccl_comm(const unsigned char* id, int rank, int nranks, int device) {
  return new NcclComm(id, rank, nranks, device);
}
void nccl_unique_id(unsigned char* out) {
  NcclId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, sizeof id.internal);
}
Comm* make_callback_comm(const ncsg_comm_ops& ops) { return new CallbackComm(ops); }
std::vector<Comm*> make_local_group(int nranks) {
  auto g = std::make_shared<LocalGroup>();
  g->n = nranks;
  g->host.resize(nranks);
  std::vector<Comm*> out;
  for (int r = 0; r < nranks; ++r) out.push_back(new LocalComm(g, r));
  return out;
}

}  // namespace ncsg
