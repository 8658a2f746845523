// C ABI (include/ncsg.h): handles, the device-resident NCS engine and the
// reference-shaped entry points.  No exceptions cross the boundary; there is
// no CPU fallback -- without a CUDA device every compute call fails loudly.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <thread>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host_rng.hpp"
#include "ncs_kernels.cuh"
#include "ncsg_comm.hpp"
#include "ncsg_internal.cuh"

namespace ncsg {

namespace {
thread_local std::string g_err;
}
void set_error(const std::string& msg) { g_err = msg; }
namespace {
std::atomic<int64_t> g_launches{0};
}
int64_t launch_count() { return g_launches.load(); }
void count_launch(int k) { g_launches += k; }
bool pdl_enabled() {
  static const bool on = std::getenv("NCSG_NO_PDL") == nullptr;
  return on;
}

template <class F>
ncsg_status guard(F&& f) {
  try {
    f();
    return NCSG_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NCSG_RUNTIME;
  }
}

void require_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw Error{NCSG_CUDA, "no CUDA device is available (the NCS path has no CPU fallback)"};
  if (device < 0 || device >= count) throw Error{NCSG_INVALID, "device index out of range"};
  NCSG_CUDA_CHECK(cudaSetDevice(device));
}

// Hermitian part of a full N x N complex mask, half spectrum stored [k][j]
// (k = 0..N/2) and scaled by `scale` (the 1/N^2 of fft.cpp:46-47).
// Rows [r0, r1) of a setup loop on all host cores (setup only).
template <class F>
void parallel_rows(int rows, F f) {
  const int nt = std::max(1, std::min<int>(16, static_cast<int>(std::thread::hardware_concurrency())));
  if (rows < 64 || nt == 1) {
    f(0, rows);
    return;
  }
  std::vector<std::thread> th;
  const int per = (rows + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int r0 = t * per, r1 = std::min(rows, r0 + per);
    if (r0 < r1) th.emplace_back(f, r0, r1);
  }
  for (auto& t : th) t.join();
}

// Hermitian part of h on the half spectrum, transposed to [k][j] (the
// device's column-major half spectrum), 32 x 32 blocks so both the reads
// (rows j and N-j of h) and the writes stay in cache.
// h given as a function of the flat bin index (no n^2 temporary).
template <class F>
std::vector<float2> half_mask_f(int n, F h, double scale) {
  const int nk = n / 2 + 1;
  std::vector<float2> out(static_cast<size_t>(nk) * n);
  parallel_rows((n + 31) / 32, [&](int b0, int b1) {
    for (int jb = b0 * 32; jb < std::min(n, b1 * 32); jb += 32)
      for (int kb = 0; kb < nk; kb += 32)
        for (int j = jb; j < std::min(n, jb + 32); ++j) {
          const size_t hr = static_cast<size_t>(j) * n;
          const size_t hc = static_cast<size_t>((n - j) % n) * n;
          for (int k = kb; k < std::min(nk, kb + 32); ++k) {
            const std::complex<double> v = 0.5 * (h(hr + k) + std::conj(h(hc + (n - k) % n))) * scale;
            out[static_cast<size_t>(k) * n + j] =
                make_float2(static_cast<float>(v.real()), static_cast<float>(v.imag()));
          }
        }
  });
  return out;
}
std::vector<float2> half_mask(int n, const std::vector<std::complex<double>>& h, double scale) {
  return half_mask_f(n, [&](size_t i) { return h[i]; }, scale);
}

std::vector<std::complex<double>> read_mask(int n, const double* m) {
  std::vector<std::complex<double>> h(static_cast<size_t>(n) * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = {m[2 * i], m[2 * i + 1]};
  return h;
}

struct Stream {
  cudaStream_t s = nullptr;
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
};

}  // namespace ncsg

using namespace ncsg;

struct ncsg_radon {
  RadonDev dev;
  Stream stream;
};

struct ncsg_sparse {
  SparseDev dev;
  Stream stream;
  int device = 0;
};

struct ncsg_problem {
  ncsg_problem_desc d{};
  int device = 0;
  Stream stream;
  std::unique_ptr<RadonDev> radon;
  const SparseDev* sparse = nullptr;  // SparseMap projector (caller keeps the handle alive)
  FftPlan fft;
  bool has_mask = false;          // an M symbol for the seminorm / screen is on the device
  bool override_mode = false;     // m_pinv given (XMode::Override)
  double gamma_m = 0.0;           // gamma of M = gamma I + alpha C (0 in Override mode)
  std::vector<std::complex<double>> mask_full;  // cfg.mask (apply_m)
  DevBuf<float2> maskT;       // herm(pinv(gamma + alpha C)) / N^2
  DevBuf<float2> maskT_orig;  // herm(C) / N^2 for apply_m (seminorm, screen)
  size_t nn = 0, m0 = 0, g = 0, range = 0;
  int batch = 1;
  float wd = 0.f, bound = 0.f;
  DevBuf<float> x, x_old, xT, u, axs, b;
  DevBuf<float> fp_part, bp_part;
  DevBuf<float2> spec;
  DevBuf<int> flag;  // [0] first bad step (INT_MAX: none), [1] step counter
  DevBuf<double> red;
  // record-step scratch (lazy)
  DevBuf<float> x_prev, u_prev, dx, du, adx, mdx, dxT;
  int64_t iter = 0;
  int64_t flag_base = 0;          // iteration at the last reset_flag
  size_t m_begin = 0, m_end = 0;  // own rays of the data block (CT)
  bool sharded = false;            // angle- or orbit-sharded (multi-GPU phases)
  bool quad_fused = false;         // this step's inverse row pass wrote the orbit member planes
  bool dual_fused = false;         // this step's inverse row pass did the x-only dual blocks
  // Orbit-interleaved copy of the sinogram dual (gather-mode adjoint input),
  // written by the dual update; fresh while u has not been written otherwise.
  DevBuf<float> u4;
  bool u4_fresh = false;
  DevBuf<uint8_t> own_angle;       // orbit sharding: own[t] (nullptr otherwise)
  bool rank0 = true;              // adds the replicated blocks to A^T u
  float* atu_ext = nullptr;       // caller-owned A^T u buffer (sharded phases)
  DevBuf<float> atu_own;
  // admm_cg_solve mode (solvers.cpp:435-440): n_cg > 0 replaces the circulant
  // x-update by n_cg CG steps on A^T A (batch 1, unsharded, no mask)
  int n_cg = 0;
  DevBuf<double> cg_x, cg_r, cg_p;  // fp64 CG iterates
  DevBuf<float> cg_p32, cg_ap;       // operator input / output
  std::map<int, cudaGraphExec_t> graphs;
  // multi-GPU (ncsg_problem_set_comm): the cross-rank exchange of a sharded
  // step; slab mode: rows [rank R, rank R + R) of the image, wc spectrum
  // columns per rank (P wc >= N/2+1, padded), the filter padded likewise
  ncsg::Comm* comm = nullptr;
  int xchg = NCSG_XCHG_ALLREDUCE;
  int slab_R = 0, slab_logR = 0, slab_wc = 0;
  DevBuf<float> atu_full, atu_slab;
  DevBuf<float2> spec_slab, spec_recv, maskT_pad;
  // P2P mode: the receive slots [src rank][R][n] and the peers' views of
  // recv_slots / spec_recv / spec_slab / x
  DevBuf<float> recv_slots;
  PeerPtrs peer_slots, peer_recv, peer_slab, peer_x;
  // phase profiling (bench.py): events recorded between the phases of do_step
  bool profiling = false;
  std::vector<cudaEvent_t> events;  // kPhases + 1 per profiled step
  size_t ev_used = 0;
  ~ncsg_problem() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (auto e : events) cudaEventDestroy(e);
  }
};

namespace {

int* step_counter(ncsg_problem* p) { return p->flag.p; }

// ---- projector of the data block: the parallel-beam RadonMap kernels or an
// explicit SparseMap (fan beam).  Both write R x as partial slots summed by
// the dual update / strip_sum, and R^T u as partial images (class-V frame,
// then class-H transposed) summed into A^T u by the FFT loader.
int proj_slots(const ncsg_problem* p) {
  return p->sparse ? 1 : (p->radon ? p->radon->fp_slots() : 0);
}
int proj_nV(const ncsg_problem* p) { return p->sparse ? 1 : p->radon->bp_chunks[0]; }
int proj_nH(const ncsg_problem* p) { return p->sparse ? 0 : p->radon->bp_chunks[1]; }
int proj_parts(const ncsg_problem* p) { return proj_nV(p) + proj_nH(p); }
void proj_prepare(ncsg_problem* p, const float* img, float* aux, int batch);
void proj_forward(ncsg_problem* p, const float* img, const float* aux, float* part, int batch) {
  if (p->sparse)
    launch_sparse_forward(*p->sparse, img, p->nn, part, p->m0, batch, p->stream.s);
  else
    launch_radon_forward_partial(*p->radon, img, aux, part, batch, p->stream.s);
}
void proj_adjoint(ncsg_problem* p, const float* u, size_t u_stride, float* part, int batch,
                  const float* u4 = nullptr) {
  if (p->sparse)
    launch_sparse_adjoint(*p->sparse, u, u_stride, part, p->nn, batch, p->stream.s);
  else
    launch_radon_adjoint_partial(*p->radon, u, u_stride, part, batch, p->stream.s, u4);
}

// Second input of the forward: x^T for class-H angles, or the symmetry
// planes in orbit mode.
float* prepare_forward_aux(const RadonDev& r, const float* img, float* aux, int batch,
                           cudaStream_t s) {
  if (r.orbit_mode) {
    launch_make_planes(img, aux, r.geo.n, batch, s);
    return aux;
  }
  if (!r.geo.cls[1].empty()) launch_transpose(img, aux, r.geo.n, batch, s);
  return aux;
}

void proj_prepare(ncsg_problem* p, const float* img, float* aux, int batch) {
  if (p->radon) prepare_forward_aux(*p->radon, img, aux, batch, p->stream.s);
}

AtuTerms atu_terms_for(ncsg_problem* p, float* u);
AtuTerms atu_terms(ncsg_problem* p) { return atu_terms_for(p, p->u.p); }

// Terms of A^T u for an arbitrary dual vector u laid out like the state's.
AtuTerms atu_terms_for(ncsg_problem* p, float* u) {
  AtuTerms T;
  T.n = p->d.n;
  if (p->d.kind != NCSG_DENOISE) {
    T.bp_part = p->bp_part.p;
    T.nV = proj_nV(p);
    T.nH = proj_nH(p);
    T.part_stride = static_cast<size_t>(proj_parts(p)) * p->nn;
    if (p->rank0 && p->d.positivity) T.ident = u + p->m0 + p->g;
  } else if (p->rank0) {
    T.ident = u;
    if (p->d.positivity) T.ident2 = u + p->m0 + p->g;
  }
  T.ident_stride = p->range;
  if (p->rank0) {
    T.ug = u + p->m0;
    T.ug_stride = p->range;
    T.wd = p->wd;
  }
  return T;
}

constexpr int kPhases = 7;  // adjoint, fft rows r2c, fft cols, fft rows c2r, make_quad, forward, dual

void mark(ncsg_problem* p) {
  if (!p->profiling) return;
  if (p->ev_used == p->events.size()) {
    cudaEvent_t e;
    NCSG_CUDA_CHECK(cudaEventCreate(&e));
    p->events.push_back(e);
  }
  NCSG_CUDA_CHECK(cudaEventRecord(p->events[p->ev_used++], p->stream.s));
}

void phase_a(ncsg_problem* p) {
  mark(p);
  if (p->d.kind != NCSG_DENOISE) {
    // u_s is the first m0 entries of each problem's dual (stride range).
    proj_adjoint(p, p->u.p, p->range, p->bp_part.p, p->batch, p->u4_fresh ? p->u4.p : nullptr);
  }
}

void x_update_cg(ncsg_problem* p);
void phase_b_circulant(ncsg_problem* p, const float* plain);
void forward_and_dual(ncsg_problem* p);

// plain != nullptr: A^T u was assembled (and all-reduced) into `plain`.
void phase_b(ncsg_problem* p, const float* plain = nullptr) {
  p->quad_fused = false;
  if (p->n_cg > 0 && !plain) {
    x_update_cg(p);
  } else {
    phase_b_circulant(p, plain);
  }
  forward_and_dual(p);
}

bool fuse_dual_terms(const ncsg_problem* p, DualFuse& df);
void phase_b_circulant(ncsg_problem* p, const float* plain) {
  cudaStream_t s = p->stream.s;
  AtuTerms T = atu_terms(p);
  if (plain) {
    T = AtuTerms();
    T.n = p->d.n;
    T.plain = plain;
  }
  T.counter = step_counter(p);
  mark(p);
  launch_fft_rows_r2c(p->fft, T, p->spec.p, p->batch, s);
  mark(p);
  launch_fft_cols_filter(p->fft, p->spec.p, p->maskT.p, p->batch, s);
  XUpdate xu;
  xu.x = p->x.p;
  xu.x_old = p->x_old.p;
  xu.xT = (p->radon && !p->radon->orbit_mode && !p->radon->geo.cls[1].empty())
              ? p->xT.p
              : nullptr;
  xu.subtract = 1;
  xu.flag = p->flag.p;
  // Orbit mode: the inverse row pass writes the member planes itself while
  // they stay in L2 until the forward reads them (C1 18.5k -> 19.3k it/s, C3
  // +0.3%); its column-direction 4-byte stores cost more than make_quad once
  // the planes are large (C5's 67 MB: +36 us in the row pass for -21 us).
  constexpr size_t kQuadFuseBytes = 24u << 20;
  if (p->d.kind != NCSG_DENOISE && p->radon && p->radon->orbit_mode && fft_writes_quad(p->fft) &&
      p->batch * p->nn * sizeof(float4) <= kQuadFuseBytes) {
    xu.quad = reinterpret_cast<float4*>(p->xT.p);  // orbit mode: xT holds the member planes
    p->quad_fused = true;
  }
  p->dual_fused = false;
  if (!plain && fuse_dual_terms(p, xu.df)) {
    xu.df.on = 1;
    p->dual_fused = true;
  }
  mark(p);
  launch_fft_rows_c2r(p->fft, p->spec.p, xu, p->batch, s);
}

// DENOISE: every dual block needs only x, so the whole dual update runs in
// the inverse row pass that produces x (unsharded power-of-two problems) and
// the step is three kernels.  (CT keeps the stand-alone dual kernel: fusing
// only its D block measured no gain at C1/C3/C5.)  Fills df (on = 0) and
// returns whether the fusion applies.
bool fuse_dual_terms(const ncsg_problem* p, DualFuse& df) {
  df = DualFuse{};
  if (p->d.kind != NCSG_DENOISE || p->sharded || p->comm) return false;
  df.alpha = static_cast<float>(p->d.alpha);
  df.s_quad = static_cast<float>(1.0 / (1.0 + p->d.alpha));
  df.wd = p->wd;
  df.bound = p->bound;
  df.u_stride = p->range;
  df.flag = p->flag.p;
  float* u = p->u.p;
  df.ud = u;  // identity (data) block, then D, then positivity
  df.bd = p->b.p;
  df.ug = u + p->m0;
  if (p->d.positivity) df.up = u + p->m0 + p->g;
  return fft_fuses_dual(p->fft, df);
}

// Engine::step after the x update (solvers.cpp:146-158): R x+ for the own
// angles and the fused dual update.
void forward_and_dual(ncsg_problem* p) {
  cudaStream_t s = p->stream.s;
  mark(p);
  if (p->d.kind != NCSG_DENOISE && p->radon && p->radon->orbit_mode && !p->quad_fused)
    launch_make_planes(p->x.p, p->xT.p, p->d.n, p->batch, s);
  p->quad_fused = false;
  mark(p);
  if (p->d.kind != NCSG_DENOISE) proj_forward(p, p->x.p, p->xT.p, p->fp_part.p, p->batch);
  mark(p);
  DualArgs a;
  a.kind = p->d.kind;
  a.n = p->d.n;
  a.positivity = p->d.positivity;
  a.alpha = static_cast<float>(p->d.alpha);
  a.s_quad = static_cast<float>(1.0 / (1.0 + p->d.alpha));
  a.wd = p->wd;
  a.bound = p->bound;
  a.fp_part = p->fp_part.p;
  a.n_strips = proj_slots(p);
  a.m = p->m0;
  a.m_begin = p->m_begin;
  a.m_end = p->m_end;
  a.own = p->own_angle.p;
  a.det = p->d.n_det;
  a.u0 = p->u.p;
  a.axs = p->axs.p;
  a.b = p->b.p;
  a.ug = p->u.p + p->m0;
  a.up = p->u.p + p->m0 + p->g;
  a.u_stride = p->range;
  a.x = p->x.p;
  a.x_old = p->x_old.p;
  a.flag = p->flag.p;
  if (p->u4.n) {
    a.u4 = p->u4.p;
    a.slot = p->radon->angle_slot.p;
    a.u4_row = p->radon->u4_row();
    a.u4_pad = kGaSW;
    a.u4_stride = p->radon->u4_size();
    // Orbit-major items touch only the listed (own) orbits' rays: used for
    // orbit shards, where the ray-major loop would visit every ray of the
    // sinogram.  Unsharded, the ray-major loop's 16-byte partial-slot loads
    // win over the coalesced u4 cells (C3 dual update 18.3 vs 22.6 us).
    if (p->d.kind == NCSG_CT && (p->radon->geo.orbit_sharded || getenv("NCSG_DUAL_ORBIT_MAJOR"))) {
      a.orb_t = p->radon->orbit_t.p;
      a.n_orb = static_cast<int>(p->radon->geo.orbits.size());
    }
  }
  // x-only blocks already updated by the inverse row pass: the data block
  // alone (CT / PET), nothing for DENOISE
  a.data_only = p->dual_fused ? 1 : 0;
  if (!(p->dual_fused && p->d.kind == NCSG_DENOISE)) launch_dual_update(a, p->batch, s);
  p->dual_fused = false;
  p->u4_fresh = p->u4.n > 0;
  mark(p);
}

// The orbit-interleaved dual copy, rebuilt from u when u was written
// outside the dual update (set_state, the raw state view).
void refresh_u4(ncsg_problem* p) {
  if (!p->u4.n || p->u4_fresh) return;
  DualArgs a;
  a.u0 = p->u.p;
  a.u_stride = p->range;
  a.m = p->m0;
  a.det = p->d.n_det;
  a.u4 = p->u4.p;
  a.slot = p->radon->angle_slot.p;
  a.u4_row = p->radon->u4_row();
  a.u4_pad = kGaSW;
  a.u4_stride = p->radon->u4_size();
  launch_u4_pack(a, p->batch, p->stream.s);
  p->u4_fresh = true;
}

// One sharded step with the communicator (Engine::step,
// solvers.cpp:124-161, with StackedMap::adjoint's sum, linear_map.cpp:47-55,
// taken across ranks).  Every rank: its partial A^T u (own angles; rank 0
// also the replicated D^T u_g / identity terms) as one image, then
//   ALLREDUCE: all-reduce of the image, replicated circulant solve;
//   SLAB:      reduce-scatter into N/P-row slabs, row FFT of the own slab,
//              all-to-all transpose to wc-column slabs, column FFT . filter .
//              inverse, all-to-all back, inverse rows + x update of the own
//              rows, all-gather of x;
// and the forward + dual update of the own rays and the replicated u_g.
void sharded_step(ncsg_problem* p) {
  cudaStream_t s = p->stream.s;
  ncsg::Comm& C = *p->comm;
  phase_a(p);
  float* atu = p->atu_full.p;
  AtuTerms T = atu_terms(p);
  if (p->xchg != NCSG_XCHG_P2P) launch_atu_assemble(T, atu, p->batch, s);
  if (p->xchg == NCSG_XCHG_ALLREDUCE) {
    C.all_reduce(atu, p->nn * p->batch, NCSG_F32, NCSG_SUM, s);
    phase_b(p, atu);
    return;
  }
  const int n = p->d.n, P = C.nranks(), R = p->slab_R, wc = p->slab_wc;
  const int r0 = C.rank() * R;
  if (p->xchg == NCSG_XCHG_P2P) {
    // every exchange fused into its producing kernel over peer memory, a
    // stream-ordered barrier between the kernels
    const int nk = n / 2 + 1, rk = C.rank();
    NCSG_CUDA_CHECK(cudaMemcpyAsync(p->x_old.p, p->x.p, p->nn * 4, cudaMemcpyDeviceToDevice, s));
    mark(p);
    launch_atu_assemble_scatter(T, p->peer_slots, R, rk, s);  // reduce-scatter
    C.barrier(s);
    AtuTerms S;
    S.n = n;
    S.bp_part = p->recv_slots.p - static_cast<size_t>(r0) * n;  // rows addressed globally
    S.nV = P;
    S.img_stride = static_cast<size_t>(R) * n;
    S.counter = step_counter(p);
    RowSlab rs{r0, R, R, static_cast<size_t>(P) * wc * R};
    rs.wc = wc;
    rs.rank = rk;
    rs.peers = p->peer_recv;
    launch_fft_rows_r2c(p->fft, S, p->spec_slab.p, 1, s, rs);  // + all-to-all
    C.barrier(s);
    mark(p);
    ColSlab cs{p->slab_logR, wc, rk * wc, std::max(0, std::min(wc, nk - rk * wc))};
    cs.rank = rk;
    cs.peers = p->peer_slab;
    launch_fft_cols_filter_slab(p->fft, p->spec_recv.p, p->maskT_pad.p, cs, s);  // + back
    C.barrier(s);
    mark(p);
    XUpdate xu;
    xu.x = p->x.p;
    xu.subtract = 1;
    xu.flag = p->flag.p;
    for (int q = 0; q < P; ++q)
      if (q != rk) xu.x_peers.p[xu.n_peers++] = p->peer_x.p[q];
    const RowSlab own{r0, R, R, static_cast<size_t>(P) * wc * R};
    launch_fft_rows_c2r(p->fft, p->spec_slab.p, xu, 1, s, own);  // + all-gather
    C.barrier(s);
    if (p->radon && !p->radon->orbit_mode && !p->radon->geo.cls[1].empty())
      launch_transpose(p->x.p, p->xT.p, n, 1, s);
    forward_and_dual(p);
    return;
  }
  mark(p);
  C.reduce_scatter(atu, p->atu_slab.p, static_cast<size_t>(R) * n, s);
  AtuTerms S;
  S.n = n;
  S.plain = p->atu_slab.p - static_cast<size_t>(r0) * n;  // rows addressed globally
  S.counter = step_counter(p);
  const RowSlab rs{r0, R, R, static_cast<size_t>(P) * wc * R};
  launch_fft_rows_r2c(p->fft, S, p->spec_slab.p, 1, s, rs);
  mark(p);
  const size_t chunk = 2 * static_cast<size_t>(wc) * R;  // floats per rank block
  C.all_to_all(reinterpret_cast<const float*>(p->spec_slab.p),
               reinterpret_cast<float*>(p->spec_recv.p), chunk, s);
  const int nk = n / 2 + 1;
  ColSlab cs{p->slab_logR, wc, C.rank() * wc, std::max(0, std::min(wc, nk - C.rank() * wc))};
  launch_fft_cols_filter_slab(p->fft, p->spec_recv.p, p->maskT_pad.p, cs, s);
  C.all_to_all(reinterpret_cast<const float*>(p->spec_recv.p),
               reinterpret_cast<float*>(p->spec_slab.p), chunk, s);
  mark(p);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(p->x_old.p, p->x.p, p->nn * 4, cudaMemcpyDeviceToDevice, s));
  XUpdate xu;
  xu.x = p->x.p;
  xu.subtract = 1;
  xu.flag = p->flag.p;
  launch_fft_rows_c2r(p->fft, p->spec_slab.p, xu, 1, s, rs);
  float* own_rows = p->x.p + static_cast<size_t>(r0) * n;
  C.all_gather(own_rows, p->x.p, static_cast<size_t>(R) * n, s);
  if (p->radon && !p->radon->orbit_mode && !p->radon->geo.cls[1].empty())
    launch_transpose(p->x.p, p->xT.p, n, 1, s);  // class-H forward input
  forward_and_dual(p);
}

void do_step(ncsg_problem* p) {
  if (p->comm) {
    sharded_step(p);
    return;
  }
  phase_a(p);
  phase_b(p);
}

// Engine::init (solvers.cpp:118-122): ax = A x for the data block (the other
// blocks are recomputed from x each step).
void engine_init(ncsg_problem* p) {
  cudaStream_t s = p->stream.s;
  if (p->d.kind != NCSG_DENOISE) {
    proj_prepare(p, p->x.p, p->xT.p, p->batch);
    proj_forward(p, p->x.p, p->xT.p, p->fp_part.p, p->batch);
    if (p->radon)
      launch_strip_sum(*p->radon, p->fp_part.p, p->axs.p, p->batch, s);
    else
      NCSG_CUDA_CHECK(cudaMemcpyAsync(p->axs.p, p->fp_part.p, p->m0 * p->batch * 4,
                                      cudaMemcpyDeviceToDevice, s));
  }
}

// Device flag words: [0] first step (counted from the reset) whose image
// iterate left the finite range, [1] the step counter, [2] first step whose
// dual iterate became NaN.  flag_base = the iteration at the reset, so the
// reported iteration is absolute like DivergenceError::iter.
void reset_flag(ncsg_problem* p) {
  int h[3] = {INT_MAX, 0, INT_MAX};
  p->flag_base = p->iter;
  NCSG_CUDA_CHECK(cudaMemcpyAsync(p->flag.p, h, sizeof(h), cudaMemcpyHostToDevice, p->stream.s));
}

// Throws DivergenceError-equivalent if any step flagged a non-finite value:
// check_finite (solvers.cpp:248-255) tests x before u, so an image failure
// in the same step wins.
void check_divergence(ncsg_problem* p, int64_t* diverged_iter = nullptr) {
  int h[3];
  if (p->comm)  // a rank's own rays / rows: every rank sees the first bad step
    p->comm->all_reduce(p->flag.p, 3, NCSG_I32, NCSG_MIN, p->stream.s);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(h, p->flag.p, sizeof(h), cudaMemcpyDeviceToHost, p->stream.s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(p->stream.s));
  if (h[0] != INT_MAX || h[2] != INT_MAX) {
    const bool img = h[0] <= h[2];
    const int64_t it = p->flag_base + (img ? h[0] : h[2]);
    if (diverged_iter) *diverged_iter = it;
    throw Error{NCSG_DIVERGED, "diverged at iteration " + std::to_string(it) + ": " +
                                   (img ? "image iterate left the finite range"
                                        : "dual iterate became NaN")};
  }
}

std::vector<double> objective_values(ncsg_problem* p) {
  cudaStream_t s = p->stream.s;
  ObjArgs a;
  a.kind = p->d.kind;
  a.n = p->d.n;
  a.positivity = p->d.positivity;
  a.with_grad = p->rank0 ? 1 : 0;
  a.wd = p->wd;
  a.axs = p->axs.p;
  a.b = p->b.p;
  a.x = p->x.p;
  a.m = p->m0;
  a.m_begin = p->m_begin;
  a.m_end = p->m_end;
  a.own = p->own_angle.p;
  a.det = p->d.n_det;
  const int nb = objective_blocks();
  a.out = p->red.p;
  launch_objective(a, p->batch, s);
  std::vector<double> h(static_cast<size_t>(p->batch) * nb * 4);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), p->red.p, h.size() * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<double> f(p->batch);
  for (int b = 0; b < p->batch; ++b) {
    double q = 0, l1 = 0, mx = 0, mn = 0;
    for (int k = 0; k < nb; ++k) {
      const double* r = &h[(static_cast<size_t>(b) * nb + k) * 4];
      q += r[0];
      l1 += r[1];
      mx = std::max(mx, r[2]);
      mn = std::min(mn, r[3]);
    }
    if (p->comm) {  // own rays' data term + rank 0's D term, summed over ranks
      double qs[2] = {q, l1};
      DevBuf<double> t;
      t.alloc(2);
      NCSG_CUDA_CHECK(cudaMemcpyAsync(t.p, qs, sizeof qs, cudaMemcpyHostToDevice, s));
      p->comm->all_reduce(t.p, 2, NCSG_F64, NCSG_SUM, s);
      NCSG_CUDA_CHECK(cudaMemcpyAsync(qs, t.p, sizeof qs, cudaMemcpyDeviceToHost, s));
      NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
      q = qs[0];
      l1 = qs[1];
    }
    // QuadraticConj / PoissonConj::objective + ScaledL1Conj::objective (prox.cpp:26-70)
    double total = (p->d.kind == NCSG_PET ? q : 0.5 * q) + static_cast<double>(p->bound) * l1;
    if (p->d.positivity) {  // NonnegConj::objective (prox.cpp:107-114)
      double tol = 1e-9 * std::max(1.0, mx);
      if (mn < -tol) total = INFINITY;
    }
    f[b] = total;
  }
  return f;
}

// Sum of per-block [a.b, c.d] partials of batch entry b (dot_pair_blocks per entry).
std::vector<double> read_dot_pairs(double* dev, int batch, cudaStream_t s) {
  const int nb = dot_pair_blocks();
  std::vector<double> h(static_cast<size_t>(batch) * nb * 2);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), dev, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<double> out(2 * static_cast<size_t>(batch), 0.0);
  for (int b = 0; b < batch; ++b)
    for (int k = 0; k < nb; ++k) {
      out[2 * b] += h[(static_cast<size_t>(b) * nb + k) * 2];
      out[2 * b + 1] += h[(static_cast<size_t>(b) * nb + k) * 2 + 1];
    }
  return out;
}

void ensure_scratch(ncsg_problem* p) {
  if (p->x_prev.n) return;
  size_t xs = p->nn * p->batch, us = p->range * p->batch;
  p->x_prev.alloc(xs);
  p->u_prev.alloc(us);
  p->dx.alloc(xs);
  p->du.alloc(us);
  p->adx.alloc(us);
  p->mdx.alloc(xs);
  p->dxT.alloc(4 * xs);
}

// Stacked forward of an image into a range vector (StackedMap::forward,
// linear_map.cpp:39-45).
void stacked_forward(ncsg_problem* p, const float* img, float* imgT, float* out) {
  cudaStream_t s = p->stream.s;
  if (p->d.kind != NCSG_DENOISE) {
    proj_prepare(p, img, imgT, p->batch);
    proj_forward(p, img, imgT, p->fp_part.p, p->batch);
  }
  StackArgs a;
  a.kind = p->d.kind;
  a.n = p->d.n;
  a.n_strips = proj_slots(p);
  a.wd = p->wd;
  a.fp_part = p->fp_part.p;
  a.x = img;
  a.out = out;
  a.m0 = p->m0;
  a.range = p->range;
  launch_stacked_rest(a, p->batch, s);
}

// out = F^-1 (maskT F img) for plain images (apply_m, circulant part).
void apply_filter(ncsg_problem* p, const float* img, const float2* maskT, float* out) {
  cudaStream_t s = p->stream.s;
  AtuTerms T;
  T.n = p->d.n;
  T.plain = img;
  launch_fft_rows_r2c(p->fft, T, p->spec.p, p->batch, s);
  launch_fft_cols_filter(p->fft, p->spec.p, maskT, p->batch, s);
  XUpdate xu;
  xu.x = out;
  xu.subtract = 0;
  launch_fft_rows_c2r(p->fft, p->spec.p, xu, p->batch, s);
}

// Engine::step_seminorm (solvers.cpp:166-177) on the last step's (dx, du).
std::vector<double> seminorm_values(ncsg_problem* p) {
  cudaStream_t s = p->stream.s;
  if (p->override_mode && !p->has_mask)  // Engine::apply_m, solvers.cpp:193-197
    throw Error{NCSG_INVALID, "m_override is required alongside m_pinv_override"};
  launch_sub(p->x.p, p->x_prev.p, p->dx.p, p->nn * p->batch, s);
  launch_sub(p->u.p, p->u_prev.p, p->du.p, p->range * p->batch, s);
  stacked_forward(p, p->dx.p, p->dxT.p, p->adx.p);
  if (p->has_mask) apply_filter(p, p->dx.p, p->maskT_orig.p, p->mdx.p);
  SemArgs a;
  a.n = p->d.n;
  a.alpha = p->d.alpha;
  a.gamma = p->gamma_m;
  a.du = p->du.p;
  a.adx = p->adx.p;
  a.range = p->range;
  a.r_begin = 0;
  a.r_end = p->range;
  a.dx = p->dx.p;
  a.mdx = p->has_mask ? p->mdx.p : nullptr;
  a.out = p->red.p;
  if (p->sharded) {
    a.m0 = p->m0;
    a.m_begin = p->m_begin;
    a.m_end = p->m_end;
    a.own = p->own_angle.p;
    a.det = p->d.n_det;
    a.rank0 = p->rank0 ? 1 : 0;
  }
  launch_seminorm(a, p->batch, s);
  const int nb = objective_blocks();
  std::vector<double> h(static_cast<size_t>(p->batch) * nb * 3);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), p->red.p, h.size() * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<double> out(p->batch);
  for (int b = 0; b < p->batch; ++b) {
    double t1 = 0, aq = 0, mq = 0;
    for (int k = 0; k < nb; ++k) {
      const double* r = &h[(static_cast<size_t>(b) * nb + k) * 3];
      t1 += r[0];
      aq += r[1];
      mq += r[2];
    }
    if (p->comm) {  // the ranks' shares of the three sums
      double v3[3] = {t1, aq, mq};
      DevBuf<double> t;
      t.alloc(3);
      NCSG_CUDA_CHECK(cudaMemcpyAsync(t.p, v3, sizeof v3, cudaMemcpyHostToDevice, s));
      p->comm->all_reduce(t.p, 3, NCSG_F64, NCSG_SUM, s);
      NCSG_CUDA_CHECK(cudaMemcpyAsync(v3, t.p, sizeof v3, cudaMemcpyDeviceToHost, s));
      NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
      t1 = v3[0];
      aq = v3[1];
      mq = v3[2];
    }
    double a_quad = p->d.alpha * p->d.alpha * aq;
    double m_quad = p->n_cg > 0 ? a_quad : p->d.alpha * mq;  // Cg: M = alpha A^T A (solvers.cpp:174)
    // seminorm_from (solvers.cpp:35-50)
    double rad = t1 + m_quad - a_quad;
    if (rad < 0.0) {
      double mag = std::max(1.0, t1 + std::abs(m_quad) + a_quad);
      if (rad < -1e-10 * mag) {
        out[b] = NAN;
        continue;
      }
      rad = 0.0;
    }
    out[b] = std::sqrt(rad);
  }
  return out;
}

// Engine::screen_step_condition (solvers.cpp:206-245) in Mask / Scaled mode:
// 40-step power_method (solvers.cpp:466-484) of alpha A^T A - M + shift I
// with shift = gamma + alpha max|h| (gamma without a mask); returns the
// estimate of the largest eigenvalue of alpha A^T A - M.  Runs on batch
// entry 0 (the operator is shared by the batch).
double screen_estimate(ncsg_problem* p, uint64_t seed, int iters, double* shift_out) {
  cudaStream_t s = p->stream.s;
  ensure_scratch(p);
  struct BatchOne {
    ncsg_problem* p;
    int saved;
    ~BatchOne() { p->batch = saved; }
  } guard_batch{p, p->batch};
  p->batch = 1;
  double shift = p->d.gamma;
  if (p->override_mode) {
    // screen_step_condition's Override branch (solvers.cpp:219-226) shifts by
    // 1.3 |power_method(M, 15)| + 1; for a circulant M the power method
    // converges to max |symbol|, used here directly (the screen only warns)
    if (!p->has_mask)
      throw Error{NCSG_INVALID, "m_override is required alongside m_pinv_override"};
    double hmax = 0.0;
    for (const auto& z : p->mask_full) hmax = std::max(hmax, std::abs(z));
    shift = 1.3 * hmax + 1.0;
  } else if (p->has_mask) {
    double hmax = 0.0;
    for (const auto& z : p->mask_full) hmax = std::max(hmax, std::abs(z));
    shift = p->d.gamma + p->d.alpha * hmax;
  }
  if (shift_out) *shift_out = shift;
  const size_t nn = p->nn;
  std::vector<double> hv(nn);
  HostRng rng(seed, 0);
  double nv = 0.0;
  for (auto& z : hv) z = rng.next_normal();
  for (double z : hv) nv += z * z;
  nv = std::sqrt(nv);
  if (nv == 0.0) return -shift;
  std::vector<float> hf(nn);
  for (size_t i = 0; i < nn; ++i) hf[i] = static_cast<float>(hv[i] / nv);
  float* v = p->dx.p;      // current vector
  float* w = p->x_prev.p;  // operator output
  float* atav = p->mdx.p;  // A^T A v
  float* cv = p->has_mask ? ncsg_atu_buffer(p) : nullptr;  // C v
  float* av = p->adx.p;    // A v (range)
  NCSG_CUDA_CHECK(cudaMemcpyAsync(v, hf.data(), nn * 4, cudaMemcpyHostToDevice, s));
  DevBuf<double> red;
  red.alloc(static_cast<size_t>(dot_pair_blocks()) * 2);
  double lambda = 0.0;
  for (int it = 0; it < iters; ++it) {
    stacked_forward(p, v, p->dxT.p, av);
    if (p->d.kind != NCSG_DENOISE)
      proj_adjoint(p, av, p->range, p->bp_part.p, 1);
    launch_atu_assemble(atu_terms_for(p, av), atav, 1, s);
    if (cv) apply_filter(p, v, p->maskT_orig.p, cv);
    launch_screen_combine(v, atav, cv, static_cast<float>(p->d.alpha),
                          static_cast<float>(p->gamma_m), static_cast<float>(shift), w, nn, s);
    launch_dot_pair(v, w, w, w, nn, 1, red.p, s);
    auto d = read_dot_pairs(red.p, 1, s);
    lambda = d[0];
    const double nw = std::sqrt(d[1]);
    if (nw == 0.0) return -shift;
    launch_scale(w, static_cast<float>(1.0 / nw), v, nn, s);
  }
  return lambda - shift;
}

// cg (solvers.cpp:442-463) on NormalMap(stacked) (linear_map.cpp:57-61) for
// batch entry 0: x_out = n_iters CG steps from 0 for A^T A x = rhs.  The
// scalars (r.r, p.Ap) are fp64 reductions read back each step, as the
// reference's loop needs them on the host to decide its breaks.
void cg_solve(ncsg_problem* p, const float* rhs, int n_iters, double* x_out) {
  cudaStream_t s = p->stream.s;
  const size_t nn = p->nn;
  double* r = p->cg_r.p;
  double* q = p->cg_p.p;
  float* q32 = p->cg_p32.p;
  float* ap = p->cg_ap.p;
  const int nb = dot_pair_blocks();
  auto sum_blocks = [&]() {
    std::vector<double> h(nb);
    NCSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), p->red.p, nb * sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    double acc = 0.0;
    for (double v : h) acc += v;
    return acc;
  };
  NCSG_CUDA_CHECK(cudaMemsetAsync(x_out, 0, nn * sizeof(double), s));
  NCSG_CUDA_CHECK(cudaMemsetAsync(r, 0, nn * sizeof(double), s));
  NCSG_CUDA_CHECK(cudaMemsetAsync(q, 0, nn * sizeof(double), s));
  // r = rhs, p = rhs (fp64), p32 = rhs; r.r comes out of the same kernel
  NCSG_CUDA_CHECK(cudaMemcpyAsync(q32, rhs, nn * 4, cudaMemcpyDeviceToDevice, s));
  launch_cg_update(r, r, q, q32, -1.0, nn, p->red.p, s);  // r = 0 + 1 * rhs
  double rs = sum_blocks();
  launch_cg_direction(q, r, 0.0, q32, nn, s);              // p = r
  for (int it = 0; it < n_iters; ++it) {
    if (rs == 0.0) break;
    stacked_forward(p, q32, p->dxT.p, p->adx.p);
    if (p->d.kind != NCSG_DENOISE)
      proj_adjoint(p, p->adx.p, p->range, p->bp_part.p, 1);
    launch_atu_assemble(atu_terms_for(p, p->adx.p), ap, 1, s);
    launch_cg_dot(q, ap, nn, p->red.p, s);
    const double pap = sum_blocks();
    if (pap <= 0.0) break;
    const double a = rs / pap;
    launch_cg_update(x_out, r, q, ap, a, nn, p->red.p, s);
    const double rs_new = sum_blocks();
    const double beta = rs_new / rs;
    launch_cg_direction(q, r, beta, q32, nn, s);
    rs = rs_new;
  }
}

// Engine::step x-update in Cg mode (solvers.cpp:138-145): w = CG(A^T A, A^T u)
// / alpha; x -= w (x_old kept for the extrapolation), finiteness flag.
void x_update_cg(ncsg_problem* p) {
  cudaStream_t s = p->stream.s;
  ensure_scratch(p);
  float* atu = ncsg_atu_buffer(p);
  AtuTerms T = atu_terms(p);
  mark(p);
  launch_atu_assemble(T, atu, 1, s);
  mark(p);
  cg_solve(p, atu, p->n_cg, p->cg_x.p);
  mark(p);
  launch_x_update(p->x.p, p->x_old.p, p->cg_x.p, 1.0 / p->d.alpha, p->nn, p->flag.p, s);
  if (p->radon && !p->radon->orbit_mode) proj_prepare(p, p->x.p, p->xT.p, 1);  // x^T for class H
}

void upload_f64(ncsg_problem* p, const double* h, float* d, size_t count) {
  std::vector<float> tmp(count);
  for (size_t i = 0; i < count; ++i) tmp[i] = static_cast<float>(h[i]);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(d, tmp.data(), count * sizeof(float), cudaMemcpyHostToDevice,
                                  p->stream.s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(p->stream.s));
}

void download_f64(cudaStream_t s, const float* d, double* h, size_t count) {
  std::vector<float> tmp(count);
  NCSG_CUDA_CHECK(cudaMemcpyAsync(tmp.data(), d, count * sizeof(float), cudaMemcpyDeviceToHost, s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < count; ++i) h[i] = tmp[i];
}

}  // namespace

extern "C" {

const char* ncsg_last_error(void) { return g_err.c_str(); }
const char* ncsg_version(void) { return "0.1.0"; }

int ncsg_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int ncsg_default_detector_count(int n) {
  // default_detector_count (radon.cpp:10-13)
  int d = static_cast<int>(std::ceil(1.41421356237309504880 * n + 1.0));
  return d % 2 == 0 ? d + 1 : d;
}

ncsg_status ncsg_radon_create(int n, int n_angles, int n_det, int device, ncsg_radon** out) {
  return guard([&] {
    if (!out) throw Error{NCSG_INVALID, "null output handle"};
    Geometry geo = build_geometry(n, n_angles, n_det, 0, 0);
    require_device(device);
    auto r = std::make_unique<ncsg_radon>();
    r->dev.geo = std::move(geo);
    r->dev.device = device;
    r->dev.upload();
    NCSG_CUDA_CHECK(cudaStreamCreateWithFlags(&r->stream.s, cudaStreamNonBlocking));
    *out = r.release();
  });
}

ncsg_status ncsg_radon_destroy(ncsg_radon* r) {
  return guard([&] { delete r; });
}

size_t ncsg_radon_domain_size(const ncsg_radon* r) {
  return static_cast<size_t>(r->dev.geo.n) * r->dev.geo.n;
}
size_t ncsg_radon_range_size(const ncsg_radon* r) {
  return static_cast<size_t>(r->dev.geo.n_angles) * r->dev.geo.n_det;
}
int64_t ncsg_radon_sample_count(const ncsg_radon* r) { return r->dev.geo.samples; }

ncsg_status ncsg_radon_forward(const ncsg_radon* r, const float* x, float* out, int batch,
                               void* stream) {
  return guard([&] {
    if (!r || !x || !out || batch < 1) throw Error{NCSG_INVALID, "bad radon_forward arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(r->dev.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : r->stream.s;
    const Geometry& g = r->dev.geo;
    size_t nn = static_cast<size_t>(g.n) * g.n, m = static_cast<size_t>(g.n_angles) * g.n_det;
    DevBuf<float> xT, part;
    xT.alloc(4 * nn * batch);
    prepare_forward_aux(r->dev, x, xT.p, batch, s);
    part.alloc(m * r->dev.fp_slots() * batch);
    part.zero(s);
    launch_radon_forward_partial(r->dev, x, xT.p, part.p, batch, s);
    launch_strip_sum(r->dev, part.p, out, batch, s);
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

ncsg_status ncsg_radon_adjoint(const ncsg_radon* r, const float* u, float* out, int batch,
                               void* stream) {
  return guard([&] {
    if (!r || !u || !out || batch < 1) throw Error{NCSG_INVALID, "bad radon_adjoint arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(r->dev.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : r->stream.s;
    RadonDev& dev = const_cast<RadonDev&>(r->dev);
    dev.plan_adjoint(batch);
    const Geometry& g = dev.geo;
    size_t nn = static_cast<size_t>(g.n) * g.n;
    DevBuf<float> part, spec_dummy;
    part.alloc(nn * dev.n_partials() * batch);
    launch_radon_adjoint_partial(dev, u, 0, part.p, batch, s);
    // Sum partial images (class-H ones are transposed) via the combine path.
    launch_sum_partials(part.p, dev.bp_chunks[0], dev.bp_chunks[1], out, g.n, batch, s);
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

ncsg_status ncsg_fan_defaults(int n, double* source_radius, double* fan_angle) {
  return guard([&] {
    if (!source_radius || !fan_angle) throw Error{NCSG_INVALID, "null output"};
    fan_defaults(n, *source_radius, *fan_angle);
  });
}

static ncsg_status sparse_upload(SparseHost&& h, int device, ncsg_sparse** out) {
  return guard([&] {
    if (!out) throw Error{NCSG_INVALID, "null output handle"};
    require_device(device);
    NCSG_CUDA_CHECK(cudaSetDevice(device));
    auto a = std::make_unique<ncsg_sparse>();
    a->device = device;
    a->dev.upload(h);
    NCSG_CUDA_CHECK(cudaStreamCreateWithFlags(&a->stream.s, cudaStreamNonBlocking));
    *out = a.release();
  });
}

ncsg_status ncsg_fanbeam_create(int n, int views, int rays, double source_radius,
                                double fan_angle, int device, ncsg_sparse** out) {
  SparseHost h;
  ncsg_status st = guard([&] { h = build_fanbeam(n, views, rays, source_radius, fan_angle); });
  if (st != NCSG_OK) return st;
  return sparse_upload(std::move(h), device, out);
}

ncsg_status ncsg_sparse_create(int n, int views, int rays, int64_t nnz, const int64_t* rows,
                               const int64_t* cols, const double* vals, int device,
                               ncsg_sparse** out) {
  SparseHost h;
  ncsg_status st = guard([&] {
    if (n < 1 || views < 1 || rays < 1 || nnz < 0 || (nnz && (!rows || !cols || !vals)))
      throw Error{NCSG_INVALID, "bad sparse map arguments"};
    h = build_sparse(n, views, rays, std::vector<int64_t>(rows, rows + nnz),
                     std::vector<int64_t>(cols, cols + nnz),
                     std::vector<double>(vals, vals + nnz));
  });
  if (st != NCSG_OK) return st;
  return sparse_upload(std::move(h), device, out);
}

ncsg_status ncsg_sparse_destroy(ncsg_sparse* a) {
  return guard([&] { delete a; });
}

int64_t ncsg_sparse_nnz(const ncsg_sparse* a) { return a ? static_cast<int64_t>(a->dev.nnz) : 0; }

ncsg_status ncsg_sparse_forward(const ncsg_sparse* a, const float* x, float* out, int batch,
                                void* stream) {
  return guard([&] {
    if (!a || !x || !out || batch < 1) throw Error{NCSG_INVALID, "bad sparse_forward arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(a->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : a->stream.s;
    launch_sparse_forward(a->dev, x, a->dev.cols, out, a->dev.rows, batch, s);
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

ncsg_status ncsg_sparse_adjoint(const ncsg_sparse* a, const float* u, float* out, int batch,
                                void* stream) {
  return guard([&] {
    if (!a || !u || !out || batch < 1) throw Error{NCSG_INVALID, "bad sparse_adjoint arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(a->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : a->stream.s;
    launch_sparse_adjoint(a->dev, u, a->dev.rows, out, a->dev.cols, batch, s);
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

static ncsg_status sparse_host(const ncsg_sparse* a, const double* in, double* out, int batch,
                               bool adjoint) {
  return guard([&] {
    if (!a || !in || !out || batch < 1) throw Error{NCSG_INVALID, "bad sparse arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(a->device));
    const size_t ni = (adjoint ? a->dev.rows : a->dev.cols) * batch;
    const size_t no = (adjoint ? a->dev.cols : a->dev.rows) * batch;
    std::vector<float> hi(in, in + ni), ho(no);
    DevBuf<float> di, dout;
    di.alloc(ni);
    dout.alloc(no);
    NCSG_CUDA_CHECK(cudaMemcpy(di.p, hi.data(), ni * 4, cudaMemcpyHostToDevice));
    ncsg_status st = adjoint ? ncsg_sparse_adjoint(a, di.p, dout.p, batch, nullptr)
                             : ncsg_sparse_forward(a, di.p, dout.p, batch, nullptr);
    if (st != NCSG_OK) throw Error{st, g_err};
    NCSG_CUDA_CHECK(cudaMemcpy(ho.data(), dout.p, no * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < no; ++i) out[i] = ho[i];
  });
}

ncsg_status ncsg_sparse_forward_host(const ncsg_sparse* a, const double* x, double* out,
                                     int batch) {
  return sparse_host(a, x, out, batch, false);
}
ncsg_status ncsg_sparse_adjoint_host(const ncsg_sparse* a, const double* u, double* out,
                                     int batch) {
  return sparse_host(a, u, out, batch, true);
}

ncsg_status ncsg_radon_forward_host(const ncsg_radon* r, const double* x, double* out,
                                    int batch) {
  return guard([&] {
    if (!r || !x || !out || batch < 1) throw Error{NCSG_INVALID, "bad radon_forward arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(r->dev.device));
    size_t nn = ncsg_radon_domain_size(r) * batch, m = ncsg_radon_range_size(r) * batch;
    std::vector<float> hx(x, x + nn), hy(m);
    DevBuf<float> dx, dy;
    dx.alloc(nn);
    dy.alloc(m);
    NCSG_CUDA_CHECK(cudaMemcpy(dx.p, hx.data(), nn * sizeof(float), cudaMemcpyHostToDevice));
    ncsg_status st = ncsg_radon_forward(r, dx.p, dy.p, batch, nullptr);
    if (st != NCSG_OK) throw Error{st, g_err};
    NCSG_CUDA_CHECK(cudaMemcpy(hy.data(), dy.p, m * sizeof(float), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < m; ++i) out[i] = hy[i];
  });
}

ncsg_status ncsg_radon_adjoint_host(const ncsg_radon* r, const double* u, double* out,
                                    int batch) {
  return guard([&] {
    if (!r || !u || !out || batch < 1) throw Error{NCSG_INVALID, "bad radon_adjoint arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(r->dev.device));
    size_t nn = ncsg_radon_domain_size(r) * batch, m = ncsg_radon_range_size(r) * batch;
    std::vector<float> hu(u, u + m), hx(nn);
    DevBuf<float> du, dx;
    du.alloc(m);
    dx.alloc(nn);
    NCSG_CUDA_CHECK(cudaMemcpy(du.p, hu.data(), m * sizeof(float), cudaMemcpyHostToDevice));
    ncsg_status st = ncsg_radon_adjoint(r, du.p, dx.p, batch, nullptr);
    if (st != NCSG_OK) throw Error{st, g_err};
    NCSG_CUDA_CHECK(cudaMemcpy(hx.data(), dx.p, nn * sizeof(float), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nn; ++i) out[i] = hx[i];
  });
}

ncsg_status ncsg_grad_forward(int n, const float* x, float* out, int batch, void* stream) {
  return guard([&] {
    if (n < 2) throw Error{NCSG_INVALID, "grad needs N >= 2"};
    launch_grad_forward(x, out, n, batch, static_cast<cudaStream_t>(stream));
    NCSG_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  });
}

ncsg_status ncsg_grad_adjoint(int n, const float* g, float* out, int batch, void* stream) {
  return guard([&] {
    if (n < 2) throw Error{NCSG_INVALID, "grad needs N >= 2"};
    launch_grad_adjoint(g, out, n, batch, static_cast<cudaStream_t>(stream));
    NCSG_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  });
}

ncsg_status ncsg_grad_forward_host(int n, const double* x, double* out, int batch) {
  return guard([&] {
    if (n < 2) throw Error{NCSG_INVALID, "grad needs N >= 2"};
    require_device(0);
    size_t nn = static_cast<size_t>(n) * n * batch, gg = 2 * static_cast<size_t>(n) * (n - 1) * batch;
    std::vector<float> hx(x, x + nn), hg(gg);
    DevBuf<float> dx, dg;
    dx.alloc(nn);
    dg.alloc(gg);
    NCSG_CUDA_CHECK(cudaMemcpy(dx.p, hx.data(), nn * 4, cudaMemcpyHostToDevice));
    launch_grad_forward(dx.p, dg.p, n, batch, nullptr);
    NCSG_CUDA_CHECK(cudaMemcpy(hg.data(), dg.p, gg * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < gg; ++i) out[i] = hg[i];
  });
}

ncsg_status ncsg_grad_adjoint_host(int n, const double* g, double* out, int batch) {
  return guard([&] {
    if (n < 2) throw Error{NCSG_INVALID, "grad needs N >= 2"};
    require_device(0);
    size_t nn = static_cast<size_t>(n) * n * batch, gg = 2 * static_cast<size_t>(n) * (n - 1) * batch;
    std::vector<float> hg(g, g + gg), hx(nn);
    DevBuf<float> dx, dg;
    dx.alloc(nn);
    dg.alloc(gg);
    NCSG_CUDA_CHECK(cudaMemcpy(dg.p, hg.data(), gg * 4, cudaMemcpyHostToDevice));
    launch_grad_adjoint(dg.p, dx.p, n, batch, nullptr);
    NCSG_CUDA_CHECK(cudaMemcpy(hx.data(), dx.p, nn * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nn; ++i) out[i] = hx[i];
  });
}

ncsg_status ncsg_mask_apply_host(int n, const double* mask, const double* x, double* out,
                                 int batch, int device) {
  return guard([&] {
    if (!mask || !x || !out || batch < 1) throw Error{NCSG_INVALID, "bad mask_apply arguments"};
    require_device(device);
    Stream st;
    NCSG_CUDA_CHECK(cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking));
    FftPlan f;
    f.init(n, st.s);
    auto h = read_mask(n, mask);
    auto hm = half_mask(n, h, 1.0 / (static_cast<double>(n) * n));
    DevBuf<float2> mT, spec;
    mT.alloc(hm.size());
    NCSG_CUDA_CHECK(cudaMemcpy(mT.p, hm.data(), hm.size() * sizeof(float2), cudaMemcpyHostToDevice));
    size_t nn = static_cast<size_t>(n) * n * batch;
    std::vector<float> hx(x, x + nn);
    DevBuf<float> dx, dy;
    dx.alloc(nn);
    dy.alloc(nn);
    spec.alloc(static_cast<size_t>(n / 2 + 1) * n * batch);
    NCSG_CUDA_CHECK(cudaMemcpy(dx.p, hx.data(), nn * 4, cudaMemcpyHostToDevice));
    AtuTerms T;
    T.n = n;
    T.plain = dx.p;
    launch_fft_rows_r2c(f, T, spec.p, batch, st.s);
    launch_fft_cols_filter(f, spec.p, mT.p, batch, st.s);
    XUpdate xu;
    xu.x = dy.p;
    xu.subtract = 0;
    launch_fft_rows_c2r(f, spec.p, xu, batch, st.s);
    NCSG_CUDA_CHECK(cudaStreamSynchronize(st.s));
    NCSG_CUDA_CHECK(cudaMemcpy(hx.data(), dy.p, nn * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nn; ++i) out[i] = hx[i];
  });
}

// NCSG_SETUP_TIMES=1: host wall time of the problem-creation stages on stderr.
struct SetupClock {
  bool on = std::getenv("NCSG_SETUP_TIMES") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "ncsg setup %-18s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

ncsg_status ncsg_problem_create(const ncsg_problem_desc* desc, ncsg_problem** out) {
  SetupClock clk;
  return guard([&] {
    if (!desc || !out) throw Error{NCSG_INVALID, "null problem descriptor"};
    const ncsg_problem_desc& d = *desc;
    if (d.kind != NCSG_CT && d.kind != NCSG_DENOISE && d.kind != NCSG_PET)
      throw Error{NCSG_INVALID, "unknown problem kind"};
    if (d.n < 2) throw Error{NCSG_INVALID, "image size must be >= 2"};
    if (d.batch < 1) throw Error{NCSG_INVALID, "batch must be >= 1"};
    // assemble_problem / Engine validation (pipeline.cpp:74-77, solvers.cpp:91-106)
    if (!(d.alpha > 0.0) || !(d.beta > 0.0))
      throw Error{NCSG_INVALID, "alpha and beta must be positive"};
    if (d.lambda < 0.0) throw Error{NCSG_INVALID, "lambda must be nonnegative"};
    if (!d.mask && !d.m_pinv && !(d.gamma > 0.0))
      throw Error{NCSG_INVALID, "gamma must be positive when no mask is set"};
    if (!d.b) throw Error{NCSG_INVALID, "missing offset b"};
    auto p = std::make_unique<ncsg_problem>();
    p->d = d;
    p->d.mask = nullptr;
    p->d.b = nullptr;
    p->d.m_pinv = p->d.m_symbol = nullptr;  // host pointers: not kept
    p->device = d.device;
    p->batch = d.batch;
    p->nn = static_cast<size_t>(d.n) * d.n;
    p->g = 2 * static_cast<size_t>(d.n) * (d.n - 1);
    p->wd = static_cast<float>(d.beta / d.alpha);
    p->bound = static_cast<float>(d.lambda * d.alpha / d.beta);
    if (d.kind != NCSG_DENOISE && d.sparse) {
      // SparseMap data block (fan beam, sparse.cpp); the handle outlives the problem
      const SparseDev& A = d.sparse->dev;
      if (A.n != d.n) throw Error{NCSG_INVALID, "sparse map / image size mismatch"};
      if (d.angle_end > 0) throw Error{NCSG_INVALID, "sparse projectors are not angle-sharded"};
      require_device(d.device);
      if (d.sparse->device != d.device)
        throw Error{NCSG_INVALID, "sparse map lives on another device"};
      p->sparse = &A;
      p->d.n_angles = A.views;
      p->d.n_det = A.rays;
      p->m0 = A.rows;
      p->m_begin = 0;
      p->m_end = p->m0;
      p->rank0 = true;
    } else if (d.kind != NCSG_DENOISE) {
      Geometry geo = build_geometry(d.n, d.n_angles, d.n_det, d.angle_begin, d.angle_end,
                                    d.shard_rank, d.shard_count);
      clk.mark("geometry");
      p->m0 = static_cast<size_t>(d.n_angles) * d.n_det;
      int ab = d.angle_end > 0 ? d.angle_begin : 0;
      int ae = d.angle_end > 0 ? d.angle_end : d.n_angles;
      p->m_begin = static_cast<size_t>(ab) * d.n_det;
      p->m_end = static_cast<size_t>(ae) * d.n_det;
      p->rank0 = ab == 0;
      require_device(d.device);
      if (geo.orbit_sharded) {  // own rays = members of own orbits, scattered over [0, m0)
        p->rank0 = d.shard_rank == 0;
        p->sharded = true;
        std::vector<uint8_t> own(geo.own.begin(), geo.own.end());
        p->own_angle.alloc(own.size());
        NCSG_CUDA_CHECK(cudaMemcpy(p->own_angle.p, own.data(), own.size(), cudaMemcpyHostToDevice));
      } else if (d.angle_end > 0) {
        p->sharded = ab != 0 || ae != d.n_angles;
      }
      p->radon = std::make_unique<RadonDev>();
      p->radon->geo = std::move(geo);
      p->radon->device = d.device;
      p->radon->batch_hint = d.batch;
      p->radon->upload();
      clk.mark("upload");
      p->radon->plan_adjoint(d.batch);
      clk.mark("plan_adjoint");
    } else {
      p->m0 = p->nn;
      p->m_begin = 0;
      p->m_end = p->nn;
      require_device(d.device);
    }
    p->range = p->m0 + p->g + (d.positivity ? p->nn : 0);
    NCSG_CUDA_CHECK(cudaStreamCreateWithFlags(&p->stream.s, cudaStreamNonBlocking));
    cudaStream_t s = p->stream.s;
    clk.mark("stream");
    p->fft.init(d.n, s);
    clk.mark("fft plan");
    // Engine::Engine (solvers.cpp:93-99): m = gamma + alpha C, m_pinv = pinv(m)
    // (pinv_mask, circulant.cpp:47-55: 1/m where |m| > tol max|m|, else 0;
    // |m| compared squared and 1/m = conj(m)/|m|^2, the same filter to fp32).
    std::vector<float2> hm;  // herm(pinv(gamma + alpha C)) / N^2 on the half spectrum
    const double scale = 1.0 / (static_cast<double>(d.n) * d.n);
    p->gamma_m = d.gamma;
    if (desc->m_pinv) {
      // Override mode (mode_from, solvers.cpp:75-79; Engine::step :138-140):
      // w = m_pinv_override(A^T u), here a circulant given by its symbol; M
      // for the seminorm / screen is the m_override symbol, stored as
      // herm(M) / (alpha N^2) so that the Mask-mode kernels' gamma v +
      // alpha (C v) become M v with gamma_m = 0.
      p->override_mode = true;
      hm = half_mask(d.n, read_mask(d.n, desc->m_pinv), scale);
      if (desc->m_symbol) {
        p->has_mask = true;
        p->mask_full = read_mask(d.n, desc->m_symbol);
        auto ho = half_mask(d.n, p->mask_full, scale / d.alpha);
        p->maskT_orig.alloc(ho.size());
        NCSG_CUDA_CHECK(cudaMemcpy(p->maskT_orig.p, ho.data(), ho.size() * sizeof(float2),
                                   cudaMemcpyHostToDevice));
      }
      p->gamma_m = 0.0;
    } else if (desc->mask) {
      p->has_mask = true;
      p->mask_full = read_mask(d.n, desc->mask);
      clk.mark("  read mask");
      // m = gamma + alpha C and its pinv, bin by bin (no n^2 temporaries):
      // max |m|^2 first, then the filter's half spectrum straight from it
      // rel_tol passes through unchanged (pinv_mask: cutoff = rel_tol * max|m|;
      // 0 inverts every nonzero bin); the 1e-12 default lives in the wrappers
      const double tol = std::max(d.pinv_rel_tol, 0.0);
      const std::vector<std::complex<double>>& C = p->mask_full;
      const double ga = d.gamma, al = d.alpha;
      std::vector<double> part_max(64, 0.0);
      std::atomic<int> slot{0};
      parallel_rows(d.n, [&](int r0, int r1) {
        double mx = 0.0;
        for (size_t i = static_cast<size_t>(r0) * d.n; i < static_cast<size_t>(r1) * d.n; ++i)
          mx = std::max(mx, std::norm(ga + al * C[i]));
        part_max[slot++ % 64] = mx;
      });
      double hmax2 = 0.0;
      for (double v : part_max) hmax2 = std::max(hmax2, v);
      const double cutoff2 = tol * tol * hmax2;
      hm = half_mask_f(d.n, [&](size_t i) {
        const std::complex<double> z = ga + al * C[i];
        const double a = z.real(), bq = z.imag(), q = a * a + bq * bq;
        return q > cutoff2 ? std::complex<double>(a / q, -bq / q) : std::complex<double>(0.0);
      }, scale);
      clk.mark("  pinv");
      auto ho = half_mask(d.n, p->mask_full, scale);
      clk.mark("  half spectrum");
      p->maskT_orig.alloc(ho.size());
      NCSG_CUDA_CHECK(cudaMemcpy(p->maskT_orig.p, ho.data(), ho.size() * sizeof(float2),
                                 cudaMemcpyHostToDevice));
    } else {
      // pdhg: M = gamma I -> w = atu / gamma (solvers.cpp:133-137), applied
      // through the same filter path with a constant spectrum.
      hm = half_mask_f(d.n, [&](size_t) { return std::complex<double>(1.0 / d.gamma, 0.0); }, scale);
    }
    clk.mark("mask pinv");
    p->maskT.alloc(hm.size());
    NCSG_CUDA_CHECK(cudaMemcpy(p->maskT.p, hm.data(), hm.size() * sizeof(float2),
                               cudaMemcpyHostToDevice));
    clk.mark("filter upload");
    size_t xs = p->nn * p->batch;
    p->x.alloc(xs);
    p->x_old.alloc(xs);
    p->xT.alloc(4 * xs);  // x^T, or the interleaved orbit member images
    p->u.alloc(p->range * p->batch);
    p->b.alloc(p->m0 * p->batch);
    upload_f64(p.get(), desc->b, p->b.p, p->m0 * p->batch);
    if (d.kind != NCSG_DENOISE) {
      p->axs.alloc(p->m0 * p->batch);
      p->fp_part.alloc(p->m0 * proj_slots(p.get()) * p->batch);
      p->fp_part.zero(s);
      p->bp_part.alloc(p->nn * proj_parts(p.get()) * p->batch);
      p->axs.zero(s);
    }
    p->spec.alloc(static_cast<size_t>(d.n / 2 + 1) * d.n * p->batch);
    p->flag.alloc(3);
    p->red.alloc(static_cast<size_t>(p->batch) * objective_blocks() * 4);
    p->x.zero(s);
    p->x_old.zero(s);
    p->xT.zero(s);
    p->u.zero(s);
    if (p->radon && p->radon->bp_orbit) {  // zero padding and absent members stay zero
      p->u4.alloc(p->radon->u4_size() * p->batch);
      p->u4.zero(s);
    }
    reset_flag(p.get());
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    clk.mark("buffers");
    *out = p.release();
  });
}

ncsg_status ncsg_problem_destroy(ncsg_problem* p) {
  return guard([&] { delete p; });
}

size_t ncsg_problem_domain_size(const ncsg_problem* p) { return p->nn; }
size_t ncsg_problem_range_size(const ncsg_problem* p) { return p->range; }
void* ncsg_problem_stream(const ncsg_problem* p) { return p->stream.s; }
float* ncsg_state_x(ncsg_problem* p) { return p->x.p; }
float* ncsg_state_u(ncsg_problem* p) {
  p->u4_fresh = false;  // the caller may write u through this view
  return p->u.p;
}
float* ncsg_atu_buffer(ncsg_problem* p) {
  if (p->atu_ext) return p->atu_ext;
  if (!p->atu_own.n) p->atu_own.alloc(p->nn * p->batch);
  return p->atu_own.p;
}

ncsg_status ncsg_set_atu_buffer(ncsg_problem* p, float* dev_ptr) {
  return guard([&] {
    // phase B reads the buffer as float4 (the r2c loader's plain input)
    if (reinterpret_cast<uintptr_t>(dev_ptr) % 16 != 0)
      throw Error{NCSG_INVALID, "the A^T u buffer must be 16-byte aligned"};
    p->atu_ext = dev_ptr;
  });
}

ncsg_status ncsg_set_state(ncsg_problem* p, const double* x, const double* u, int64_t iter) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream.s;
    if (x)
      upload_f64(p, x, p->x.p, p->nn * p->batch);
    else
      p->x.zero(s);
    if (u)
      upload_f64(p, u, p->u.p, p->range * p->batch);
    else
      p->u.zero(s);
    p->u4_fresh = false;
    p->iter = iter;
    engine_init(p);
    reset_flag(p);
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

ncsg_status ncsg_get_state(ncsg_problem* p, double* x, double* u, int64_t* iter) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    if (x) download_f64(p->stream.s, p->x.p, x, p->nn * p->batch);
    if (u) download_f64(p->stream.s, p->u.p, u, p->range * p->batch);
    if (iter) *iter = p->iter;
  });
}

// A sharded problem holds only its rank's part of A^T u: its steps need the
// cross-rank sum between the phases (ncsg_step_phase_a / _b, or the
// communicator path), so the whole-step entry points refuse it without a
// communicator.
void reject_sharded(const ncsg_problem* p, const char* what) {
  if (p->sharded && !p->comm)
    throw Error{NCSG_INVALID, std::string(what) +
                                  " needs the unsharded problem (a sharded one steps through "
                                  "ncsg_step_phase_a/_b with the cross-rank sum in between, "
                                  "or with a communicator: ncsg_problem_set_comm)"};
}

ncsg_status ncsg_step(ncsg_problem* p, int iters) {
  return guard([&] {
    reject_sharded(p, "ncsg_step");
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    for (int k = 0; k < iters; ++k) do_step(p);
    p->iter += iters;
  });
}

ncsg_status ncsg_step_graph(ncsg_problem* p, int iters) {
  return guard([&] {
    reject_sharded(p, "ncsg_step_graph");
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    if (iters <= 0) return;
    if (p->n_cg > 0 || (p->comm && !p->comm->capturable())) {
      // CG reads its scalars back every step, host-driven transports
      // synchronise inside the step: neither is capturable
      for (int k = 0; k < iters; ++k) do_step(p);
      p->iter += iters;
      return;
    }
    refresh_u4(p);  // the captured steps read u4 from their first adjoint on
    auto it = p->graphs.find(iters);
    if (it == p->graphs.end()) {
      cudaGraph_t graph;
      NCSG_CUDA_CHECK(cudaStreamBeginCapture(p->stream.s, cudaStreamCaptureModeThreadLocal));
      try {
        for (int k = 0; k < iters; ++k) do_step(p);
      } catch (...) {
        cudaStreamEndCapture(p->stream.s, &graph);
        throw;
      }
      NCSG_CUDA_CHECK(cudaStreamEndCapture(p->stream.s, &graph));
      cudaGraphExec_t exec;
      NCSG_CUDA_CHECK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      it = p->graphs.emplace(iters, exec).first;
    }
    NCSG_CUDA_CHECK(cudaGraphLaunch(it->second, p->stream.s));
    p->iter += iters;
  });
}

ncsg_status ncsg_sync(ncsg_problem* p, int64_t* diverged_iter) {
  ncsg_status st = guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    check_divergence(p, diverged_iter);
  });
  return st;
}

ncsg_status ncsg_objective(ncsg_problem* p, double* out) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    auto f = objective_values(p);
    std::copy(f.begin(), f.end(), out);
  });
}

ncsg_status ncsg_last_seminorm(ncsg_problem* p, double* out) {
  return guard([&] {
    if (!p->x_prev.n) throw Error{NCSG_INVALID, "no recorded step to measure"};
    auto v = seminorm_values(p);
    std::copy(v.begin(), v.end(), out);
  });
}

ncsg_status ncsg_profile_begin(ncsg_problem* p) {
  return guard([&] {
    p->profiling = true;
    p->ev_used = 0;
  });
}

ncsg_status ncsg_profile_end(ncsg_problem* p, double* phase_ms, int n_phase, int* steps) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaStreamSynchronize(p->stream.s));
    p->profiling = false;
    const size_t per = kPhases + 1;
    const size_t ns = p->ev_used / per;
    for (int k = 0; k < n_phase; ++k) phase_ms[k] = 0.0;
    for (size_t st = 0; st < ns; ++st)
      for (int k = 0; k < kPhases && k < n_phase; ++k) {
        float ms = 0.f;
        NCSG_CUDA_CHECK(cudaEventElapsedTime(&ms, p->events[st * per + k], p->events[st * per + k + 1]));
        phase_ms[k] += ms;
      }
    if (steps) *steps = static_cast<int>(ns);
    p->ev_used = 0;
  });
}

int64_t ncsg_launch_count(void) { return ncsg::launch_count(); }

struct ncsg_comm {
  std::unique_ptr<ncsg::Comm> c;
};

ncsg_status ncsg_nccl_unique_id(unsigned char id[128]) {
  return guard([&] { ncsg::nccl_unique_id(id); });
}

ncsg_status ncsg_comm_create_nccl(const unsigned char id[128], int rank, int nranks, int device,
                                  ncsg_comm** out) {
  return guard([&] {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
      throw Error{NCSG_INVALID, "invalid NCCL communicator arguments"};
    auto c = std::make_unique<ncsg_comm>();
    c->c.reset(ncsg::make_nccl_comm(id, rank, nranks, device));
    *out = c.release();
  });
}

ncsg_status ncsg_comm_create_callbacks(const ncsg_comm_ops* ops, ncsg_comm** out) {
  return guard([&] {
    if (!ops || !out || ops->nranks < 1 || ops->rank < 0 || ops->rank >= ops->nranks)
      throw Error{NCSG_INVALID, "invalid communicator callbacks"};
    auto c = std::make_unique<ncsg_comm>();
    c->c.reset(ncsg::make_callback_comm(*ops));
    *out = c.release();
  });
}

ncsg_status ncsg_comm_create_local(int nranks, ncsg_comm** out) {
  return guard([&] {
    if (!out || nranks < 1) throw Error{NCSG_INVALID, "invalid local group size"};
    auto g = ncsg::make_local_group(nranks);
    for (int r = 0; r < nranks; ++r) {
      out[r] = new ncsg_comm;
      out[r]->c.reset(g[r]);
    }
  });
}

ncsg_status ncsg_comm_create_null(int rank, int nranks, ncsg_comm** out) {
  return guard([&] {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks)
      throw Error{NCSG_INVALID, "invalid null communicator arguments"};
    auto c = std::make_unique<ncsg_comm>();
    c->c.reset(ncsg::make_null_comm(rank, nranks));
    *out = c.release();
  });
}

ncsg_status ncsg_comm_destroy(ncsg_comm* c) {
  return guard([&] { delete c; });
}

ncsg_status ncsg_problem_set_comm(ncsg_problem* p, ncsg_comm* c, int exchange) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);  // captured without / with it
    p->graphs.clear();
    if (!c) {
      p->comm = nullptr;
      return;
    }
    ncsg::Comm& C = *c->c;
    if (exchange != NCSG_XCHG_ALLREDUCE && exchange != NCSG_XCHG_SLAB &&
        exchange != NCSG_XCHG_P2P)
      throw Error{NCSG_INVALID, "unknown exchange mode"};
    if (p->n_cg > 0) throw Error{NCSG_INVALID, "the CG x-update needs the unsharded problem"};
    if (p->d.shard_count > 1 && (p->d.shard_count != C.nranks() || p->d.shard_rank != C.rank()))
      throw Error{NCSG_INVALID, "orbit shard does not match the communicator's rank / size"};
    const int n = p->d.n, P = C.nranks();
    p->atu_full.alloc(p->nn * p->batch);
    if (exchange != NCSG_XCHG_ALLREDUCE) {
      const int R = n / P;
      if (p->batch != 1) throw Error{NCSG_INVALID, "the slab FFT runs one problem (batch 1)"};
      if (n % P != 0 || R % 2 != 0 || (R & (R - 1)) != 0)
        throw Error{NCSG_INVALID, "the slab FFT needs N / ranks to be an even power of two"};
      const int nk = n / 2 + 1, wc = (nk + P - 1) / P;
      p->slab_R = R;
      p->slab_logR = 0;
      while ((1 << p->slab_logR) < R) ++p->slab_logR;
      p->slab_wc = wc;
      p->atu_slab.alloc(static_cast<size_t>(R) * n);
      p->spec_slab.alloc(static_cast<size_t>(P) * wc * R);
      p->spec_recv.alloc(static_cast<size_t>(P) * wc * R);
      p->spec_slab.zero(p->stream.s);  // padded columns stay finite
      p->spec_recv.zero(p->stream.s);
      p->maskT_pad.alloc(static_cast<size_t>(P) * wc * n);
      p->maskT_pad.zero(p->stream.s);
      NCSG_CUDA_CHECK(cudaMemcpyAsync(p->maskT_pad.p, p->maskT.p,
                                      static_cast<size_t>(nk) * n * sizeof(float2),
                                      cudaMemcpyDeviceToDevice, p->stream.s));
      ensure_scratch(p);
      if (exchange == NCSG_XCHG_P2P) {
        if (P > kMaxPeers) throw Error{NCSG_INVALID, "the P2P exchange spans at most 8 ranks"};
        p->recv_slots.alloc(static_cast<size_t>(P) * R * n);
        NCSG_CUDA_CHECK(cudaStreamSynchronize(p->stream.s));
        auto share = [&](void* mine, PeerPtrs& out) {
          std::vector<void*> v = C.share_pointers(mine);
          if (static_cast<int>(v.size()) != P)
            throw Error{NCSG_INVALID, std::string("the ") + C.name() +
                                          " transport has no peer memory for the P2P exchange"};
          for (int q = 0; q < P; ++q) out.p[q] = v[q];
        };
        share(p->recv_slots.p, p->peer_slots);
        share(p->spec_recv.p, p->peer_recv);
        share(p->spec_slab.p, p->peer_slab);
        share(p->x.p, p->peer_x);
      }
    }
    NCSG_CUDA_CHECK(cudaStreamSynchronize(p->stream.s));
    p->comm = &C;
    p->xchg = exchange;
  });
}

ncsg_status ncsg_problem_plan(const ncsg_problem* p, ncsg_plan_info* out) {
  return guard([&] {
    if (!p || !out) throw Error{NCSG_INVALID, "null argument"};
    ncsg_plan_info r{};
    if (p->radon) {
      r.orbit_forward = p->radon->orbit_mode ? 1 : 0;
      r.gather_adjoint = p->radon->bp_orbit ? 1 : 0;
      r.n_orbits = static_cast<int>(p->radon->geo.orbits.size());
      r.samples = p->radon->geo.samples;
      r.transposed_copy = (!p->radon->orbit_mode && !p->radon->geo.cls[1].empty()) ? 1 : 0;
      r.adjoint_table_bytes =
          p->radon->bp_orbit && p->radon->ga_wtab_state == 1
              ? static_cast<int64_t>(p->radon->ga_wtab.n * sizeof(uint4))
              : 0;
    }
    if (p->d.kind != NCSG_DENOISE) {
      r.fp_slots = proj_slots(p);
      r.bp_partials = proj_parts(p);
    }
    r.m0 = static_cast<int64_t>(p->m0);
    r.g = static_cast<int64_t>(p->g);
    r.range = static_cast<int64_t>(p->range);
    r.batch = p->batch;
    DualFuse df;
    r.dual_fused = fuse_dual_terms(p, df) ? 1 : 0;
    *out = r;
  });
}

ncsg_status ncsg_step_phase_a(ncsg_problem* p) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    phase_a(p);
    launch_atu_assemble(atu_terms(p), ncsg_atu_buffer(p), p->batch, p->stream.s);
  });
}

ncsg_status ncsg_step_phase_b(ncsg_problem* p) {
  return guard([&] {
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    phase_b(p, ncsg_atu_buffer(p));
    p->iter += 1;
  });
}

ncsg_status ncsg_solve(ncsg_problem* p, int max_iters, int record_every,
                       int check_step_condition, uint64_t seed, const double* f_star,
                       ncsg_record_row* rows, int max_rows, int* n_rows, double* screen_est) {
  return guard([&] {
    // solve_template (solvers.cpp:267-337)
    if (max_iters < 0) throw Error{NCSG_INVALID, "max_iters must be nonnegative"};
    if (record_every < 1) throw Error{NCSG_INVALID, "record_every must be >= 1"};
    reject_sharded(p, "ncsg_solve");
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream.s;
    p->iter = 0;
    engine_init(p);
    reset_flag(p);
    if (screen_est) *screen_est = NAN;
    if (check_step_condition && p->n_cg == 0) {  // solvers.cpp:207, 278 (warning only)
      if (p->sharded)
        throw Error{NCSG_INVALID, "the step-condition screen needs the unsharded problem"};
      double e = screen_estimate(p, seed, 40, nullptr);
      if (screen_est) *screen_est = e;
    }
    const int B = p->batch;
    std::vector<std::vector<ncsg_record_row>> rec(B);
    auto t0 = std::chrono::steady_clock::now();
    auto emit = [&](int64_t k, const std::vector<double>& sem) {
      auto f = objective_values(p);
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      const int64_t axis = p->n_cg > 0 ? p->n_cg : 1;  // solvers.cpp:279
      for (int b = 0; b < B; ++b) rec[b].push_back({k * axis, f[b], 0.0, sem[b], ms});
    };
    emit(0, std::vector<double>(B, 0.0));
    ensure_scratch(p);
    int k = 1;
    while (k <= max_iters) {
      // next recorded step: the smallest multiple of record_every >= k, or the last
      int next = ((k + record_every - 1) / record_every) * record_every;
      next = std::min(next, max_iters);
      int plain = next - k;  // unrecorded steps before it
      if (plain > 0) {
        for (int j = 0; j < plain; ++j) do_step(p);
        p->iter += plain;
      }
      NCSG_CUDA_CHECK(cudaMemcpyAsync(p->x_prev.p, p->x.p, p->nn * B * 4, cudaMemcpyDeviceToDevice, s));
      NCSG_CUDA_CHECK(cudaMemcpyAsync(p->u_prev.p, p->u.p, p->range * B * 4, cudaMemcpyDeviceToDevice, s));
      do_step(p);
      p->iter += 1;
      check_divergence(p);
      emit(next, seminorm_values(p));
      k = next + 1;
    }
    // rel_subopt against f_star or the best objective seen (solvers.cpp:321-332)
    int nr = static_cast<int>(rec[0].size());
    for (int b = 0; b < B; ++b) {
      double f_ref;
      if (f_star) {
        f_ref = f_star[b];
      } else {
        f_ref = INFINITY;
        for (auto& r : rec[b]) f_ref = std::min(f_ref, r.objective);
      }
      for (auto& r : rec[b])
        r.rel_subopt = std::isfinite(f_ref) ? (r.objective - f_ref) / std::max(1.0, std::abs(f_ref)) : 0.0;
      for (int i = 0; i < std::min(nr, max_rows); ++i) rows[static_cast<size_t>(b) * max_rows + i] = rec[b][i];
    }
    if (n_rows) *n_rows = std::min(nr, max_rows);
  });
}


ncsg_status ncsg_set_cg(ncsg_problem* p, int n_cg) {
  return guard([&] {
    // admm_cg_solve (solvers.cpp:435-440) / Engine Cg mode (solvers.cpp:111-113)
    if (n_cg < 0) throw Error{NCSG_INVALID, "n_cg must be >= 1"};
    if (n_cg > 0) {
      if (p->has_mask || p->override_mode)
        throw Error{NCSG_INVALID, "admm_cg uses M = alpha A^T A; drop the mask/overrides"};
      if (p->batch != 1) throw Error{NCSG_INVALID, "the CG x-update runs one problem (batch 1)"};
      if (p->sharded) throw Error{NCSG_INVALID, "the CG x-update needs the unsharded problem"};
      NCSG_CUDA_CHECK(cudaSetDevice(p->device));
      if (!p->cg_x.n) {
        p->cg_x.alloc(p->nn);
        p->cg_r.alloc(p->nn);
        p->cg_p.alloc(p->nn);
        p->cg_p32.alloc(p->nn);
        p->cg_ap.alloc(p->nn);
      }
    }
    p->n_cg = n_cg;
  });
}

/* ---------------------------------------------------------------- setup path */

ncsg_status ncsg_calibrate_scale(const ncsg_radon* r, int n_samples, uint64_t seed,
                                 double* scale) {
  return guard([&] {
    // calibrate_scale(NormalMap(R), radon_mask(n, 1, 1), n_samples, seed)
    // (circulant.cpp:142-169, called by measurement_mask, pipeline.cpp:100-110).
    // With T = F^-1 diag(t) F (t = template, DC bin excluded; real and even),
    //   num = sum_bins Re(conj(t Fv) F(R^T R v)) = N^2 <T v, R^T R v>,
    //   den = sum_bins |t Fv|^2                  = N^2 <T v, T v>,
    // so each probe needs R, R^T and one real filter pass.
    if (!r || !scale) throw Error{NCSG_INVALID, "bad calibrate_scale arguments"};
    if (n_samples < 1) throw Error{NCSG_INVALID, "n_samples must be positive"};
    NCSG_CUDA_CHECK(cudaSetDevice(r->dev.device));
    RadonDev& dev = const_cast<RadonDev&>(r->dev);
    const Geometry& g = dev.geo;
    const int n = g.n;
    cudaStream_t s = r->stream.s;
    const size_t nn = static_cast<size_t>(n) * n, m = static_cast<size_t>(g.n_angles) * g.n_det;
    std::vector<std::complex<double>> t(nn);
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const double mj = std::min(j, n - j), mk = std::min(k, n - k);
        t[static_cast<size_t>(j) * n + k] = (j == 0 && k == 0) ? 0.0 : 1.0 / std::sqrt(mj * mj + mk * mk);
      }
    FftPlan f;
    f.init(n, s);
    auto hm = half_mask(n, t, 1.0 / static_cast<double>(nn));
    DevBuf<float2> mT;
    mT.alloc(hm.size());
    NCSG_CUDA_CHECK(cudaMemcpy(mT.p, hm.data(), hm.size() * sizeof(float2), cudaMemcpyHostToDevice));
    const int B = std::min(n_samples, 8);
    dev.plan_adjoint(B);
    DevBuf<float> v, av, y, aux, sino, fpart, bpart;
    DevBuf<float2> spec;
    DevBuf<double> red;
    v.alloc(nn * B);
    av.alloc(nn * B);
    y.alloc(nn * B);
    aux.alloc(4 * nn * B);
    sino.alloc(m * B);
    fpart.alloc(m * dev.fp_slots() * B);
    fpart.zero(s);
    bpart.alloc(nn * dev.n_partials() * B);
    spec.alloc(static_cast<size_t>(n / 2 + 1) * n * B);
    red.alloc(static_cast<size_t>(dot_pair_blocks()) * 2 * B);
    std::vector<float> hv(nn * B);
    double num = 0.0, den = 0.0;
    for (int s0 = 0; s0 < n_samples; s0 += B) {
      const int nb = std::min(B, n_samples - s0);
      for (int b = 0; b < nb; ++b) {  // probe_image (circulant.cpp:89-94)
        HostRng rng(seed, static_cast<uint64_t>(s0 + b));
        for (size_t i = 0; i < nn; ++i) hv[b * nn + i] = static_cast<float>(rng.next_normal());
      }
      NCSG_CUDA_CHECK(cudaMemcpyAsync(v.p, hv.data(), nb * nn * 4, cudaMemcpyHostToDevice, s));
      prepare_forward_aux(dev, v.p, aux.p, nb, s);
      launch_radon_forward_partial(dev, v.p, aux.p, fpart.p, nb, s);
      launch_strip_sum(dev, fpart.p, sino.p, nb, s);
      launch_radon_adjoint_partial(dev, sino.p, 0, bpart.p, nb, s);
      launch_sum_partials(bpart.p, dev.bp_chunks[0], dev.bp_chunks[1], av.p, n, nb, s);
      AtuTerms T;
      T.n = n;
      T.plain = v.p;
      launch_fft_rows_r2c(f, T, spec.p, nb, s);
      launch_fft_cols_filter(f, spec.p, mT.p, nb, s);
      XUpdate xu;
      xu.x = y.p;
      xu.subtract = 0;
      launch_fft_rows_c2r(f, spec.p, xu, nb, s);
      launch_dot_pair(y.p, av.p, y.p, y.p, nn, nb, red.p, s);
      auto sums = read_dot_pairs(red.p, nb, s);
      for (int b = 0; b < nb; ++b) {
        num += sums[2 * b];
        den += sums[2 * b + 1];
      }
    }
    if (den == 0.0) throw Error{NCSG_INVALID, "calibrate_scale: template response is zero"};
    *scale = num / den;
  });
}

ncsg_status ncsg_sparse_empirical_mask(const ncsg_sparse* a, int n_samples, uint64_t seed,
                                       double* mask, int* n_dead) {
  return guard([&] {
    // measurement_mask for non-parallel geometry: empirical_mask(NormalMap(A),
    // n, samples, seed) (pipeline.cpp:100-110, circulant.cpp:98-140).  Per bin
    // the mean over probes of F(A^T A v) / F(v), skipping bins with
    // |F v| < 1e-12 ||F v||; computed on half spectra (F v of a real v is
    // conjugate-symmetric) and expanded to the full N x N mask on the host.
    if (!a || !mask) throw Error{NCSG_INVALID, "bad empirical_mask arguments"};
    if (n_samples < 1) throw Error{NCSG_INVALID, "n_samples must be positive"};
    const SparseDev& A = a->dev;
    const int n = A.n;
    NCSG_CUDA_CHECK(cudaSetDevice(a->device));
    cudaStream_t s = a->stream.s;
    const size_t nn = A.cols, nk = static_cast<size_t>(n / 2 + 1), half = nk * n;
    FftPlan f;
    f.init(n, s);
    const int B = std::min(n_samples, 8);
    DevBuf<float> v, mid, av;
    DevBuf<float2> fv, fav;
    DevBuf<double2> sum;
    DevBuf<int> hits;
    DevBuf<double> red, cut;
    v.alloc(nn * B);
    av.alloc(nn * B);
    mid.alloc(A.rows * B);
    fv.alloc(half * B);
    fav.alloc(half * B);
    sum.alloc(half);
    hits.alloc(half);
    red.alloc(static_cast<size_t>(dot_pair_blocks()) * B);
    cut.alloc(B);
    NCSG_CUDA_CHECK(cudaMemsetAsync(sum.p, 0, half * sizeof(double2), s));
    NCSG_CUDA_CHECK(cudaMemsetAsync(hits.p, 0, half * sizeof(int), s));
    std::vector<float> hv(nn * B);
    for (int s0 = 0; s0 < n_samples; s0 += B) {
      const int nb = std::min(B, n_samples - s0);
      for (int b = 0; b < nb; ++b) {  // probe_image (circulant.cpp:89-94)
        HostRng rng(seed, static_cast<uint64_t>(s0 + b));
        for (size_t i = 0; i < nn; ++i) hv[b * nn + i] = static_cast<float>(rng.next_normal());
      }
      NCSG_CUDA_CHECK(cudaMemcpyAsync(v.p, hv.data(), nb * nn * 4, cudaMemcpyHostToDevice, s));
      launch_sparse_forward(A, v.p, nn, mid.p, A.rows, nb, s);
      launch_sparse_adjoint(A, mid.p, A.rows, av.p, nn, nb, s);
      AtuTerms T;
      T.n = n;
      T.plain = v.p;
      launch_fft_rows_r2c(f, T, fv.p, nb, s);
      launch_fft_cols_forward(f, fv.p, nb, s);
      T.plain = av.p;
      launch_fft_rows_r2c(f, T, fav.p, nb, s);
      launch_fft_cols_forward(f, fav.p, nb, s);
      launch_spec_norm(fv.p, n, nb, red.p, s);
      std::vector<double> h(static_cast<size_t>(dot_pair_blocks()) * nb), cutoff(nb, 0.0);
      NCSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), red.p, h.size() * sizeof(double),
                                      cudaMemcpyDeviceToHost, s));
      NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
      for (int b = 0; b < nb; ++b) {
        double acc = 0.0;
        for (int k = 0; k < dot_pair_blocks(); ++k) acc += h[static_cast<size_t>(b) * dot_pair_blocks() + k];
        cutoff[b] = 1e-12 * std::sqrt(acc);
      }
      NCSG_CUDA_CHECK(cudaMemcpyAsync(cut.p, cutoff.data(), nb * sizeof(double),
                                      cudaMemcpyHostToDevice, s));
      launch_mask_accumulate(fv.p, fav.p, cut.p, nb, half, sum.p, hits.p, s);
    }
    std::vector<double2> hs(half);
    std::vector<int> hh(half);
    NCSG_CUDA_CHECK(cudaMemcpyAsync(hs.data(), sum.p, half * sizeof(double2),
                                    cudaMemcpyDeviceToHost, s));
    NCSG_CUDA_CHECK(cudaMemcpyAsync(hh.data(), hits.p, half * sizeof(int), cudaMemcpyDeviceToHost, s));
    NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
    int dead = 0;
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        // bin (j, k) = row frequency j, column frequency k; half spectrum holds k <= n/2
        const bool direct = k <= n / 2;
        const size_t src = direct ? static_cast<size_t>(k) * n + j
                                  : static_cast<size_t>(n - k) * n + (n - j) % n;
        double* o = mask + 2 * (static_cast<size_t>(j) * n + k);
        if (hh[src] == 0) {
          o[0] = o[1] = 0.0;
          ++dead;
          continue;
        }
        o[0] = hs[src].x / hh[src];
        o[1] = (direct ? 1.0 : -1.0) * hs[src].y / hh[src];
      }
    if (n_dead) *n_dead = dead;
  });
}

ncsg_status ncsg_radon_dc_response(const ncsg_radon* r, double* dc) {
  return guard([&] {
    // <1, R^T R 1> / N^2 = ||R 1||^2 / N^2: the DC bin of radon_mask.
    if (!r || !dc) throw Error{NCSG_INVALID, "bad dc_response arguments"};
    NCSG_CUDA_CHECK(cudaSetDevice(r->dev.device));
    const RadonDev& dev = r->dev;
    cudaStream_t s = r->stream.s;
    const size_t nn = static_cast<size_t>(dev.geo.n) * dev.geo.n;
    const size_t m = static_cast<size_t>(dev.geo.n_angles) * dev.geo.n_det;
    DevBuf<float> one, aux, sino, fpart;
    DevBuf<double> red;
    one.alloc(nn);
    std::vector<float> h(nn, 1.0f);
    NCSG_CUDA_CHECK(cudaMemcpyAsync(one.p, h.data(), nn * 4, cudaMemcpyHostToDevice, s));
    aux.alloc(4 * nn);
    sino.alloc(m);
    fpart.alloc(m * dev.fp_slots());
    fpart.zero(s);
    red.alloc(static_cast<size_t>(dot_pair_blocks()) * 2);
    prepare_forward_aux(dev, one.p, aux.p, 1, s);
    launch_radon_forward_partial(dev, one.p, aux.p, fpart.p, 1, s);
    launch_strip_sum(dev, fpart.p, sino.p, 1, s);
    launch_dot_pair(sino.p, sino.p, sino.p, sino.p, m, 1, red.p, s);
    *dc = read_dot_pairs(red.p, 1, s)[0] / static_cast<double>(nn);
  });
}

ncsg_status ncsg_screen_step_condition(ncsg_problem* p, uint64_t seed, int iters, double* est,
                                       double* shift_out) {
  return guard([&] {
    if (!p || !est) throw Error{NCSG_INVALID, "bad screen arguments"};
    if (iters < 1) throw Error{NCSG_INVALID, "iters must be positive"};
    if (p->sharded)
      throw Error{NCSG_INVALID, "the step-condition screen needs the unsharded problem"};
    NCSG_CUDA_CHECK(cudaSetDevice(p->device));
    *est = screen_estimate(p, seed, iters, shift_out);
  });
}

}  // extern "C"
