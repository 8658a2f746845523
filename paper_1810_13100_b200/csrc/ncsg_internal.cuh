// Internal declarations of the B200 NCS hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ncsg.h"

namespace ncsg {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
// Kernel launches issued by this library (bench.py's gpu_launches).
int64_t launch_count();
void count_launch(int k = 1);
struct Error {
  ncsg_status code;
  std::string msg;
};

#define NCSG_CUDA_CHECK(expr)                                                        \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      throw ::ncsg::Error{NCSG_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

// ------------------------------------------------- programmatic launches
// The NCS step's kernels are launched with programmatic stream serialization
// (PDL): each may be scheduled while its predecessor drains and waits in
// pdl_wait() -- its first statement, before any global access -- until the
// predecessor has completed and its writes are visible. NCSG_NO_PDL=1 turns
// it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size): the attribute only ever grows, so repeated launches skip the call.
void ensure_smem(const void* kernel, size_t bytes);
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  NCSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// ------------------------------------------------------------- geometry
// Fixed-point sample positions: value * 2^-32 pixels, int64.  The lattice
// point (s, tau) of angle t sits at
//   px = P0 + s*ax + tau*bx,   py = P0 + s*ay + tau*by   (P0 = c * 2^32)
// with ax = round(cos*2^32), ay = bx = round(-sin*2^32), by = round(-cos*2^32):
// the exact-math positions of radon.cpp:52-66 to 4e-7 px, computed in exact
// integer arithmetic so every kernel agrees on every sample's cell.
//
// Kernel frame: class V angles (|cos| >= |sin|) use (X, Y) = (px, py) on the
// image; class H angles use (X, Y) = (py, px) on the transposed image, so that
// in both classes one sample step advances Y by dY >= 0.707 px and |dX| <= dY.
struct AngleGeom {
  long long aX, aY;  // per unit s (kernel frame)
  long long dX, dY;  // per step (tau advanced by `dir`), dY > 0
  int t;             // angle index into the sinogram
  int dir;           // tau = dir * k
  float aXf, aYf;    // aX, aY as floats in pixel units (range estimates)
  float inv_dY16;    // 65536 / dY  (step estimates on (diff >> 16))
  float inv_adX16;   // 65536 / |dX| (0 when dX == 0)
  int dXq, dYq;      // dX, dY rounded to Q9.23 (tile-local stepping)
  int bp_stride;     // adjoint lane ray stride (>= 3), chosen per angle on the host
  int fp_rq;         // orbit forward: rays per quarter-warp (4..8, host bank-cost model)
};

struct RayRange {  // valid tau interval [first, last] of one ray (empty: first > last)
  int first, last;
};

// Dihedral orbit of an angle theta in [0, 45 deg] (n_angles % 4 == 0): the
// members theta, theta+90, 180-theta, 90-theta sample the image at the
// images of theta's lattice under the grid symmetries, so R for all four is
// theta's lattice walk over four transformed copies of x (planes):
//   plane 0: x,  plane 1: x1[r][c] = x[N-1-c][r],  plane 2: x2[r][c] = x[r][N-1-c],
//   plane 3: x3[r][c] = x[N-1-c][N-1-r].
// Members 2 and 3 walk tau in the opposite direction (neg).  t[k] < 0: the
// member coincides with another one (theta = 0 or 45 deg).
struct OrbitGeom {
  AngleGeom rep;  // theta's class-V geometry (kernel frame = image frame)
  int t[4];
};

struct Geometry {
  int n = 0, n_angles = 0, n_det = 0;
  int s_mid = 0;
  long long P0 = 0;
  std::vector<AngleGeom> cls[2];   // class 0 = V, class 1 = H
  std::vector<RayRange> rays;      // [t][d]
  std::vector<OrbitGeom> orbits;   // filled when every angle belongs to an orbit
  std::vector<uint8_t> own;        // own[t]: angle t belongs to this shard
  bool orbit_sharded = false;
  bool strides_ready = false;      // AngleGeom::bp_stride chosen (choose_adjoint_strides)
  int64_t samples = 0;
};
// Orbit representative of angle t (n_angles % 4 == 0): the member in [0, A/4].
inline int orbit_rep(int t, int n_angles) {
  const int q = n_angles / 4;
  if (t <= q) return t;
  if (t < 2 * q) return 2 * q - t;
  if (t <= 3 * q) return t - 2 * q;
  return n_angles - t;
}

// Replays the reference's fp64 ray table and per-sample box check
// (radon.cpp:35-72, 85-90) and builds the fixed-point angle table.
// Throws Error{NCSG_INVALID} with the reference's messages.
Geometry build_geometry(int n, int n_angles, int n_det, int angle_begin, int angle_end,
                        int shard_rank = 0, int shard_count = 0);
// Lane strides of the per-angle scatter adjoint (once per geometry).
void choose_adjoint_strides(Geometry& g);

// Explicit sparse projector (SparseMap, sparse.cpp): CSR over sinogram rows
// (view-major) and its stored transpose over image pixels, fp64 on the host.
struct SparseHost {
  int n = 0, views = 0, rays = 0;
  std::vector<int64_t> row_ptr, t_row_ptr;
  std::vector<int> col, t_col;
  std::vector<double> val, t_val;
};
// SparseMap(n, views, rays, triplets) layout (sparse.cpp:9-45).
SparseHost build_sparse(int n, int views, int rays, std::vector<int64_t> rows,
                        std::vector<int64_t> cols, std::vector<double> vals);
// build_fanbeam (fanbeam.cpp:43-111) and FanBeamGeometry::defaults (:10-17).
SparseHost build_fanbeam(int n, int views, int rays, double source_radius, double fan_angle);
void fan_defaults(int n, double& source_radius, double& fan_angle);

// ------------------------------------------------------- device buffers
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) NCSG_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void zero(cudaStream_t s) {
    if (n) NCSG_CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// --------------------------------------------------------- Radon plan
// Tiling constants of the projector kernels.
constexpr int kFpW = 128;    // forward strip width (pixels)
constexpr int kFpT = 32;     // forward tile-row height
constexpr int kFpWarps = 4;  // forward: warps per CTA = angles per CTA
#ifndef NCSG_BP_WARPS
#define NCSG_BP_WARPS 4
#endif
#ifndef NCSG_BP_WAVES
#define NCSG_BP_WAVES 4
#endif
// Adjoint output tile (W x T): 172 x 20 where 172-wide tiles cover n with
// <= 5% waste (n = 512: 3 tiles), else 128 x 28. Both keep 4 accumulators of
// (T + 5) x (W + 4) floats under 75 KB so 3 CTAs fit per SM; the wider tile
// packs more rays per lane group (sweep in profiles/r1_summary.md).
#ifndef NCSG_BP_WIDE_T
#define NCSG_BP_WIDE_T 20
#endif
#ifndef NCSG_BP_WIDE_P
#define NCSG_BP_WIDE_P 176
#endif
constexpr int kBpWideT = NCSG_BP_WIDE_T, kBpWideP = NCSG_BP_WIDE_P;
inline void bp_tile_shape(int n, int& W, int& T, int& P) {
  if ((n + 171) / 172 * 172 <= n + n / 20) {
    W = 172;
    T = kBpWideT;
    P = kBpWideP;
  } else {
    W = 128;
    T = 28;
    P = 132;
  }
}
constexpr int kBpWarps = NCSG_BP_WARPS;  // adjoint: warps per CTA (private accumulators)
constexpr int kBpWaves = NCSG_BP_WAVES;  // adjoint: target CTAs = 148 * 3 * waves

// Orbit-mode adjoint (bp_gather_kernel): pixel-driven, TW x TH pixel tiles
// of the representative's frame, kGaPx pixels per thread, orbits staged in
// batches of kGaBatch.
#ifndef NCSG_GA_TH
#define NCSG_GA_TH 32
#endif
#ifndef NCSG_GA_BATCH
#define NCSG_GA_BATCH 16
#endif
#ifndef NCSG_GA_WAVES
#define NCSG_GA_WAVES 4
#endif
constexpr int kGaTW = 32, kGaTH = NCSG_GA_TH, kGaThreads = 256;
constexpr int kGaPx = kGaTW * kGaTH / kGaThreads;  // pixels per thread
constexpr int kGaBatch = NCSG_GA_BATCH, kGaWaves = NCSG_GA_WAVES;
#ifndef NCSG_GA_SW_EXTRA
#define NCSG_GA_SW_EXTRA 0  // extra staged cells (experiments with taller tiles: epilogue space)
#endif
constexpr int kGaSW = kGaTW + kGaTH + 8 + NCSG_GA_SW_EXTRA;  // staged rays per orbit and tile
#ifndef NCSG_GA_WT_PF
#define NCSG_GA_WT_PF 2
#endif
constexpr int kGaWtPf = NCSG_GA_WT_PF;  // table mode: orbits prefetched ahead into L2
constexpr int kGaMaxChunk = 1024;                   // orbits per chunk (lowest-ray table)
// Per-orbit constants of the gather (host fp64 from the Q32 lattice): the
// lattice is p(s, k) = c + s a + k d, and pixel (X, Y) has the continuous
// lattice coordinates (sigma, kappa) = M^-1 (q - c), M = [a d], kept in Q32
// fixed point as affine functions of (X, Y).
// One skipped window sample of a border pixel (bp_gather_kernel): ray s of
// the orbit, the members it is invalid for (bit m), its bilinear weight.
struct GaBorderEntry {
  float w;
  short s;
  unsigned char mask;
  unsigned char pad;
};
struct GatherGeom {
  long long s0, sx, sy;  // sigma(X, Y) = s0 + X sx + Y sy   (Q32)
  long long k0, kx, ky;  // kappa(X, Y) = k0 + X kx + Y ky   (Q32)
  float ax, ay, dx, dy;  // lattice vectors (pixels)
  float rho, inv_dy;     // sigma half-extent of the |e| < 1 window, 1 / dy
  int t[4];              // member angles (-1: absent)
  int dir;               // tau = dir * k
  int pad;
};

// SparseMap on the device (sparse_kernels.cu): fp32 values, int32 indices.
struct SparseDev {
  int n = 0, views = 0, rays = 0;
  size_t rows = 0, cols = 0, nnz = 0;
  DevBuf<int64_t> row_ptr, t_row_ptr;
  DevBuf<int> col, t_col;
  DevBuf<float> val, t_val;
  void upload(const SparseHost& h);
};
// y[b] = A x[b] (rows = sinogram bins) / y[b] = A^T u[b] (rows = pixels).
void launch_sparse_forward(const SparseDev& A, const float* x, size_t x_stride, float* y,
                           size_t y_stride, int batch, cudaStream_t s);
void launch_sparse_adjoint(const SparseDev& A, const float* u, size_t u_stride, float* y,
                           size_t y_stride, int batch, cudaStream_t s);

struct RadonDev {
  Geometry geo;
  int device = 0;
  DevBuf<AngleGeom> angles[2];
  DevBuf<RayRange> rays;
  int n_strips = 0;
  int fp_rmax[2] = {0, 0};  // max rays per (strip, angle) per class
  int bp_chunks[2] = {0, 0};
  int bp_chunk_len[2] = {0, 0};
  int bp_batch_planned = 0;
  // Orbit-mode adjoint (bp_gather_kernel): bp_orbit_chunks chunks of
  // bp_orbit_len orbits, four image-frame partials per chunk
  // (bp_chunks[0] = 4 * chunks, bp_chunks[1] = 0).
  bool bp_orbit = false;
  int bp_orbit_chunks = 0, bp_orbit_len = 0;
  int bp_cluster = 1;  // chunk CTAs folded per thread-block cluster (1, 2 or 4)
  DevBuf<GatherGeom> gather;
  // Border-pixel corrections of the gather adjoint (plan_adjoint): for each
  // edge tile e (ga_tile_edge[tile] = e, -1 inside), item (orbit o, border
  // pixel k in row-major order) at ga_bt_base[e] + o * nbp_e + k owns the
  // entries [ga_bt_off[item], ga_bt_off[item + 1]) -- the window samples of
  // that pixel the reference skips (outside the image square or the member
  // rays' replayed ranges), in candidate order
  DevBuf<int> ga_tile_edge, ga_bt_base, ga_bt_off;
  DevBuf<GaBorderEntry> ga_bt_ent;
  // Window-weight table of the gather adjoint: W[orbit][tile][plane][thread]
  // uint4 (three 21-bit fixed-point weights = 8 bytes per (pixel, orbit)); state 0 = not built yet, 1 = in use,
  // -1 = unavailable (disabled, over the size cap or out of memory)
  DevBuf<uint4> ga_wtab;
  int ga_wtab_state = 0;
  // Orbit-interleaved dual (optional gather input): angle t's member slot
  // 4 * orbit + member (-1: none) and the padded row of rays per orbit.
  DevBuf<int> angle_slot;
  DevBuf<int4> orbit_t;  // member angles of each orbit (-1: absent)
  int u4_row() const { return geo.n_det + 2 * kGaSW; }
  size_t u4_size() const { return geo.orbits.size() * static_cast<size_t>(u4_row()) * 4; }
  DevBuf<int2> strip_range[2];                // [angle][strip] s-range (forward)
  std::vector<int2> strip_range_host[2];
  // Orbit-mode forward (fp_orbit_kernel): strips x segments of rows; each
  // ray's partial sums land in the slot of its monotone staircase path.
  bool orbit_mode = false;
  int n_segs = 1;
  int orb_seg = 64;      // rows per forward segment (upload chooses 32 or 64)
  int batch_hint = 1;    // problems per launch the plan is sized for (set before upload)
  int orb_rmax = 0;
  int orb_warps = 8;     // warps per forward CTA
  int orb_split = 1;     // warps per orbit (small grids: 4, each every 4th ray group)
  DevBuf<OrbitGeom> orbits;
  DevBuf<int2> orb_range;                     // [orbit][strip][seg] s-range
  // Cached TMA descriptor of the orbit forward's member-image buffer (encoded
  // once per (buffer, batch), not per launch).
  struct QuadMap {
    alignas(64) unsigned char bytes[128];
    const float* ptr = nullptr;
    int batch = 0;
    bool ok = false;
  };
  mutable QuadMap quad_map;
  void upload();
  void plan_adjoint(int batch);
  void build_gather_border_table();
  void build_gather_weight_table();
  bool gather_table_streams(int batch) const;
  int n_partials() const { return bp_chunks[0] + bp_chunks[1]; }
  // Forward partial slots per ray (fp_partial[batch][slots][m]).
  int fp_slots() const { return orbit_mode ? n_strips + n_segs - 1 : n_strips; }
};
// Orbit-mode forward input: the four dihedral member images interleaved per
// pixel, [batch][n][n][4] floats (4*n*n per problem).
void launch_make_planes(const float* x, float* planes, int n, int batch, cudaStream_t s);

// Projector launches.  img / imgT: batch images (stride n*n), imgT may be
// null when class H is empty.  fp_partial: [batch][n_strips][m] (zeros where
// a strip has no rays; written entries overwritten each call).
// Orbit mode: imgT = the symmetry planes buffer [batch][3][n][n].
void launch_radon_forward_partial(const RadonDev& r, const float* img, const float* imgT,
                                  float* fp_partial, int batch, cudaStream_t s);
// Sums partial strips into out[batch][m] (stand-alone forward).
void launch_strip_sum(const RadonDev& r, const float* fp_partial, float* out, int batch,
                      cudaStream_t s);
// Adjoint partial images: bp_part[batch][n_partials][n*n]; class-H partials
// are stored transposed.
// u4 (nullable, gather mode): the orbit-interleaved copy of u written by the
// dual update (RadonDev::u4_size() floats per problem), staged instead of u.
void launch_radon_adjoint_partial(const RadonDev& r, const float* u, size_t u_stride,
                                  float* bp_part, int batch, cudaStream_t s,
                                  const float* u4 = nullptr);
// out[b] = sum of the class-V partials + transposed class-H partials.
void launch_sum_partials(const float* part, int nV, int nH, float* out, int n, int batch,
                         cudaStream_t s);

// ------------------------------------------------------------------ FFT
// Radix schedule of a length-n Stockham FFT: powers of two use the radix-8
// fast path (logn >= 0); other sizes n = 2^a 3^b 5^c 7^d run mixed-radix
// stages (logn = -1).
struct FftShape {
  int n = 0, logn = -1, nst = 0;
  int rad[24] = {};
};
struct FftPlan {
  int n = 0;
  FftShape shape;
  DevBuf<float2> tw;   // exp(-2 pi i k / n), k < n
  DevBuf<float2> tw2;  // stage twiddles of the power-of-two engine (fft_pow2.cuh), or empty
  void init(int n_, cudaStream_t s);
};
// Spectrum layout: specT[batch][n/2+1][n] complex (column-major half spectrum).
// Peer memory of the fused P2P exchange (<= kMaxPeers ranks of one node):
// rank q's buffer as this rank's kernels store to it.
constexpr int kMaxPeers = 8;
struct PeerPtrs {
  void* p[kMaxPeers] = {};
};
// Row slabs (sharded slab FFT): the row passes cover image rows [r0, r0 +
// rows) and address bin (k, y) at k * ld + (y - r0), batch stride bstride;
// the unsharded layout is {0, n, n, (n/2+1) n}.  With peers set (fused P2P
// all-to-all), the R2C pass stores bin (k, y) straight into rank q = k / wc's
// receive blocks at ((rank * wc + k % wc) * ld + (y - r0)).
struct RowSlab {
  int r0 = 0, rows = 0, ld = 0;
  size_t bstride = 0;
  int wc = 0, rank = 0;
  PeerPtrs peers;
  static RowSlab full(int n) {
    RowSlab r;
    r.rows = n;
    r.ld = n;
    r.bstride = static_cast<size_t>(n / 2 + 1) * n;
    return r;
  }
};
// Column slab of the sharded column pass: after the all-to-all a rank holds
// P blocks [source rank i][wc columns][R rows]; bin (local column c, row j)
// sits at ((j >> logR) * wc + c) * R + (j & (R-1)); its global column is
// k0 + c (filter column).  ncols local columns are transformed.
// With peers set (fused P2P all-to-all back), block i of the result is
// stored straight into rank i's row-slab spectrum at ((rank * wc + c) << logR)
// + (j & (R-1)).
struct ColSlab {
  int logR = 0, wc = 0, k0 = 0, ncols = 0;
  int rank = 0;
  PeerPtrs peers;
};
// Real-to-half-spectrum row pass; `terms` (combine) describes how the real
// input image is assembled (see ncs_kernels.cu).
struct AtuTerms;
void launch_fft_rows_r2c(const FftPlan& f, const AtuTerms& terms, float2* specT, int batch,
                         cudaStream_t s, RowSlab rs = RowSlab{});
// Column pass: forward FFT along j, multiply by maskT[k][j], inverse FFT.
void launch_fft_cols_filter(const FftPlan& f, float2* specT, const float2* maskT, int batch,
                            cudaStream_t s);
// The sharded column pass (batch 1) on a rank's column slab (ColSlab layout).
void launch_fft_cols_filter_slab(const FftPlan& f, float2* slab, const float2* maskT, ColSlab cs,
                                 cudaStream_t s);
// Column pass without the filter: forward FFT only (half spectrum of F x).
void launch_fft_cols_forward(const FftPlan& f, float2* specT, int batch, cudaStream_t s);
// Inverse rows (C2R) fused with the x update: out = x_in - w (or w when
// x_in == nullptr); optional x_old copy, transposed copy, finiteness flag.
// The dual update of the blocks whose forward map needs only x -- identity
// (DENOISE data, QuadraticConj), D (ScaledL1Conj) and positivity (NonnegConj)
// -- fused into the inverse row pass that produces x (Engine::step's dual
// half, solvers.cpp:146-156, for those blocks).  Each CTA then keeps 2G - 1
// rows and also transforms the next row, which the v-block of D needs.
struct DualFuse {
  int on = 0;
  float alpha = 0.f, s_quad = 0.f, wd = 0.f, bound = 0.f;
  float* ud = nullptr;       // identity-block dual (DENOISE data), nullable
  const float* bd = nullptr; // its data term b
  float* ug = nullptr;       // gradient dual (h block then v block), nullable
  float* up = nullptr;       // positivity dual, nullable
  size_t u_stride = 0;       // per-problem stride of the duals
  int* flag = nullptr;       // [2] = min(step counter [1]) over NaN duals
};
struct XUpdate {
  float* x = nullptr;       // updated in place (x -= w) ; if subtract == 0: x = w
  float* x_old = nullptr;   // receives the pre-update x (nullable)
  float* xT = nullptr;      // receives the transposed result (nullable)
  // orbit mode: receives the new x as the four dihedral member planes
  // (make_quad_kernel's layout), power-of-two full-row path only (nullable)
  float4* quad = nullptr;
  int subtract = 1;
  int* flag = nullptr;      // [0] = min(step counter [1]) over non-finite results (nullable)
  // fused P2P all-gather: the updated rows also go to these ranks' images
  // (the own x among them counts once: x itself)
  PeerPtrs x_peers;
  int n_peers = 0;
  DualFuse df;              // power-of-two path, unsharded rows only
};
// Whether launch_fft_rows_c2r can take XUpdate::df = df (the power-of-two
// path, staging within shared memory; NCSG_FUSE_DUAL=0 turns the fusion off).
bool fft_fuses_dual(const FftPlan& f, const DualFuse& df);
// Whether launch_fft_rows_c2r can take XUpdate::quad (the power-of-two path;
// NCSG_FUSE_QUAD=0 keeps the stand-alone make_quad_kernel).
bool fft_writes_quad(const FftPlan& f);
void launch_fft_rows_c2r(const FftPlan& f, const float2* specT, const XUpdate& xu, int batch,
                         cudaStream_t s, RowSlab rs = RowSlab{});

// ------------------------------------------------------------ NCS kernels
// Terms summed into the image fed to the FFT: A^T u for the stacked problem.
struct AtuTerms {
  int n = 0;
  const float* bp_part = nullptr;  // [batch][nV+nH][n*n] (nullable)
  int nV = 0, nH = 0;
  const float* ident = nullptr;    // identity-block dual (DENOISE data / positivity), nullable
  const float* ident2 = nullptr;   // second identity term (positivity with DENOISE), nullable
  const float* ug = nullptr;       // gradient dual [batch][2n(n-1)], nullable
  float wd = 0.f;                  // D-block weight beta/alpha
  const float* plain = nullptr;    // plain image input (mask apply), overrides the rest
  size_t part_stride = 0;          // per-batch stride of bp_part
  size_t img_stride = 0;           // stride between partial images (0: n*n)
  size_t ident_stride = 0, ug_stride = 0;
  int* counter = nullptr;          // flag buffer: counter[1] += 1 once per step (nullable)
};

}  // namespace ncsg
