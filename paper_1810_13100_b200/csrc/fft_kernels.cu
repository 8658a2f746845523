// Circulant solve w = Re(F^-1 (h .* F a)) as a real 2-D FFT on sm_100a.
//
// Replaces MaskApplier::apply + Fft2D (circulant.cpp:27-37, fft.cpp:37-48).
// For real input the reference's c2c transform followed by Re() equals a
// real-to-half-spectrum transform with the Hermitian part of h, so the work is
// three passes over an N x (N/2+1) half spectrum stored column-major
// (specT[k][j], k = 0..N/2), each pass a batch of shared-memory Stockham FFTs
// (radix-8 stages in registers, one radix-2/4 stage when log2 N % 3 != 0):
//   1. rows, real -> half spectrum (two real rows packed per complex FFT);
//      the row loader assembles a = A^T u on the fly (adjoint partial images,
//      transposed class-H partials, D^T u_g, identity blocks): the "combine"
//      of StackedMap::adjoint (linear_map.cpp:47-55) costs no extra pass;
//   2. columns: forward FFT, multiply by the stored filter (pinv mask with the
//      1/N^2 of fft.cpp:46-47 folded in), inverse FFT -- one kernel;
//   3. rows, half spectrum -> real, fused with x <- x - w, the x_old copy,
//      the transposed copy used by the class-H projector, and the
//      check_finite flag (solvers.cpp:145,248-255).
// Twiddles are fp64-derived fp32 constants.  N must be a power of two >= 8.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "fft_pow2.cuh"
#include "ncs_device.cuh"
#include "ncsg_internal.cuh"

namespace ncsg {

namespace {

#ifndef NCSG_FFT_ROWS
#define NCSG_FFT_ROWS 4
#endif
constexpr int kRowsPerBlock = NCSG_FFT_ROWS;  // rows per row-pass CTA (packed pairs)

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// ---- Stockham autosort FFT (natural order in and out) -------------------
// Stage with radix R and span Ns (Ns = product of the previous radices): for
// j < n/R, k = j mod Ns, the R inputs in[j + r n/R] are twiddled by
// w_{Ns R}^{r k}, transformed by an R-point DFT in registers and written to
// out[(j - k) R + k + r Ns].  tw[i] = exp(-2 pi i i / n), i < n (fp64-derived).
template <int SIGN>
__device__ __forceinline__ float2 mul_i(float2 a) {  // * (-i) forward, * (+i) inverse
  return SIGN < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
template <int SIGN>
__device__ __forceinline__ void dft2(float2* v) {
  const float2 t = v[0];
  v[0] = cadd(t, v[1]);
  v[1] = csub(t, v[1]);
}
template <int SIGN>
__device__ __forceinline__ void dft4(float2* v) {
  const float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  const float2 a2 = cadd(v[1], v[3]), a3 = mul_i<SIGN>(csub(v[1], v[3]));
  v[0] = cadd(a0, a2);
  v[2] = csub(a0, a2);
  v[1] = cadd(a1, a3);
  v[3] = csub(a1, a3);
}
template <int SIGN>
__device__ __forceinline__ void dft8(float2* v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  dft4<SIGN>(e);
  dft4<SIGN>(o);
  const float c = 0.70710678118654752440f;
  o[1] = SIGN < 0 ? make_float2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x))
                  : make_float2(c * (o[1].x - o[1].y), c * (o[1].x + o[1].y));
  o[2] = mul_i<SIGN>(o[2]);
  o[3] = SIGN < 0 ? make_float2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y))
                  : make_float2(-c * (o[3].x + o[3].y), c * (o[3].x - o[3].y));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = cadd(e[k], o[k]);
    v[k + 4] = csub(e[k], o[k]);
  }
}
template <int R, int SIGN>
__device__ __forceinline__ void dftR(float2* v) {
  if (R == 2) dft2<SIGN>(v);
  if (R == 4) dft4<SIGN>(v);
  if (R == 8) dft8<SIGN>(v);
}

template <int R, int SIGN>
__device__ void stockham_stage(const float2* in, float2* out, int nfft, int n, int logn, int Ns,
                               int lns, const float2* __restrict__ tw) {
  constexpr int LR = R == 2 ? 1 : R == 4 ? 2 : 3;
  const int lm = logn - LR;  // log2(n / R)
  const int m = 1 << lm;
  const int lstep = logn - lns - LR;  // log2(n / (Ns R))
  for (int bi = threadIdx.x; bi < (nfft << lm); bi += blockDim.x) {
    const int q = bi >> lm, j = bi & (m - 1);
    const float2* src = in + (q << logn);
    float2* dst = out + (q << logn);
    const int k = j & (Ns - 1);
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[j + r * m];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      float2 w = __ldg(tw + ((r * k) << lstep));
      if (SIGN > 0) w.y = -w.y;
      v[r] = cmul(v[r], w);
    }
    dftR<R, SIGN>(v);
    const int idx = ((j - k) << LR) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[idx + r * Ns] = v[r];
  }
}

// nfft contiguous length-n transforms held in `a`; `b` is scratch of the same
// size.  Returns the buffer holding the (natural-order) result.
template <int SIGN>
__device__ float2* fft_stockham(float2* a, float2* b, int nfft, int n, int logn,
                                const float2* __restrict__ tw) {
  int lns = 0;
  const int rem = logn % 3;
  if (rem) {
    __syncthreads();
    if (rem == 1)
      stockham_stage<2, SIGN>(a, b, nfft, n, logn, 1, 0, tw);
    else
      stockham_stage<4, SIGN>(a, b, nfft, n, logn, 1, 0, tw);
    lns = rem;
    float2* t = a;
    a = b;
    b = t;
  }
  for (; lns < logn; lns += 3) {
    __syncthreads();
    stockham_stage<8, SIGN>(a, b, nfft, n, logn, 1 << lns, lns, tw);
    float2* t = a;
    a = b;
    b = t;
  }
  __syncthreads();
  return a;
}

// ---- mixed-radix Stockham (sizes that are not powers of 2: radix 2/3/4/5/7/8
// butterflies in registers, any other prime factor by stockham_stage_prime)
template <int R, int SIGN>
__device__ __forceinline__ void dft_small(float2* v) {
  if constexpr (R == 2 || R == 4 || R == 8) {
    dftR<R, SIGN>(v);
  } else {
  float2 out[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    float re = 0.f, im = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float sn, cs;
      sincospif(2.0f * static_cast<float>((r * k) % R) / R, &sn, &cs);
      sn *= static_cast<float>(SIGN);
      re += v[r].x * cs - v[r].y * sn;
      im += v[r].x * sn + v[r].y * cs;
    }
    out[k] = make_float2(re, im);
  }
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = out[k];
  }
}

template <int R, int SIGN>
__device__ void stockham_stage_mixed(const float2* in, float2* out, int nfft, int n, int Ns,
                                     const float2* __restrict__ tw) {
  const int m = n / R;
  const int step = n / (Ns * R);
  for (int bi = threadIdx.x; bi < nfft * m; bi += blockDim.x) {
    const int q = bi / m, j = bi - q * m;
    const float2* src = in + q * n;
    float2* dst = out + q * n;
    const int k = j % Ns;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[j + r * m];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      float2 w = __ldg(tw + r * k * step);
      if (SIGN > 0) w.y = -w.y;
      v[r] = cmul(v[r], w);
    }
    dft_small<R, SIGN>(v);
    const int idx = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[idx + r * Ns] = v[r];
  }
}

// Any other prime radix R (11, 13, ... up to n itself): one OUTPUT element per
// thread, out[(j - k) R + k + ro Ns] = sum_r in[j + r n/R] w_n^{r e}, with
// e = k n/(Ns R) + ro n/R (the stage twiddle w_{Ns R}^{r k} and the R-point
// DFT factor w_R^{r ro} are both powers of w_n, so one table entry per term).
// O(n R) per sequence: the reference's FFTW takes any N (fft.cpp:18-29), so
// does this path; sizes with large prime factors are slow, not rejected.
template <int SIGN>
__device__ void stockham_stage_prime(const float2* in, float2* out, int nfft, int n, int Ns, int R,
                                     const float2* __restrict__ tw) {
  const int m = n / R;
  const int step = n / (Ns * R);
  for (int oi = threadIdx.x; oi < nfft * n; oi += blockDim.x) {
    const int q = oi / n, o = oi - q * n;
    // o = (j - k) R + k + ro Ns with k < Ns, ro < R
    const int blk = o / (Ns * R), rem = o - blk * (Ns * R);
    const int ro = rem / Ns, k = rem - ro * Ns;
    const int j = blk * Ns + k;
    const float2* src = in + q * n + j;
    const int e = k * step + ro * m;  // < n
    float re = 0.f, im = 0.f;
    int idx = 0;
    for (int r = 0; r < R; ++r) {
      float2 w = __ldg(tw + idx);
      if (SIGN > 0) w.y = -w.y;
      const float2 v = src[r * m];
      re += v.x * w.x - v.y * w.y;
      im += v.x * w.y + v.y * w.x;
      idx += e;
      if (idx >= n) idx -= n;
    }
    out[oi] = make_float2(re, im);
  }
}

template <int SIGN>
__device__ float2* fft_mixed(float2* a, float2* b, int nfft, const FftShape& sh,
                             const float2* __restrict__ tw) {
  int Ns = 1;
  for (int st = 0; st < sh.nst; ++st) {
    __syncthreads();
    const int R = sh.rad[st];
    switch (R) {
      case 2: stockham_stage_mixed<2, SIGN>(a, b, nfft, sh.n, Ns, tw); break;
      case 3: stockham_stage_mixed<3, SIGN>(a, b, nfft, sh.n, Ns, tw); break;
      case 4: stockham_stage_mixed<4, SIGN>(a, b, nfft, sh.n, Ns, tw); break;
      case 5: stockham_stage_mixed<5, SIGN>(a, b, nfft, sh.n, Ns, tw); break;
      case 7: stockham_stage_mixed<7, SIGN>(a, b, nfft, sh.n, Ns, tw); break;
      case 8: stockham_stage_mixed<8, SIGN>(a, b, nfft, sh.n, Ns, tw); break;
      default: stockham_stage_prime<SIGN>(a, b, nfft, sh.n, Ns, R, tw); break;
    }
    Ns *= R;
    float2* t = a;
    a = b;
    b = t;
  }
  __syncthreads();
  return a;
}

template <int SIGN>
__device__ __forceinline__ float2* fft_run(float2* a, float2* b, int nfft, const FftShape& sh,
                                           const float2* __restrict__ tw) {
  return sh.logn >= 0 ? fft_stockham<SIGN>(a, b, nfft, sh.n, sh.logn, tw)
                      : fft_mixed<SIGN>(a, b, nfft, sh, tw);
}

// Row block bx of problem b (the kernel's blockIdx.x / .y; the fused solve
// calls it per work item).
// PEERS: the fused P2P all-to-all store (a separate instance, so the plain
// passes keep their register budget: the peer table indexed at run time
// lives in local memory).
template <bool PEERS>
__device__ __forceinline__ void rows_r2c_body(const AtuTerms& T, float2* __restrict__ specT,
                                              const float2* __restrict__ tw, const FftShape& sh,
                                              const RowSlab& rs, int bx, int b) {
  extern __shared__ float2 zs[];
  const int n = T.n;
  const int y0 = rs.r0 + bx * kRowsPerBlock;
  const int yend = rs.r0 + rs.rows;  // rows [r0, r0 + rows) of the image
  const int npair = kRowsPerBlock / 2;
  float2* zb = zs + npair * n;  // Stockham scratch
  if (T.counter && bx == 0 && b == 0 && threadIdx.x == 0) atomicAdd(T.counter + 1, 1);
  // Phase 1: row-major terms, coalesced along x (4 pixels per thread when
  // the rows are float4-aligned).
  if ((n & 3) == 0) {
    for (int i = threadIdx.x; i < kRowsPerBlock * n / 4; i += blockDim.x) {
      const int r = (4 * i) / n, x = 4 * i - r * n;
      const int y = y0 + r;
      const float4 v = y < yend ? atu_rowmajor4(T, b, y, x) : make_float4(0.f, 0.f, 0.f, 0.f);
      float2* slot = zs + (r >> 1) * n + x;
      if (r & 1) {
        slot[0].y = v.x, slot[1].y = v.y, slot[2].y = v.z, slot[3].y = v.w;
      } else {
        slot[0].x = v.x, slot[1].x = v.y, slot[2].x = v.z, slot[3].x = v.w;
      }
    }
  } else {
    for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
      const int r = i / n, x = i - r * n;
      const int y = y0 + r;
      const float v = y < yend ? atu_rowmajor(T, b, y, x) : 0.f;
      float2* slot = zs + (r >> 1) * n + x;
      if (r & 1)
        slot->y = v;
      else
        slot->x = v;
    }
  }
  // Phase 2: transposed (class-H) partials, coalesced along y.
  if (!T.plain && T.bp_part && T.nH > 0) {
    __syncthreads();
    const size_t nn = static_cast<size_t>(n) * n;
    const float* base = T.bp_part + b * T.part_stride + T.nV * nn;
    for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
      const int x = i / kRowsPerBlock, r = i - x * kRowsPerBlock;
      const int y = y0 + r;
      if (y >= yend) continue;
      float v = 0.f;
      const float* p = base + static_cast<size_t>(x) * n + y;
      for (int c = 0; c < T.nH; ++c) v += p[c * nn];
      float2* slot = zs + (r >> 1) * n + x;
      if (r & 1)
        slot->y += v;
      else
        slot->x += v;
    }
  }
  const float2* z = fft_run<-1>(zs, zb, npair, sh, tw);
  // Unpack the two real rows of each pair: A = (Z_k + conj Z_-k)/2,
  // B = (Z_k - conj Z_-k)/(2i); write specT[k][y] (k = 0..n/2).
  const int nk = n / 2 + 1;
  float2* out = specT + static_cast<size_t>(b) * rs.bstride;
  // one thread per (row pair, k): both rows' bins leave as one float4 (even n)
  for (int i = threadIdx.x; i < nk * (kRowsPerBlock / 2); i += blockDim.x) {
    const int k = i / (kRowsPerBlock / 2), q = i - k * (kRowsPerBlock / 2);
    const int y = y0 + 2 * q;
    if (y >= yend) continue;
    const float2* zq = z + q * n;
    const float2 zk = zq[k];
    const float2 zm = zq[(n - k) % n];
    const float2 va = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
    const float2 vb = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    float2* dst;
    if (PEERS) {  // fused all-to-all: straight into rank k / wc's blocks
      const int q = k / rs.wc;
      dst = static_cast<float2*>(rs.peers.p[q]) +
            static_cast<size_t>(rs.rank * rs.wc + (k - q * rs.wc)) * rs.ld + (y - rs.r0);
    } else {
      dst = out + static_cast<size_t>(k) * rs.ld + (y - rs.r0);
    }
    if (y + 1 < yend && ((n | rs.ld | rs.r0) & 1) == 0) {
      *reinterpret_cast<float4*>(dst) = make_float4(va.x, va.y, vb.x, vb.y);
    } else {
      dst[0] = va;
      if (y + 1 < yend) dst[1] = vb;
    }
  }
}

template <bool PEERS>
__global__ void fft_rows_r2c_kernel(AtuTerms T, float2* __restrict__ specT,
                                    const float2* __restrict__ tw, FftShape sh, RowSlab rs) {
  pdl_wait();
  rows_r2c_body<PEERS>(T, specT, tw, sh, rs, blockIdx.x, blockIdx.y);
}

#ifndef NCSG_FFT_COLS
#define NCSG_FFT_COLS 2
#endif
constexpr int kColsPerBlock = NCSG_FFT_COLS;  // columns per column-pass CTA

__device__ __forceinline__ void cols_filter_body(float2* __restrict__ specT,
                                                 const float2* __restrict__ maskT,
                                                 const float2* __restrict__ tw, const FftShape& sh,
                                                 int bx, int b) {
  const int n = sh.n;
  extern __shared__ float2 zs[];
  const int k0 = bx * kColsPerBlock;
  const int nk = n / 2 + 1;
  const int nc = min(kColsPerBlock, nk - k0);
  float2* col = specT + (static_cast<size_t>(b) * nk + k0) * n;  // nc contiguous columns
  const float2* mk = maskT + static_cast<size_t>(k0) * n;
  float2* zb = zs + kColsPerBlock * n;
  // the filter goes to the scratch half now, so its load overlaps the
  // column load instead of stalling between the two transforms
  if ((n & 1) == 0) {  // two bins per 16-byte access
    const float4* c4 = reinterpret_cast<const float4*>(col);
    const float4* m4 = reinterpret_cast<const float4*>(mk);
    for (int j = threadIdx.x; j < nc * n / 2; j += blockDim.x) {
      reinterpret_cast<float4*>(zs)[j] = c4[j];
      reinterpret_cast<float4*>(zb)[j] = __ldg(m4 + j);
    }
  } else {
    for (int j = threadIdx.x; j < nc * n; j += blockDim.x) {
      zs[j] = col[j];
      zb[j] = __ldg(mk + j);
    }
  }
  __syncthreads();
  // the forward transform reuses zb as scratch: each thread keeps its
  // filter values in registers meanwhile (<= 8 per thread for every size the
  // launch configures; larger sizes read the filter again)
  constexpr int kMaxPer = 8;
  float2 fr[kMaxPer];
  const bool in_regs = nc * n <= kMaxPer * static_cast<int>(blockDim.x);
#pragma unroll
  for (int t = 0; t < kMaxPer; ++t) {
    const int j = threadIdx.x + t * blockDim.x;
    if (in_regs && j < nc * n) fr[t] = zb[j];
  }
  float2* z = fft_run<-1>(zs, zb, nc, sh, tw);
  if (in_regs) {
#pragma unroll
    for (int t = 0; t < kMaxPer; ++t) {
      const int j = threadIdx.x + t * blockDim.x;
      if (j < nc * n) z[j] = cmul(z[j], fr[t]);
    }
  } else {
    for (int j = threadIdx.x; j < nc * n; j += blockDim.x) z[j] = cmul(z[j], __ldg(mk + j));
  }
  z = fft_run<+1>(z, z == zs ? zb : zs, nc, sh, tw);
  if ((n & 1) == 0) {
    for (int j = threadIdx.x; j < nc * n / 2; j += blockDim.x)
      reinterpret_cast<float4*>(col)[j] = reinterpret_cast<const float4*>(z)[j];
  } else {
    for (int j = threadIdx.x; j < nc * n; j += blockDim.x) col[j] = z[j];
  }
}

__global__ void fft_cols_filter_kernel(float2* __restrict__ specT, const float2* __restrict__ maskT,
                                       const float2* __restrict__ tw, FftShape sh) {
  pdl_wait();
  cols_filter_body(specT, maskT, tw, sh, blockIdx.x, blockIdx.y);
}

// Sharded column pass: the same transform on a rank's column slab after the
// all-to-all (ColSlab addressing: P row blocks of R bins per column).
template <bool PEERS>
__global__ void fft_cols_filter_slab_kernel(float2* __restrict__ slab,
                                            const float2* __restrict__ maskT,
                                            const float2* __restrict__ tw, FftShape sh,
                                            ColSlab cs) {
  pdl_wait();
  const int n = sh.n;
  extern __shared__ float2 zs[];
  const int c0 = blockIdx.x * kColsPerBlock;
  const int nc = min(kColsPerBlock, cs.ncols - c0);
  const int R = 1 << cs.logR;
  float2* zb = zs + kColsPerBlock * n;
  auto at = [&](int c, int j) -> size_t {
    return (static_cast<size_t>((j >> cs.logR) * cs.wc + c0 + c) << cs.logR) + (j & (R - 1));
  };
  for (int i = threadIdx.x; i < nc * n; i += blockDim.x) {
    const int c = i / n, j = i - c * n;
    zs[i] = slab[at(c, j)];
  }
  float2* z = fft_run<-1>(zs, zb, nc, sh, tw);
  for (int i = threadIdx.x; i < nc * n; i += blockDim.x) {
    const int c = i / n, j = i - c * n;
    z[i] = cmul(z[i], __ldg(maskT + static_cast<size_t>(cs.k0 + c0 + c) * n + j));
  }
  z = fft_run<+1>(z, z == zs ? zb : zs, nc, sh, tw);
  for (int i = threadIdx.x; i < nc * n; i += blockDim.x) {
    const int c = i / n, j = i - c * n;
    if (PEERS)  // fused all-to-all back: block j >> logR to its rank
      static_cast<float2*>(cs.peers.p[j >> cs.logR])
          [(static_cast<size_t>(cs.rank * cs.wc + c0 + c) << cs.logR) + (j & (R - 1))] = z[i];
    else
      slab[at(c, j)] = z[i];
  }
}

// Forward column FFTs only (in place): with the row pass this is the
// unnormalised forward 2-D FFT of a real image as a half spectrum
// (empirical_mask's F v, circulant.cpp:111-117).
__global__ void fft_cols_forward_kernel(float2* __restrict__ specT,
                                        const float2* __restrict__ tw, FftShape sh) {
  const int n = sh.n;
  extern __shared__ float2 zs[];
  const int k0 = blockIdx.x * kColsPerBlock;
  const int b = blockIdx.y;
  const int nk = n / 2 + 1;
  const int nc = min(kColsPerBlock, nk - k0);
  float2* col = specT + (static_cast<size_t>(b) * nk + k0) * n;
  float2* zb = zs + kColsPerBlock * n;
  for (int j = threadIdx.x; j < nc * n; j += blockDim.x) zs[j] = col[j];
  const float2* z = fft_run<-1>(zs, zb, nc, sh, tw);
  for (int j = threadIdx.x; j < nc * n; j += blockDim.x) col[j] = z[j];
}

template <bool PEERS>
__device__ __forceinline__ void rows_c2r_body(const float2* __restrict__ specT, const XUpdate& xu,
                                              const float2* __restrict__ tw, const FftShape& sh,
                                              const RowSlab& rs, int bx, int b) {
  const int n = sh.n;
  extern __shared__ float2 zs[];
  const int y0 = rs.r0 + bx * kRowsPerBlock;
  const int yend = rs.r0 + rs.rows;
  const int nk = n / 2 + 1;
  const size_t nn = static_cast<size_t>(n) * n;
  const float2* in = specT + static_cast<size_t>(b) * rs.bstride;
  float2* zb = zs + (kRowsPerBlock / 2) * n;  // Stockham scratch
  // x (to be updated) streams into shared memory with cp.async now, so its
  // latency overlaps the spectrum load and the transform
  float* xs = reinterpret_cast<float*>(zs + kRowsPerBlock * n);
  const bool x_pre = xu.subtract && (n & 3) == 0;
  if (x_pre) {
    for (int i = threadIdx.x; i < kRowsPerBlock * n / 4; i += blockDim.x) {
      const int r = (4 * i) / n, x = 4 * i - r * n;
      if (y0 + r >= yend) continue;
      const float* src = xu.x + b * nn + static_cast<size_t>(y0 + r) * n + x;
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(xs + 4 * i));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // Build Z = G_a + i G_b with Hermitian extension (G_r[n-k] = conj G_r[k]):
  // one thread per (row pair, k) reads both rows' bins as one float4 and
  // writes Z[k] and Z[n-k] (no other thread touches them).
  for (int i = threadIdx.x; i < nk * (kRowsPerBlock / 2); i += blockDim.x) {
    const int k = i / (kRowsPerBlock / 2), q = i - k * (kRowsPerBlock / 2);
    const int y = y0 + 2 * q;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);  // (G_a, G_b) of rows y, y + 1
    const float2* src = in + static_cast<size_t>(k) * rs.ld + (y - rs.r0);
    if (y + 1 < yend && ((n | rs.ld | rs.r0) & 1) == 0) {  // 16-byte aligned pair
      g = *reinterpret_cast<const float4*>(src);
    } else if (y < yend) {
      const float2 ga = src[0];
      g.x = ga.x, g.y = ga.y;
      if (y + 1 < yend) {
        const float2 gb = src[1];
        g.z = gb.x, g.w = gb.y;
      }
    }
    float2* zq = zs + q * n;
    zq[k] = make_float2(g.x - g.w, g.y + g.z);
    if (k > 0 && 2 * k != n) zq[n - k] = make_float2(g.x + g.w, g.z - g.y);
  }
  float2* z = fft_run<+1>(zs, zb, kRowsPerBlock / 2, sh, tw);
  // x update, row-major.
  int bad = 0;
  if (x_pre) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  // four pixels per thread (x_pre implies n % 4 == 0): float4 in and out
  for (int i4 = threadIdx.x; i4 < kRowsPerBlock * n / 4 && x_pre; i4 += blockDim.x) {
    const int i = 4 * i4;
    const int r = i / n, x = i - r * n;
    const int y = y0 + r;
    if (y >= yend) continue;
    float2* zr = z + (r >> 1) * n + x;
    const float4 xo = *reinterpret_cast<const float4*>(xs + i);
    const size_t gi = b * nn + static_cast<size_t>(y) * n + x;
    float4 xn;
    if (r & 1)
      xn = make_float4(xo.x - zr[0].y, xo.y - zr[1].y, xo.z - zr[2].y, xo.w - zr[3].y);
    else
      xn = make_float4(xo.x - zr[0].x, xo.y - zr[1].x, xo.z - zr[2].x, xo.w - zr[3].x);
    if (xu.x_old) *reinterpret_cast<float4*>(xu.x_old + gi) = xo;
    *reinterpret_cast<float4*>(xu.x + gi) = xn;
    for (int q = 0; PEERS && q < xu.n_peers; ++q)  // fused all-gather of the own rows
      *reinterpret_cast<float4*>(static_cast<float*>(xu.x_peers.p[q]) + gi) = xn;
    bad |= !isfinite(xn.x) || !isfinite(xn.y) || !isfinite(xn.z) || !isfinite(xn.w);
    if (xu.xT) {
      if (r & 1) {
        zr[0].y = xn.x, zr[1].y = xn.y, zr[2].y = xn.z, zr[3].y = xn.w;
      } else {
        zr[0].x = xn.x, zr[1].x = xn.y, zr[2].x = xn.z, zr[3].x = xn.w;
      }
    }
  }
  for (int i = threadIdx.x; i < kRowsPerBlock * n && !x_pre; i += blockDim.x) {
    const int r = i / n, x = i - r * n;
    const int y = y0 + r;
    if (y >= yend) continue;
    const float2 zz = z[(r >> 1) * n + x];
    const float w = (r & 1) ? zz.y : zz.x;
    const size_t gi = b * nn + static_cast<size_t>(y) * n + x;
    float xn;
    if (xu.subtract) {
      const float xo = xu.x[gi];
      if (xu.x_old) xu.x_old[gi] = xo;
      xn = xo - w;
    } else {
      xn = w;
    }
    xu.x[gi] = xn;
    for (int q = 0; PEERS && q < xu.n_peers; ++q) static_cast<float*>(xu.x_peers.p[q])[gi] = xn;
    bad |= !isfinite(xn);
    if (xu.xT) {
      if (r & 1)
        z[(r >> 1) * n + x].y = xn;
      else
        z[(r >> 1) * n + x].x = xn;
    }
  }
  if (xu.flag && __syncthreads_or(bad) && threadIdx.x == 0)
    atomicMin(xu.flag, *(volatile int*)(xu.flag + 1));
  if (xu.xT) {
    __syncthreads();
    for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
      const int x = i / kRowsPerBlock, r = i - x * kRowsPerBlock;
      const int y = y0 + r;
      if (y >= yend) continue;
      const float2 zz = z[(r >> 1) * n + x];
      xu.xT[b * nn + static_cast<size_t>(x) * n + y] = (r & 1) ? zz.y : zz.x;
    }
  }
}

template <bool PEERS>
__global__ void fft_rows_c2r_kernel(const float2* __restrict__ specT, XUpdate xu,
                                    const float2* __restrict__ tw, FftShape sh, RowSlab rs) {
  pdl_wait();
  rows_c2r_body<PEERS>(specT, xu, tw, sh, rs, blockIdx.x, blockIdx.y);
}

// ---- power-of-two fast path: the register-resident engine (fft_pow2.cuh) --
// Same passes and fusions as above; each row pass CTA holds G row pairs (one
// transform group of N/16 threads each, extra threads only load), the column
// pass G columns.

__device__ __forceinline__ void mbar_init1(unsigned bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait0(unsigned bar) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar)
      : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void cp_async8(float2* dst, const float2* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

template <int LOGN, bool PEERS>
__global__ void __launch_bounds__(512) fft_rows_r2c_p2(AtuTerms T, float2* __restrict__ specT,
                                                       const float2* __restrict__ twt, RowSlab rs,
                                                       int G) {
  pdl_wait();
  using Ge = p2::Geo<LOGN>;
  constexpr int N = Ge::N, NP = Ge::NP, TT = Ge::T;
  extern __shared__ float2 zs[];
  const int b = blockIdx.y;
  const int rows = 2 * G;
  const int y0 = rs.r0 + blockIdx.x * rows;
  const int yend = rs.r0 + rs.rows;
  if (T.counter && blockIdx.x == 0 && b == 0 && threadIdx.x == 0) atomicAdd(T.counter + 1, 1);
  // row-major terms, four pixels per thread (N % 4 == 0), into pair r/2's
  // buffer (real part: even row, imaginary part: odd row)
  for (int i = threadIdx.x; i < rows * N / 4; i += blockDim.x) {
    const int r = (4 * i) >> LOGN, x = 4 * i - (r << LOGN);
    const int y = y0 + r;
    const float4 v = y < yend ? atu_rowmajor4(T, b, y, x) : make_float4(0.f, 0.f, 0.f, 0.f);
    float2* slot = zs + (r >> 1) * NP + p2::pad(x);
    if (r & 1) {
      slot[0].y = v.x, slot[1].y = v.y, slot[2].y = v.z, slot[3].y = v.w;
    } else {
      slot[0].x = v.x, slot[1].x = v.y, slot[2].x = v.z, slot[3].x = v.w;
    }
  }
  // transposed (class-H) partials, coalesced along y
  if (!T.plain && T.bp_part && T.nH > 0) {
    __syncthreads();
    const size_t nn = static_cast<size_t>(N) * N;
    const float* base = T.bp_part + b * T.part_stride + T.nV * nn;
    for (int i = threadIdx.x; i < rows * N; i += blockDim.x) {
      const int x = i / rows, r = i - x * rows;
      const int y = y0 + r;
      if (y >= yend) continue;
      float v = 0.f;
      const float* p = base + static_cast<size_t>(x) * N + y;
      for (int c = 0; c < T.nH; ++c) v += p[c * nn];
      float2* slot = zs + (r >> 1) * NP + p2::pad(x);
      if (r & 1)
        slot->y += v;
      else
        slot->x += v;
    }
  }
  __syncthreads();
  const int g = threadIdx.x / TT, t = threadIdx.x % TT;
  const bool active = g < G;
  float2* buf = zs + (active ? g : 0) * NP;
  float2 v[Ge::E];
  if (active) {
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) v[e] = buf[p2::pad(t + TT * e)];
  }
  p2::fft<LOGN, -1>(v, buf, t, twt, active);
  __syncthreads();
  if (active) {
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) buf[p2::pad(t + TT * e)] = v[e];
  }
  __syncthreads();
  // unpack the two real rows of each pair: A = (Z_k + conj Z_-k)/2,
  // B = (Z_k - conj Z_-k)/(2i); both rows' bin k leave as one float4
  const int nk = N / 2 + 1;
  float2* out = specT + static_cast<size_t>(b) * rs.bstride;
  for (int i = threadIdx.x; i < nk * G; i += blockDim.x) {
    const int k = i / G, q = i - k * G;
    const int y = y0 + 2 * q;
    if (y >= yend) continue;
    const float2* zq = zs + q * NP;
    const float2 zk = zq[p2::pad(k)];
    const float2 zm = zq[p2::pad((N - k) & (N - 1))];
    const float2 va = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
    const float2 vb = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    float2* dst;
    if (PEERS) {  // fused all-to-all: straight into rank k / wc's blocks
      const int qq = k / rs.wc;
      dst = static_cast<float2*>(rs.peers.p[qq]) +
            static_cast<size_t>(rs.rank * rs.wc + (k - qq * rs.wc)) * rs.ld + (y - rs.r0);
    } else {
      dst = out + static_cast<size_t>(k) * rs.ld + (y - rs.r0);
    }
    if (y + 1 < yend && ((rs.ld | rs.r0) & 1) == 0) {
      *reinterpret_cast<float4*>(dst) = make_float4(va.x, va.y, vb.x, vb.y);
    } else {
      dst[0] = va;
      if (y + 1 < yend) dst[1] = vb;
    }
  }
}

template <int LOGN>
__global__ void __launch_bounds__(512) fft_cols_filter_p2(float2* __restrict__ specT,
                                                          const float2* __restrict__ maskT,
                                                          const float2* __restrict__ twt, int G) {
  pdl_wait();
  using Ge = p2::Geo<LOGN>;
  constexpr int N = Ge::N, NP = Ge::NP, TT = Ge::T;
  extern __shared__ float2 zs[];
  const int b = blockIdx.y;
  const int nk = N / 2 + 1;
  const int g = threadIdx.x / TT, t = threadIdx.x % TT;
  const int k = blockIdx.x * G + g;
  const bool active = g < G && k < nk;
  float2* buf = zs + (g < G ? g : 0) * NP;
  float2* fm = zs + G * NP + (g < G ? g : 0) * N;  // this group's filter column
  float2* col = specT + (static_cast<size_t>(b) * nk + (active ? k : 0)) * N;
  float2 v[Ge::E];
  if (active) {
    // the filter streams into shared memory while the column transforms;
    // each thread later reads only the entries it copied (no barrier)
    const float2* mk = maskT + static_cast<size_t>(k) * N;
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) cp_async8(fm + t + TT * e, mk + t + TT * e);
    asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) v[e] = col[t + TT * e];
  }
  p2::fft<LOGN, -1>(v, buf, t, twt, active);
  if (active) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) v[e] = p2::cmul(v[e], fm[t + TT * e]);
  }
  p2::fft<LOGN, +1>(v, buf, t, twt, active);
  if (active) {
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) col[t + TT * e] = v[e];
  }
}

template <int LOGN, bool PEERS>
__global__ void __launch_bounds__(512) fft_rows_c2r_p2(const float2* __restrict__ specT, XUpdate xu,
                                                       const float2* __restrict__ twt, RowSlab rs,
                                                       int G) {
  pdl_wait();
  using Ge = p2::Geo<LOGN>;
  constexpr int N = Ge::N, NP = Ge::NP, TT = Ge::T;
  extern __shared__ float2 zs[];
  const DualFuse& df = xu.df;
  const int b = blockIdx.y;
  const int rows = 2 * G;                      // rows transformed
  const int keep = df.on ? rows - 1 : rows;    // rows owned (x written)
  const int y0 = rs.r0 + blockIdx.x * keep;
  const int yend = rs.r0 + rs.rows;
  const int yown = min(yend, y0 + keep);       // owned rows [y0, yown)
  const int ylim = df.on ? min(N, y0 + rows) : yend;  // transformed rows [y0, ylim)
  const int nk = N / 2 + 1;
  const size_t nn = static_cast<size_t>(N) * N;
  const float2* in = specT + static_cast<size_t>(b) * rs.bstride;
  float* xs = reinterpret_cast<float*>(zs + G * NP);  // rows x N: x before the update
  const bool pre = xu.subtract != 0;
  if (pre) {  // x streams in while the spectrum loads and transforms
    for (int i = threadIdx.x; i < rows * N / 4; i += blockDim.x) {
      const int r = (4 * i) >> LOGN, x = 4 * i - (r << LOGN);
      if (y0 + r >= ylim) continue;
      const float* src = xu.x + b * nn + static_cast<size_t>(y0 + r) * N + x;
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(xs + 4 * i));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // fused dual: the owned rows of every x-only dual block (and the data
  // term) stream into shared memory by bulk copies while the row transforms
  // run -- each block's owned rows are one contiguous range, 16-byte aligned
  // (N % 4 == 0) except the h block's, whose range is widened to alignment
  __shared__ __align__(8) unsigned long long dbar;
  const unsigned dbar_a = static_cast<unsigned>(__cvta_generic_to_shared(&dbar));
  float* dsm = xs + rows * N;  // [ud | bd | up] keep x N each, then h, then v
  const int nown = max(0, yown - y0);
  const int nv = max(0, min(nown, N - 1 - y0));
  const size_t h0 = static_cast<size_t>(y0) * (N - 1), h0a = h0 & ~static_cast<size_t>(3);
  float* s_ud = dsm;
  float* s_bd = s_ud + (df.ud ? keep * N : 0);
  float* s_up = s_bd + (df.ud ? keep * N : 0);
  float* s_h = s_up + (df.up ? keep * N : 0);
  float* s_v = s_h + (df.ug ? keep * N + 4 : 0);
  if (df.on && threadIdx.x == 0) {
    mbar_init1(dbar_a);
    unsigned bytes = 0;
    const size_t rowoff = static_cast<size_t>(y0) * N;
    if (df.ud && nown) bytes += 2u * nown * N * 4;
    if (df.up && nown) bytes += nown * N * 4;
    size_t hb = 0;
    if (df.ug && nown) {
      const size_t h1 = static_cast<size_t>(y0 + nown) * (N - 1);
      hb = ((h1 + 3) & ~static_cast<size_t>(3)) - h0a;
      bytes += static_cast<unsigned>(hb * 4) + nv * N * 4;
    }
    mbar_arrive_tx(dbar_a, bytes);
    if (df.ud && nown) {
      bulk_g2s(s_ud, df.ud + b * df.u_stride + rowoff, nown * N * 4, dbar_a);
      bulk_g2s(s_bd, df.bd + b * nn + rowoff, nown * N * 4, dbar_a);
    }
    if (df.up && nown) bulk_g2s(s_up, df.up + b * df.u_stride + rowoff, nown * N * 4, dbar_a);
    if (df.ug && nown) {
      const float* ug = df.ug + b * df.u_stride;
      bulk_g2s(s_h, ug + h0a, static_cast<unsigned>(hb * 4), dbar_a);
      if (nv) bulk_g2s(s_v, ug + static_cast<size_t>(N) * (N - 1) + rowoff, nv * N * 4, dbar_a);
    }
  }
  // Z = G_a + i G_b with the Hermitian extension (G_r[N-k] = conj G_r[k]):
  // one thread per (row pair, k) reads both rows' bins as one float4
  for (int i = threadIdx.x; i < nk * G; i += blockDim.x) {
    const int k = i / G, q = i - k * G;
    const int y = y0 + 2 * q;
    float4 gg = make_float4(0.f, 0.f, 0.f, 0.f);
    const float2* src = in + static_cast<size_t>(k) * rs.ld + (y - rs.r0);
    if (y + 1 < ylim && (((y - rs.r0) | rs.ld) & 1) == 0) {  // 16-byte aligned pair
      gg = *reinterpret_cast<const float4*>(src);
    } else if (y < ylim) {
      const float2 ga = src[0];
      gg.x = ga.x, gg.y = ga.y;
      if (y + 1 < ylim) {
        const float2 gb = src[1];
        gg.z = gb.x, gg.w = gb.y;
      }
    }
    float2* zq = zs + q * NP;
    zq[p2::pad(k)] = make_float2(gg.x - gg.w, gg.y + gg.z);
    if (k > 0 && 2 * k != N) zq[p2::pad(N - k)] = make_float2(gg.x + gg.w, gg.z - gg.y);
  }
  __syncthreads();
  const int g = threadIdx.x / TT, t = threadIdx.x % TT;
  const bool active = g < G;
  float2* buf = zs + (active ? g : 0) * NP;
  float2 v[Ge::E];
  if (active) {
#pragma unroll
    for (int e = 0; e < Ge::E; ++e) v[e] = buf[p2::pad(t + TT * e)];
  }
  p2::fft<LOGN, +1>(v, buf, t, twt, active);
  if (pre) asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  int bad = 0;
  if (active) {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int r = 2 * g + rr;
      const int y = y0 + r;
      if (y >= ylim) continue;
      const bool own = y < yown;
      float* xrow = xu.x + b * nn + static_cast<size_t>(y) * N;
      float* orow = xu.x_old ? xu.x_old + b * nn + static_cast<size_t>(y) * N : nullptr;
#pragma unroll
      for (int e = 0; e < Ge::E; ++e) {
        const int x = t + TT * e;
        const float w = rr ? v[e].y : v[e].x;
        float xn;
        if (pre) {
          const float xo = xs[r * N + x];
          if (orow && own) orow[x] = xo;
          xn = xo - w;
        } else {
          xn = w;
        }
        if (own) {
          xrow[x] = xn;
          for (int qq = 0; PEERS && qq < xu.n_peers; ++qq)
            static_cast<float*>(xu.x_peers.p[qq])[b * nn + static_cast<size_t>(y) * N + x] = xn;
          bad |= !isfinite(xn);
        }
        if (rr)
          v[e].y = xn;
        else
          v[e].x = xn;
      }
    }
  }
  if (xu.flag && __syncthreads_or(bad) && threadIdx.x == 0)
    atomicMin(xu.flag, *(volatile int*)(xu.flag + 1));
  if (xu.xT || xu.quad || df.on) {  // the new rows in natural order: zs[pair][pad(x)]
    __syncthreads();
    if (active) {
#pragma unroll
      for (int e = 0; e < Ge::E; ++e) buf[p2::pad(t + TT * e)] = v[e];
    }
    __syncthreads();
  }
  if (xu.xT) {
    for (int i = threadIdx.x; i < keep * N; i += blockDim.x) {
      const int x = i / keep, r = i - x * keep;
      const int y = y0 + r;
      if (y >= yown) continue;
      const float2 zz = zs[(r >> 1) * NP + p2::pad(x)];
      xu.xT[b * nn + static_cast<size_t>(x) * N + y] = (r & 1) ? zz.y : zz.x;
    }
  }
  if (xu.quad) {
    // orbit mode: the new rows go straight into the member planes the
    // forward reads (make_quad_kernel's layout, no separate pass):
    //   quad[r][c] = (x[r][c], x[N-1-c][r], x[r][N-1-c], x[N-1-c][N-1-r]),
    // so x[y][x] is member 0 of quad[y][x], 2 of quad[y][N-1-x] (along quad
    // rows), 1 of quad[x][N-1-y] and 3 of quad[N-1-x][N-1-y] (along quad
    // columns: the CTA's rows are consecutive cells there)
    float* qf = reinterpret_cast<float*>(xu.quad + b * nn);
    for (int i = threadIdx.x; i < keep * N; i += blockDim.x) {
      const int r = i >> LOGN, x = i & (N - 1);
      const int y = y0 + r;
      if (y >= yown) continue;
      const float2 zz = zs[(r >> 1) * NP + p2::pad(x)];
      const float v = (r & 1) ? zz.y : zz.x;
      qf[4 * (static_cast<size_t>(y) * N + x)] = v;
      qf[4 * (static_cast<size_t>(y) * N + (N - 1 - x)) + 2] = v;
    }
    for (int i = threadIdx.x; i < keep * N; i += blockDim.x) {
      const int x = i / keep, r = i - x * keep;
      const int y = y0 + r;
      if (y >= yown) continue;
      const float2 zz = zs[(r >> 1) * NP + p2::pad(x)];
      const float v = (r & 1) ? zz.y : zz.x;
      qf[4 * (static_cast<size_t>(x) * N + (N - 1 - y)) + 1] = v;
      qf[4 * (static_cast<size_t>(N - 1 - x) * N + (N - 1 - y)) + 3] = v;
    }
  }
  if (df.on) {
    // dual update of the owned rows (dual_update_kernel's identity, D and
    // positivity sections, same arithmetic): x_new from zs, x_old from xs,
    // the duals and data from the bulk-copied rows
    mbar_wait0(dbar_a);
    auto xn_at = [&](int r, int x) -> float {
      const float2 zz = zs[(r >> 1) * NP + p2::pad(x)];
      return (r & 1) ? zz.y : zz.x;
    };
    const float alpha = df.alpha;
    int badu = 0;
    if (df.ud) {
      float* ud = df.ud + b * df.u_stride + static_cast<size_t>(y0) * N;
      for (int i = threadIdx.x; i < nown * N; i += blockDim.x) {
        const int r = i >> LOGN, x = i & (N - 1);
        const float un = (s_ud[i] + alpha * (2.f * xn_at(r, x) - xs[i] - s_bd[i])) * df.s_quad;
        ud[i] = un;
        badu |= isnan(un);
      }
    }
    if (df.ug) {
      float* ug = df.ug + b * df.u_stride;
      const float wd = df.wd, bd = df.bound;
      const int hoff = static_cast<int>(h0 - h0a);
      // h block: rows of N - 1 edges
      for (int i = threadIdx.x; i < nown * (N - 1); i += blockDim.x) {
        const int r = i / (N - 1), x = i - r * (N - 1);
        const float an = wd * (xn_at(r, x) - xn_at(r, x + 1));
        const float ao = wd * (xs[r * N + x] - xs[r * N + x + 1]);
        const float z = s_h[hoff + i] + alpha * (2.f * an - ao - 0.f);
        ug[h0 + i] = z < -bd ? -bd : (z > bd ? bd : z);
        badu |= isnan(z);
      }
      // v block: rows y < N - 1 (row y + 1 is transformed here too)
      float* vb = ug + static_cast<size_t>(N) * (N - 1) + static_cast<size_t>(y0) * N;
      for (int i = threadIdx.x; i < nv * N; i += blockDim.x) {
        const int r = i >> LOGN, x = i & (N - 1);
        const float an = wd * (xn_at(r, x) - xn_at(r + 1, x));
        const float ao = wd * (xs[i] - xs[i + N]);
        const float z = s_v[i] + alpha * (2.f * an - ao - 0.f);
        vb[i] = z < -bd ? -bd : (z > bd ? bd : z);
        badu |= isnan(z);
      }
    }
    if (df.up) {
      float* up = df.up + b * df.u_stride + static_cast<size_t>(y0) * N;
      for (int i = threadIdx.x; i < nown * N; i += blockDim.x) {
        const int r = i >> LOGN, x = i & (N - 1);
        const float z = s_up[i] + alpha * (2.f * xn_at(r, x) - xs[i]);
        up[i] = z < 0.f ? z : 0.f;
        badu |= isnan(z);
      }
    }
    // dual NaN (check_finite's second test, solvers.cpp:252-254): flag word 2
    if (df.flag && __syncthreads_or(badu) && threadIdx.x == 0)
      atomicMin(df.flag + 2, *(volatile int*)(df.flag + 1));
  }
}

int log2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

bool p2_enabled(int logn) {
  static const bool off = std::getenv("NCSG_FFT_P2") && std::atoi(std::getenv("NCSG_FFT_P2")) == 0;
  return !off && logn >= p2::kMinLog && logn <= p2::kMaxLog;
}
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
// Row pairs per row-pass CTA / columns per column-pass CTA.
int p2_row_groups() {
  static const int g = std::max(1, std::min(8, env_int("NCSG_FFT_RG", 2)));
  return g;
}
// Shared memory of the dual-fused inverse row pass with G row pairs and
// `arrays` bulk-copied dual / data rows.
size_t p2_fuse_smem(int n, int G, int arrays) {
  return sizeof(float2) * G * p2::pad(n) + sizeof(float) * 2 * G * n +
         sizeof(float) * arrays * (2 * G - 1) * n + 16;
}
constexpr size_t kFuseSmemCap = 200 * 1024;
// Row pairs per CTA of the dual-fused inverse row pass (2G - 1 rows kept):
// the largest of 4, 3, 2 whose staging fits (0: none does).
int p2_fuse_groups(int n, int arrays) {
  static const int g = env_int("NCSG_FFT_FG", 0);
  int G = g > 0 ? std::max(2, std::min(8, g)) : (n >= 512 ? 4 : 2);
  while (G >= 2 && p2_fuse_smem(n, G, arrays) > kFuseSmemCap) --G;
  return G >= 2 ? G : 0;
}
int fuse_arrays(const DualFuse& df) {
  return (df.ud ? 2 : 0) + (df.up ? 1 : 0) + (df.ug ? 2 : 0);
}
int p2_col_groups(int T) {
  static const int cg = env_int("NCSG_FFT_CG", 0);
  if (cg > 0) return std::max(1, std::min(16, cg));
  return std::max(1, 128 / T);
}

#define NCSG_P2_SWITCH(LOGN_EXPR, MACRO) \
  switch (LOGN_EXPR) {                   \
    case 6: MACRO(6); break;             \
    case 7: MACRO(7); break;             \
    case 8: MACRO(8); break;             \
    case 9: MACRO(9); break;             \
    case 10: MACRO(10); break;           \
    case 11: MACRO(11); break;           \
    case 12: MACRO(12); break;           \
    default: break;                      \
  }

int fft_threads(int work) { return std::max(64, std::min(512, work)); }

}  // namespace

void FftPlan::init(int n_, cudaStream_t s) {
  if (n_ < 2) throw Error{NCSG_INVALID, "GPU circulant solve needs an image size >= 2"};
  n = n_;
  shape = FftShape{};
  shape.n = n;
  if (n >= 8 && (n & (n - 1)) == 0) {
    shape.logn = log2i(n);  // radix-8 fast path
  } else {
    // radix 8 / 4 / 2 for the power of two, then 3, 5, 7, then any other prime
    int r = n;
    auto push = [&](int f) {
      if (shape.nst >= 24) throw Error{NCSG_INVALID, "FFT size has too many factors"};
      shape.rad[shape.nst++] = f;
    };
    while (r % 8 == 0) push(8), r /= 8;
    while (r % 4 == 0) push(4), r /= 4;
    while (r % 2 == 0) push(2), r /= 2;
    for (int f : {3, 5, 7})
      while (r % f == 0) push(f), r /= f;
    // remaining prime factors (11, 13, ...): the generic one-output-per-thread stage
    for (int f = 11; r > 1; f += 2) {
      if (static_cast<long long>(f) * f > r) f = r;
      while (r % f == 0) push(f), r /= f;
    }
  }
  std::vector<float2> h(n);
  for (int k = 0; k < n; ++k) {
    double ang = -2.0 * 3.14159265358979323846 * k / n;
    h[k] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
  }
  tw.alloc(h.size());
  NCSG_CUDA_CHECK(cudaMemcpyAsync(tw.p, h.data(), h.size() * sizeof(float2),
                                  cudaMemcpyHostToDevice, s));
  // stage twiddles of the register-resident engine: stage s (span Ns = 16^s,
  // radix R) at tw_off(s) + (r - 1) Ns + k = exp(-2 pi i r k / (Ns R))
  std::vector<float2> h2;
  if (shape.logn >= 0 && p2_enabled(shape.logn)) {
    const int logn = shape.logn;
    const int le = p2::kLE, E = 1 << le;
    const int nst = (logn + le - 1) / le, llr = logn - le * (nst - 1);
    h2.assign(p2::tw_len(logn), make_float2(0.f, 0.f));
    long long ns = E;
    for (int st = 1; st < nst; ++st, ns *= E) {
      const int R = st == nst - 1 ? (1 << llr) : E;
      for (int r = 1; r < R; ++r)
        for (long long k = 0; k < ns; ++k) {
          const double ang = -2.0 * 3.14159265358979323846 * static_cast<double>(r * k) /
                             static_cast<double>(ns * R);
          h2[p2::tw_off(st) + (r - 1) * ns + k] =
              make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
        }
    }
    tw2.alloc(h2.size());
    NCSG_CUDA_CHECK(cudaMemcpyAsync(tw2.p, h2.data(), h2.size() * sizeof(float2),
                                    cudaMemcpyHostToDevice, s));
  } else {
    tw2.release();
  }
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
}

void launch_fft_rows_r2c(const FftPlan& f, const AtuTerms& terms, float2* specT, int batch,
                         cudaStream_t s, RowSlab rs) {
  const int n = f.n;
  if (rs.rows == 0) rs = RowSlab::full(n);
  const bool peers = rs.peers.p[0] != nullptr;
  if (f.tw2.p) {
    const int G = p2_row_groups(), T = n >> p2::kLE;
    const size_t sm = sizeof(float2) * G * p2::pad(n);
    const int threads = std::max(G * T, std::min(512, G * n / 2));
    dim3 grid((rs.rows + 2 * G - 1) / (2 * G), batch);
#define NCSG_R2C(L)                                                                        \
  {                                                                                        \
    auto kern = peers ? fft_rows_r2c_p2<L, true> : fft_rows_r2c_p2<L, false>;              \
    ensure_smem(reinterpret_cast<const void*>(kern), sm);                                  \
    launch_pdl(kern, grid, dim3(threads), sm, s, terms, specT, f.tw2.p, rs, G);            \
  }
    NCSG_P2_SWITCH(f.shape.logn, NCSG_R2C)
#undef NCSG_R2C
    NCSG_CUDA_CHECK(cudaGetLastError());
    count_launch();
    return;
  }
  size_t smem = 2 * sizeof(float2) * (kRowsPerBlock / 2) * n;
  auto kern = peers ? fft_rows_r2c_kernel<true> : fft_rows_r2c_kernel<false>;
  ensure_smem(reinterpret_cast<const void*>(kern), smem);
  dim3 grid((rs.rows + kRowsPerBlock - 1) / kRowsPerBlock, batch);
  // the loader (sums of adjoint partial images) wants more threads than the FFT
  launch_pdl(kern, grid, dim3(fft_threads(kRowsPerBlock * n / 4)), smem, s, terms,
             specT, f.tw.p, f.shape, rs);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_fft_cols_filter(const FftPlan& f, float2* specT, const float2* maskT, int batch,
                            cudaStream_t s) {
  const int n = f.n;
  if (f.tw2.p) {
    const int T = n >> p2::kLE, G = p2_col_groups(T);
    const size_t sm = sizeof(float2) * G * (p2::pad(n) + n);
    dim3 grid((n / 2 + 1 + G - 1) / G, batch);
#define NCSG_COLS(L)                                                                   \
  {                                                                                    \
    ensure_smem(reinterpret_cast<const void*>(fft_cols_filter_p2<L>), sm);             \
    launch_pdl(fft_cols_filter_p2<L>, grid, dim3(G * T), sm, s, specT, maskT, f.tw2.p, G); \
  }
    NCSG_P2_SWITCH(f.shape.logn, NCSG_COLS)
#undef NCSG_COLS
    NCSG_CUDA_CHECK(cudaGetLastError());
    count_launch();
    return;
  }
  size_t smem = 2 * sizeof(float2) * kColsPerBlock * n;
  ensure_smem(reinterpret_cast<const void*>(fft_cols_filter_kernel), smem);
  dim3 grid((n / 2 + 1 + kColsPerBlock - 1) / kColsPerBlock, batch);
  launch_pdl(fft_cols_filter_kernel, grid, dim3(fft_threads(kColsPerBlock * n / 8)), smem, s,
             specT, maskT, f.tw.p, f.shape);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_fft_cols_forward(const FftPlan& f, float2* specT, int batch, cudaStream_t s) {
  const int n = f.n;
  size_t smem = 2 * sizeof(float2) * kColsPerBlock * n;
  ensure_smem(reinterpret_cast<const void*>(fft_cols_forward_kernel), smem);
  dim3 grid((n / 2 + 1 + kColsPerBlock - 1) / kColsPerBlock, batch);
  fft_cols_forward_kernel<<<grid, fft_threads(kColsPerBlock * n / 8), smem, s>>>(specT, f.tw.p,
                                                                               f.shape);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_fft_cols_filter_slab(const FftPlan& f, float2* slab, const float2* maskT, ColSlab cs,
                                 cudaStream_t s) {
  const int n = f.n;
  if (cs.ncols <= 0) return;
  size_t smem = 2 * sizeof(float2) * kColsPerBlock * n;
  auto kern = cs.peers.p[0] ? fft_cols_filter_slab_kernel<true> : fft_cols_filter_slab_kernel<false>;
  ensure_smem(reinterpret_cast<const void*>(kern), smem);
  dim3 grid((cs.ncols + kColsPerBlock - 1) / kColsPerBlock, 1);
  launch_pdl(kern, grid, dim3(fft_threads(kColsPerBlock * n / 8)), smem, s,
             slab, maskT, f.tw.p, f.shape, cs);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

bool fft_writes_quad(const FftPlan& f) {
  static const bool off = std::getenv("NCSG_FUSE_QUAD") && std::atoi(std::getenv("NCSG_FUSE_QUAD")) == 0;
  return !off && f.tw2.p != nullptr;
}

bool fft_fuses_dual(const FftPlan& f, const DualFuse& df) {
  static const bool off = std::getenv("NCSG_FUSE_DUAL") && std::atoi(std::getenv("NCSG_FUSE_DUAL")) == 0;
  return !off && f.tw2.p != nullptr && p2_fuse_groups(f.n, fuse_arrays(df)) > 0;
}

void launch_fft_rows_c2r(const FftPlan& f, const float2* specT, const XUpdate& xu, int batch,
                         cudaStream_t s, RowSlab rs) {
  const int n = f.n;
  if (rs.rows == 0) rs = RowSlab::full(n);
  if (f.tw2.p) {
    const int G = xu.df.on ? p2_fuse_groups(n, fuse_arrays(xu.df)) : p2_row_groups(), T = n >> p2::kLE;
    if (G == 0) throw Error{NCSG_INVALID, "fused dual update does not fit in shared memory"};
    const size_t sm = xu.df.on ? p2_fuse_smem(n, G, fuse_arrays(xu.df))
                               : sizeof(float2) * G * p2::pad(n) + sizeof(float) * 2 * G * n;
    // the fused dual's loops and bulk-copied rows want more threads than the
    // transform (C2: 256 -> 512 threads, 20.4 -> 18.3 us)
    static const int c2r_threads = env_int("NCSG_FFT_C2R_THREADS", 0);
    const int threads = std::max(G * T, c2r_threads > 0 ? c2r_threads : (xu.df.on ? 512 : 128));
    const int keep = xu.df.on ? 2 * G - 1 : 2 * G;
    dim3 grid((rs.rows + keep - 1) / keep, batch);
    const bool peers = xu.n_peers > 0;
#define NCSG_C2R(L)                                                                 \
  {                                                                                 \
    auto kern = peers ? fft_rows_c2r_p2<L, true> : fft_rows_c2r_p2<L, false>;       \
    ensure_smem(reinterpret_cast<const void*>(kern), sm);                           \
    launch_pdl(kern, grid, dim3(threads), sm, s, specT, xu, f.tw2.p, rs, G);        \
  }
    NCSG_P2_SWITCH(f.shape.logn, NCSG_C2R)
#undef NCSG_C2R
    NCSG_CUDA_CHECK(cudaGetLastError());
    count_launch();
    return;
  }
  size_t smem = 2 * sizeof(float2) * (kRowsPerBlock / 2) * n + sizeof(float) * kRowsPerBlock * n;
  auto kern = xu.n_peers > 0 ? fft_rows_c2r_kernel<true> : fft_rows_c2r_kernel<false>;
  ensure_smem(reinterpret_cast<const void*>(kern), smem);
  dim3 grid((rs.rows + kRowsPerBlock - 1) / kRowsPerBlock, batch);
  launch_pdl(kern, grid, dim3(fft_threads((kRowsPerBlock / 2) * n / 4)), smem, s,
             specT, xu, f.tw.p, f.shape, rs);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

}  // namespace ncsg
