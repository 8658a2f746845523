// Circulant solve w = Re(F^-1 (h .* F a)) as a real 2-D FFT on sm_100a.
//
// Replaces MaskApplier::apply + Fft2D (circulant.cpp:27-37, fft.cpp:37-48).
// For real input the reference's c2c transform followed by Re() equals a
// real-to-half-spectrum transform with the Hermitian part of h, so the work is
// three passes over an N x (N/2+1) half spectrum stored column-major
// (specT[k][j], k = 0..N/2), each pass a batch of shared-memory radix-2 FFTs:
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
#include <vector>

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

__device__ __forceinline__ unsigned bitrev(unsigned v, int logn) { return __brev(v) >> (32 - logn); }

// In-place radix-2 DIT over `nfft` contiguous length-n sequences (bit-reversed
// input, natural output).  sign: -1 forward, +1 inverse (unnormalised).
__device__ void fft_dit(float2* z, int nfft, int n, int logn, const float2* __restrict__ tw,
                        int sign) {
  const int half = n >> 1;
  const int total = nfft * half;
  for (int lh = 0; lh < logn; ++lh) {
    const int h = 1 << lh;
    const int tstride = half >> lh;  // n / (2h)
    __syncthreads();
    for (int bi = threadIdx.x; bi < total; bi += blockDim.x) {
      const int q = bi / half;
      const int t = bi - q * half;
      const int j = t & (h - 1);
      const int i0 = ((t >> lh) << (lh + 1)) + j;
      float2 w = __ldg(tw + j * tstride);
      if (sign > 0) w.y = -w.y;
      float2* zq = z + q * n;
      const float2 u = zq[i0];
      const float2 v = cmul(zq[i0 + h], w);
      zq[i0] = cadd(u, v);
      zq[i0 + h] = csub(u, v);
    }
  }
  __syncthreads();
}

// In-place radix-2 DIF (natural input, bit-reversed output).
__device__ void fft_dif(float2* z, int nfft, int n, int logn, const float2* __restrict__ tw,
                        int sign) {
  const int half = n >> 1;
  const int total = nfft * half;
  for (int lh = logn - 1; lh >= 0; --lh) {
    const int h = 1 << lh;
    const int tstride = half >> lh;
    __syncthreads();
    for (int bi = threadIdx.x; bi < total; bi += blockDim.x) {
      const int q = bi / half;
      const int t = bi - q * half;
      const int j = t & (h - 1);
      const int i0 = ((t >> lh) << (lh + 1)) + j;
      float2 w = __ldg(tw + j * tstride);
      if (sign > 0) w.y = -w.y;
      float2* zq = z + q * n;
      const float2 u = zq[i0];
      const float2 v = zq[i0 + h];
      zq[i0] = cadd(u, v);
      zq[i0 + h] = cmul(csub(u, v), w);
    }
  }
  __syncthreads();
}

__global__ void fft_rows_r2c_kernel(AtuTerms T, float2* __restrict__ specT,
                                    const float2* __restrict__ tw, int logn) {
  extern __shared__ float2 zs[];
  const int n = T.n;
  const int y0 = blockIdx.x * kRowsPerBlock;
  const int b = blockIdx.y;
  const int npair = kRowsPerBlock / 2;
  if (T.counter && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    atomicAdd(T.counter + 1, 1);
  // Phase 1: row-major terms, coalesced along x.
  for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
    const int r = i / n, x = i - r * n;
    const int y = y0 + r;
    const float v = y < n ? atu_rowmajor(T, b, y, x) : 0.f;
    float2* slot = zs + (r >> 1) * n + bitrev(x, logn);
    if (r & 1)
      slot->y = v;
    else
      slot->x = v;
  }
  // Phase 2: transposed (class-H) partials, coalesced along y.
  if (!T.plain && T.bp_part && T.nH > 0) {
    __syncthreads();
    const size_t nn = static_cast<size_t>(n) * n;
    const float* base = T.bp_part + b * T.part_stride + T.nV * nn;
    for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
      const int x = i / kRowsPerBlock, r = i - x * kRowsPerBlock;
      const int y = y0 + r;
      if (y >= n) continue;
      float v = 0.f;
      const float* p = base + static_cast<size_t>(x) * n + y;
      for (int c = 0; c < T.nH; ++c) v += p[c * nn];
      float2* slot = zs + (r >> 1) * n + bitrev(x, logn);
      if (r & 1)
        slot->y += v;
      else
        slot->x += v;
    }
  }
  fft_dit(zs, npair, n, logn, tw, -1);
  // Unpack the two real rows of each pair: A = (Z_k + conj Z_-k)/2,
  // B = (Z_k - conj Z_-k)/(2i); write specT[k][y] (k = 0..n/2).
  const int nk = n / 2 + 1;
  float2* out = specT + static_cast<size_t>(b) * nk * n;
  for (int i = threadIdx.x; i < nk * kRowsPerBlock; i += blockDim.x) {
    const int k = i / kRowsPerBlock, r = i - k * kRowsPerBlock;
    const int y = y0 + r;
    if (y >= n) continue;
    const float2* zq = zs + (r >> 1) * n;
    const float2 zk = zq[k];
    const float2 zm = zq[(n - k) & (n - 1)];
    float2 v;
    if (r & 1)
      v = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    else
      v = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
    out[static_cast<size_t>(k) * n + y] = v;
  }
}

__global__ void fft_cols_filter_kernel(float2* __restrict__ specT, const float2* __restrict__ maskT,
                                       const float2* __restrict__ tw, int n, int logn) {
  extern __shared__ float2 zs[];
  const int k = blockIdx.x;
  const int b = blockIdx.y;
  const int nk = n / 2 + 1;
  float2* col = specT + (static_cast<size_t>(b) * nk + k) * n;
  const float2* mk = maskT + static_cast<size_t>(k) * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) zs[bitrev(j, logn)] = col[j];
  fft_dit(zs, 1, n, logn, tw, -1);
  for (int j = threadIdx.x; j < n; j += blockDim.x) zs[j] = cmul(zs[j], __ldg(mk + j));
  fft_dif(zs, 1, n, logn, tw, +1);
  for (int j = threadIdx.x; j < n; j += blockDim.x) col[j] = zs[bitrev(j, logn)];
}

__global__ void fft_rows_c2r_kernel(const float2* __restrict__ specT, XUpdate xu,
                                    const float2* __restrict__ tw, int n, int logn) {
  extern __shared__ float2 zs[];
  const int y0 = blockIdx.x * kRowsPerBlock;
  const int b = blockIdx.y;
  const int nk = n / 2 + 1;
  const size_t nn = static_cast<size_t>(n) * n;
  const float2* in = specT + static_cast<size_t>(b) * nk * n;
  // Build Z = G_a + i G_b with Hermitian extension (G_r[n-k] = conj G_r[k]).
  for (int i = threadIdx.x; i < nk * kRowsPerBlock; i += blockDim.x) {
    const int k = i / kRowsPerBlock, r = i - k * kRowsPerBlock;
    const int y = y0 + r;
    const float2 g = y < n ? in[static_cast<size_t>(k) * n + y] : make_float2(0.f, 0.f);
    float2* zq = zs + (r >> 1) * n;
    const unsigned ik = bitrev(k, logn);
    const unsigned im = bitrev((n - k) & (n - 1), logn);
    if ((r & 1) == 0) {
      // a part: Z[k] += G_a[k], Z[n-k] += conj(G_a[k])
      zq[ik].x = g.x;
      zq[ik].y = g.y;
      if (k > 0 && k < n / 2) {
        zq[im].x = g.x;
        zq[im].y = -g.y;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nk * kRowsPerBlock; i += blockDim.x) {
    const int k = i / kRowsPerBlock, r = i - k * kRowsPerBlock;
    const int y = y0 + r;
    if ((r & 1) == 0) continue;
    const float2 g = y < n ? in[static_cast<size_t>(k) * n + y] : make_float2(0.f, 0.f);
    float2* zq = zs + (r >> 1) * n;
    const unsigned ik = bitrev(k, logn);
    const unsigned im = bitrev((n - k) & (n - 1), logn);
    // b part: Z[k] += i G_b[k], Z[n-k] += i conj(G_b[k])
    zq[ik].x -= g.y;
    zq[ik].y += g.x;
    if (k > 0 && k < n / 2) {
      zq[im].x += g.y;
      zq[im].y += g.x;
    }
  }
  fft_dit(zs, kRowsPerBlock / 2, n, logn, tw, +1);
  // x update, row-major.
  int bad = 0;
  for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
    const int r = i / n, x = i - r * n;
    const int y = y0 + r;
    if (y >= n) continue;
    const float2 z = zs[(r >> 1) * n + x];
    const float w = (r & 1) ? z.y : z.x;
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
    bad |= !isfinite(xn);
    if (xu.xT) {
      if (r & 1)
        zs[(r >> 1) * n + x].y = xn;
      else
        zs[(r >> 1) * n + x].x = xn;
    }
  }
  if (xu.flag && __syncthreads_or(bad) && threadIdx.x == 0)
    atomicMin(xu.flag, *(volatile int*)(xu.flag + 1));
  if (xu.xT) {
    __syncthreads();
    for (int i = threadIdx.x; i < kRowsPerBlock * n; i += blockDim.x) {
      const int x = i / kRowsPerBlock, r = i - x * kRowsPerBlock;
      const int y = y0 + r;
      if (y >= n) continue;
      const float2 z = zs[(r >> 1) * n + x];
      xu.xT[b * nn + static_cast<size_t>(x) * n + y] = (r & 1) ? z.y : z.x;
    }
  }
}

int log2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

int fft_threads(int work) { return std::max(32, std::min(512, work)); }

}  // namespace

void FftPlan::init(int n_, cudaStream_t s) {
  if (n_ < 8 || (n_ & (n_ - 1)))
    throw Error{NCSG_INVALID, "GPU circulant solve needs a power-of-two image size >= 8"};
  n = n_;
  std::vector<float2> h(n / 2);
  for (int k = 0; k < n / 2; ++k) {
    double ang = -2.0 * 3.14159265358979323846 * k / n;
    h[k] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
  }
  tw.alloc(h.size());
  NCSG_CUDA_CHECK(cudaMemcpyAsync(tw.p, h.data(), h.size() * sizeof(float2),
                                  cudaMemcpyHostToDevice, s));
  NCSG_CUDA_CHECK(cudaStreamSynchronize(s));
}

void launch_fft_rows_r2c(const FftPlan& f, const AtuTerms& terms, float2* specT, int batch,
                         cudaStream_t s) {
  const int n = f.n;
  size_t smem = sizeof(float2) * (kRowsPerBlock / 2) * n;
  NCSG_CUDA_CHECK(cudaFuncSetAttribute(fft_rows_r2c_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  dim3 grid((n + kRowsPerBlock - 1) / kRowsPerBlock, batch);
  fft_rows_r2c_kernel<<<grid, fft_threads((kRowsPerBlock / 2) * n / 2), smem, s>>>(
      terms, specT, f.tw.p, log2i(n));
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_fft_cols_filter(const FftPlan& f, float2* specT, const float2* maskT, int batch,
                            cudaStream_t s) {
  const int n = f.n;
  size_t smem = sizeof(float2) * n;
  dim3 grid(n / 2 + 1, batch);
  fft_cols_filter_kernel<<<grid, fft_threads(n / 2), smem, s>>>(specT, maskT, f.tw.p, n,
                                                                log2i(n));
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_fft_rows_c2r(const FftPlan& f, const float2* specT, const XUpdate& xu, int batch,
                         cudaStream_t s) {
  const int n = f.n;
  size_t smem = sizeof(float2) * (kRowsPerBlock / 2) * n;
  NCSG_CUDA_CHECK(cudaFuncSetAttribute(fft_rows_c2r_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  dim3 grid((n + kRowsPerBlock - 1) / kRowsPerBlock, batch);
  fft_rows_c2r_kernel<<<grid, fft_threads((kRowsPerBlock / 2) * n / 2), smem, s>>>(
      specT, xu, f.tw.p, n, log2i(n));
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

}  // namespace ncsg
