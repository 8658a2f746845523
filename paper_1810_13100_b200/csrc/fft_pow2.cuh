// Register-resident Stockham FFT for power-of-two lengths 64 <= N <= 4096
// (the circulant solve's fast path, circulant.cpp:27-37 / fft.cpp:37-48).
//
// A group of T = N/E threads (E = 16, or 8 with NCSG_FFT_LE=3) transforms one
// length-N sequence.  Thread t of the group holds the E values of indices
// t + T*e (the cyclic distribution) in registers, both on entry and on exit,
// so global loads and stores of a row or column are coalesced across the
// group.  The transform is NST = ceil(log2 N / log2 E) Stockham stages: radix
// E (16 as a 4 x 4 split in registers) except a smaller last stage when
// log2 N is not a multiple of log2 E.  Stage 0
// runs on the registers as loaded; between stages the group exchanges through
// a shared-memory buffer padded by one slot per 16 (pad(p) = p + p/16), which
// makes the stride-16 writes of the early stages conflict-free per half-warp.
// Twiddles of stage s (span Ns = 16^s, radix R) come from a table laid out
// [r-1][k] (k = j mod Ns contiguous), so consecutive threads load consecutive
// entries.  Barriers are CTA-wide: every thread of the CTA calls the engine
// (threads outside a group pass active = false and only take the barriers).
#pragma once

#include <cuda_runtime.h>

namespace ncsg {
namespace p2 {

constexpr int kMinLog = 6, kMaxLog = 12;

__host__ __device__ constexpr int pad(int p) { return p + (p >> 4); }

// Values per thread E = 2^LE (16 by default; 8 doubles the threads per
// transform for more latency hiding at the price of one more stage).
#ifndef NCSG_FFT_LE
#define NCSG_FFT_LE 4
#endif
constexpr int kLE = NCSG_FFT_LE;

template <int LOGN>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int LE = kLE;
  static constexpr int E = 1 << LE;                      // values per thread
  static constexpr int T = N / E;                        // threads per transform
  static constexpr int NST = (LOGN + LE - 1) / LE;       // stages
  static constexpr int LLR = LOGN - LE * (NST - 1);      // log2 of the last stage's radix
  static constexpr int NP = pad(N);                      // padded buffer length (float2)
};

// Offset of stage s's twiddles (s >= 1) in the table: every stage before the
// last is radix E with (E - 1) * Ns entries.
__host__ __device__ constexpr int tw_off(int s) {
  int off = 0, ns = 1 << kLE;
  for (int i = 1; i < s; ++i) off += ((1 << kLE) - 1) * ns, ns <<= kLE;
  return off;
}
// Table length for log2 N = logn.
__host__ __device__ constexpr int tw_len(int logn) {
  const int nst = (logn + kLE - 1) / kLE;
  const int llr = logn - kLE * (nst - 1);
  int ns = 1;
  for (int i = 1; i < nst; ++i) ns <<= kLE;
  return tw_off(nst - 1) + ((1 << llr) - 1) * ns;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
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
// w_8^1 and w_8^3 times a (forward sign -1, inverse +1)
template <int SIGN>
__device__ __forceinline__ float2 mul_w8_1(float2 a) {
  const float c = 0.70710678118654752440f;
  return SIGN < 0 ? make_float2(c * (a.x + a.y), c * (a.y - a.x))
                  : make_float2(c * (a.x - a.y), c * (a.x + a.y));
}
template <int SIGN>
__device__ __forceinline__ float2 mul_w8_3(float2 a) {
  const float c = 0.70710678118654752440f;
  return SIGN < 0 ? make_float2(c * (a.y - a.x), -c * (a.x + a.y))
                  : make_float2(-c * (a.x + a.y), c * (a.x - a.y));
}
template <int SIGN>
__device__ __forceinline__ void dft8(float2* v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  dft4<SIGN>(e);
  dft4<SIGN>(o);
  o[1] = mul_w8_1<SIGN>(o[1]);
  o[2] = mul_i<SIGN>(o[2]);
  o[3] = mul_w8_3<SIGN>(o[3]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = cadd(e[k], o[k]);
    v[k + 4] = csub(e[k], o[k]);
  }
}
// exp(SIGN * 2 pi i m / 16) for m = 1, 3 (the others are w_8 / +-i multiples)
template <int SIGN>
__device__ __forceinline__ float2 mul_w16(float2 a, int m) {
  const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
  // m = 1: (c1, SIGN s1); m = 3: (s1, SIGN c1)
  const float cr = m == 1 ? c1 : s1, ci = static_cast<float>(SIGN) * (m == 1 ? s1 : c1);
  return make_float2(a.x * cr - a.y * ci, a.x * ci + a.y * cr);
}
// 16-point DFT in natural order: n = 4 n1 + n2, k = k1 + 4 k2.
template <int SIGN>
__device__ __forceinline__ void dft16(float2* v) {
  float2 a[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) a[n2][n1] = v[4 * n1 + n2];
    dft4<SIGN>(a[n2]);
  }
  // twiddles w_16^(n2 k1)
  a[1][1] = mul_w16<SIGN>(a[1][1], 1);
  a[1][2] = mul_w8_1<SIGN>(a[1][2]);
  a[1][3] = mul_w16<SIGN>(a[1][3], 3);
  a[2][1] = mul_w8_1<SIGN>(a[2][1]);
  a[2][2] = mul_i<SIGN>(a[2][2]);
  a[2][3] = mul_w8_3<SIGN>(a[2][3]);
  a[3][1] = mul_w16<SIGN>(a[3][1], 3);
  a[3][2] = mul_w8_3<SIGN>(a[3][2]);
  // w_16^9 = -w_16^1
  {
    const float2 t = mul_w16<SIGN>(a[3][3], 1);
    a[3][3] = make_float2(-t.x, -t.y);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 b[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
    dft4<SIGN>(b);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = b[k2];
  }
}
template <int R, int SIGN>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 2) dft2<SIGN>(v);
  if constexpr (R == 4) dft4<SIGN>(v);
  if constexpr (R == 8) dft8<SIGN>(v);
  if constexpr (R == 16) dft16<SIGN>(v);
}

// Stage S >= 1: read the group's buffer (cyclic), twiddle, DFT; the outputs
// of item q at r land in v[q + Q r] (Q = 16 / R items per thread).
template <int LOGN, int S, int SIGN>
__device__ __forceinline__ void stage_in(float2 (&v)[1 << kLE], const float2* buf, int t,
                                         const float2* __restrict__ twt) {
  using G = Geo<LOGN>;
  constexpr int R = (S == G::NST - 1) ? (1 << G::LLR) : G::E;
  constexpr int Q = G::E / R;
  constexpr int Ns = 1 << (kLE * S);
  constexpr int NR = G::N / R;
  const float2* tw = twt + tw_off(S);
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = t + G::T * q;
    const int k = j & (Ns - 1);
    float2 w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = buf[pad(j + r * NR)];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      float2 c = __ldg(tw + (r - 1) * Ns + k);
      if (SIGN > 0) c.y = -c.y;
      w[r] = cmul(w[r], c);
    }
    dft<R, SIGN>(w);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q + Q * r] = w[r];
  }
}

// Write a radix-E stage's outputs (item j = t, span Ns) to Stockham positions.
template <int S>
__device__ __forceinline__ void stage_out(const float2 (&v)[1 << kLE], float2* buf, int t) {
  constexpr int E = 1 << kLE;
  constexpr int Ns = 1 << (kLE * S);
  const int k = t & (Ns - 1);
  const int o = (t - k) * E + k;
#pragma unroll
  for (int r = 0; r < E; ++r) buf[pad(o + r * Ns)] = v[r];
}

template <int LOGN, int S, int SIGN>
struct Stages {
  __device__ __forceinline__ static void run(float2 (&v)[1 << kLE], float2* buf, int t,
                                             const float2* __restrict__ twt, bool active) {
    using G = Geo<LOGN>;
    if (active) stage_in<LOGN, S, SIGN>(v, buf, t, twt);
    if constexpr (S < G::NST - 1) {
      __syncthreads();  // every thread has read this stage's inputs
      if (active) stage_out<S>(v, buf, t);
      __syncthreads();
      Stages<LOGN, S + 1, SIGN>::run(v, buf, t, twt, active);
    }
  }
};

// In: v[e] = x[t + T e]; out: v[e] = X[t + T e] (unnormalised, SIGN -1
// forward / +1 inverse).  buf: the group's NP-entry buffer, clobbered; the
// engine's first barrier orders its writes after any earlier reads of buf.
template <int LOGN, int SIGN>
__device__ __forceinline__ void fft(float2 (&v)[1 << kLE], float2* buf, int t,
                                    const float2* __restrict__ twt, bool active) {
  if (active) dft<(1 << kLE), SIGN>(v);
  __syncthreads();
  if (active) stage_out<0>(v, buf, t);
  __syncthreads();
  Stages<LOGN, 1, SIGN>::run(v, buf, t, twt, active);
}

}  // namespace p2
}  // namespace ncsg
