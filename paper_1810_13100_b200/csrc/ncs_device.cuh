// Device helpers shared by the FFT row pass and the stand-alone A^T u
// assembly (sharded multi-GPU path).
#pragma once

#include "ncsg_internal.cuh"

namespace ncsg {

// Loads of the partial-image sums kept in flight per thread (the row pass
// loader sums up to 48 adjoint partials per pixel at C3).
#ifndef NCSG_PART_UNROLL
#define NCSG_PART_UNROLL 4
#endif
constexpr int kPartUnroll = NCSG_PART_UNROLL;

// A^T u (or a plain image) at (y, x) from the row-major terms.  The
// transposed class-H partials are added separately (coalesced by columns).
__device__ __forceinline__ float atu_rowmajor(const AtuTerms& T, int b, int y, int x) {
  const int n = T.n;
  const size_t nn = static_cast<size_t>(n) * n;
  const size_t i = static_cast<size_t>(y) * n + x;
  if (T.plain) return T.plain[b * nn + i];
  float v = 0.f;
  if (T.bp_part) {
    const float* p = T.bp_part + b * T.part_stride + i;
    const size_t ps = T.img_stride ? T.img_stride : nn;
#pragma unroll kPartUnroll
    for (int c = 0; c < T.nV; ++c) v += p[c * ps];
  }
  if (T.ident) v += T.ident[b * T.ident_stride + i];
  if (T.ident2) v += T.ident2[b * T.ident_stride + i];
  if (T.ug) {
    // D^T g (grad.cpp:66-84): h block N x (N-1), then v block (N-1) x N.
    const float* g = T.ug + b * T.ug_stride;
    const float* hb = g;
    const float* vb = g + static_cast<size_t>(n) * (n - 1);
    float d = 0.f;
    if (x < n - 1) d += hb[static_cast<size_t>(y) * (n - 1) + x];
    if (x > 0) d -= hb[static_cast<size_t>(y) * (n - 1) + x - 1];
    if (y < n - 1) d += vb[static_cast<size_t>(y) * n + x];
    if (y > 0) d -= vb[static_cast<size_t>(y - 1) * n + x];
    v += T.wd * d;
  }
  return v;
}

// Four consecutive pixels (x % 4 == 0, n % 4 == 0) of A^T u: the partial
// images are read as float4 (a quarter of the load instructions, so more of
// the many partial reads are in flight); the other terms per pixel.
__device__ __forceinline__ float4 atu_rowmajor4(const AtuTerms& T, int b, int y, int x) {
  const int n = T.n;
  const size_t nn = static_cast<size_t>(n) * n;
  const size_t i = static_cast<size_t>(y) * n + x;
  if (T.plain) return *reinterpret_cast<const float4*>(T.plain + b * nn + i);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (T.bp_part) {
    const float* p = T.bp_part + b * T.part_stride + i;
    const size_t ps = T.img_stride ? T.img_stride : nn;
#pragma unroll kPartUnroll
    for (int c = 0; c < T.nV; ++c) {
      const float4 q = *reinterpret_cast<const float4*>(p + c * ps);
      v.x += q.x, v.y += q.y, v.z += q.z, v.w += q.w;
    }
  }
  // float4 paths need 16-byte aligned rows (n % 4 == 0 here): checked on the
  // problem's pointers
  const auto a16 = [](const float* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool al = (!T.ident || a16(T.ident + b * T.ident_stride)) &&
                  (!T.ident2 || a16(T.ident2 + b * T.ident_stride));
  if (T.ident && al) {
    const float4 q = *reinterpret_cast<const float4*>(T.ident + b * T.ident_stride + i);
    v.x += q.x, v.y += q.y, v.z += q.z, v.w += q.w;
  }
  if (T.ident2 && al) {
    const float4 q = *reinterpret_cast<const float4*>(T.ident2 + b * T.ident_stride + i);
    v.x += q.x, v.y += q.y, v.z += q.z, v.w += q.w;
  }
  if (T.ug && al && a16(T.ug + b * T.ug_stride + static_cast<size_t>(n) * (n - 1))) {
    // D^T g for pixels x..x+3 (grad.cpp:66-84): h block rows of n-1 (scalar),
    // v block rows of n (float4)
    const float* g = T.ug + b * T.ug_stride;
    const float* hr = g + static_cast<size_t>(y) * (n - 1);
    const float* vb = g + static_cast<size_t>(n) * (n - 1);
    float h[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int c = x - 1 + q;  // h columns x-1 .. x+3
      h[q] = (c >= 0 && c < n - 1) ? hr[c] : 0.f;
    }
    const float4 vc = y < n - 1 ? *reinterpret_cast<const float4*>(vb + static_cast<size_t>(y) * n + x)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 vp = y > 0 ? *reinterpret_cast<const float4*>(vb + static_cast<size_t>(y - 1) * n + x)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    const float w = T.wd;
    v.x += w * ((h[1] - h[0]) + (vc.x - vp.x));
    v.y += w * ((h[2] - h[1]) + (vc.y - vp.y));
    v.z += w * ((h[3] - h[2]) + (vc.z - vp.z));
    v.w += w * ((h[4] - h[3]) + (vc.w - vp.w));
  } else if (T.ug || ((T.ident || T.ident2) && !al)) {
    AtuTerms R = T;
    R.plain = nullptr;
    R.bp_part = nullptr;
    if (al) R.ident = R.ident2 = nullptr;  // already added as float4
    v.x += atu_rowmajor(R, b, y, x);
    v.y += atu_rowmajor(R, b, y, x + 1);
    v.z += atu_rowmajor(R, b, y, x + 2);
    v.w += atu_rowmajor(R, b, y, x + 3);
  }
  return v;
}

}  // namespace ncsg
