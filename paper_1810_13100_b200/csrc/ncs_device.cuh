// Device helpers shared by the FFT row pass and the stand-alone A^T u
// assembly (sharded multi-GPU path).
#pragma once

#include "ncsg_internal.cuh"

namespace ncsg {

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
    for (int c = 0; c < T.nV; ++c) v += p[c * nn];
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

}  // namespace ncsg
