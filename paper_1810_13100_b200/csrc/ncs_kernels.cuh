// Launch interfaces of the streaming NCS kernels (ncs_kernels.cu).
#pragma once

#include "ncsg_internal.cuh"

namespace ncsg {

struct DualArgs {
  int kind = 0, n = 0, positivity = 0;
  float alpha = 0.f, s_quad = 0.f, wd = 0.f, bound = 0.f;
  // data block (CT: sinogram rays [m_begin, m_end) of [batch][m]; DENOISE: nn pixels)
  const float* fp_part = nullptr;
  int n_strips = 0;
  size_t m = 0, m_begin = 0, m_end = 0;
  float* u0 = nullptr;   // data-block dual, batch stride u_stride
  float* axs = nullptr;  // cached R x [batch][m] (CT)
  const float* b = nullptr;
  float* ug = nullptr;   // gradient dual, batch stride u_stride
  float* up = nullptr;   // positivity dual, batch stride u_stride
  size_t u_stride = 0;
  const float* x = nullptr;
  const float* x_old = nullptr;
  int* flag = nullptr;
  const uint8_t* own = nullptr;  // orbit sharding: own[t] of ray t*det + d (nullable)
  int det = 0;
  // Orbit gather input (nullable): the new data-block dual also goes to
  // u4[b][orbit][pad + d].member (slot[t] = 4 * orbit + member, -1: none).
  float* u4 = nullptr;
  const int* slot = nullptr;
  int u4_row = 0, u4_pad = 0;
  size_t u4_stride = 0;  // floats per problem
  // Orbit-major data block (nullable; CT with u4): item (orbit o, detector d)
  // updates the rays d of the member angles orb_t[o] (-1: absent) and stores
  // their four duals as one coalesced 16-byte u4 cell.  Covers exactly the
  // rays of the listed (own) orbits.
  const int4* orb_t = nullptr;
  int n_orb = 0;
  int data_only = 0;  // section 0 only (the x-only blocks were fused into the row pass)
};
void launch_dual_update(const DualArgs& a, int batch, cudaStream_t s);
// Rebuilds u4 from u0 (fields u0, u_stride, m, det, u4, slot, u4_row, u4_pad, u4_stride).
void launch_u4_pack(const DualArgs& a, int batch, cudaStream_t s);

struct ObjArgs {
  int kind = 0, n = 0, positivity = 0, with_grad = 1;
  float wd = 0.f;
  const float* axs = nullptr;  // CT cached R x
  const float* b = nullptr;
  const float* x = nullptr;
  size_t m = 0, m_begin = 0, m_end = 0;
  const uint8_t* own = nullptr;  // orbit sharding (nullable)
  int det = 0;
  double* out = nullptr;  // [batch][objective_blocks()][4]
};
int objective_blocks();
void launch_objective(const ObjArgs& a, int batch, cudaStream_t s);

struct SemArgs {
  int n = 0;
  double alpha = 0.0, gamma = 0.0;
  const float* du = nullptr;
  const float* adx = nullptr;
  size_t range = 0, r_begin = 0, r_end = 0;
  const float* dx = nullptr;
  const float* mdx = nullptr;  // nullable (PDHG: M = gamma I handled by caller)
  double* out = nullptr;       // [batch][objective_blocks()][3]
  // sharded problems: data rays i < m0 count when in [m_begin, m_end) and
  // own[i / det] (own nullable); the replicated rest of the range and the
  // x-space term only on rank 0 (summed across ranks by the caller)
  size_t m0 = 0, m_begin = 0, m_end = ~size_t(0);
  const uint8_t* own = nullptr;
  int det = 1;
  int rank0 = 1;
};
void launch_seminorm(const SemArgs& a, int batch, cudaStream_t s);

struct StackArgs {
  int kind = 0, n = 0, n_strips = 0;
  float wd = 0.f;
  const float* fp_part = nullptr;
  const float* x = nullptr;
  float* out = nullptr;
  size_t m0 = 0, range = 0;
};
void launch_stacked_rest(const StackArgs& a, int batch, cudaStream_t s);

void launch_grad_forward(const float* x, float* out, int n, int batch, cudaStream_t s);
void launch_grad_adjoint(const float* g, float* out, int n, int batch, cudaStream_t s);
void launch_transpose(const float* in, float* out, int n, int batch, cudaStream_t s);
void launch_f64_to_f32(const double* in, float* out, size_t count, cudaStream_t s);
void launch_f32_to_f64(const float* in, double* out, size_t count, cudaStream_t s);
void launch_sub(const float* a, const float* b, float* out, size_t count, cudaStream_t s);

}  // namespace ncsg

namespace ncsg {
// out[batch][n*n] = A^T u assembled from `T` (sharded multi-GPU path).
void launch_atu_assemble(const AtuTerms& T, float* out, int batch, cudaStream_t s);
// The same sum, batch 1, row y stored into rank y / R's slot `rank` over peer
// memory (the fused P2P reduce-scatter of the sharded slab step).
void launch_atu_assemble_scatter(const AtuTerms& T, const PeerPtrs& slots, int R, int rank,
                                 cudaStream_t s);

// Setup path (calibrate_scale, power-method screen): out[batch][blocks][2] =
// per-block [sum a*b, sum c*d] over `count` elements of each batch entry.
int dot_pair_blocks();
void launch_dot_pair(const float* a, const float* b, const float* c, const float* d, size_t count,
                     int batch, double* out, cudaStream_t s);
void launch_screen_combine(const float* v, const float* atav, const float* cv, float alpha,
                           float gamma, float shift, float* w, size_t count, cudaStream_t s);
void launch_scale(const float* in, float sc, float* out, size_t count, cudaStream_t s);

// ADMM-CG x-update (admm_cg_solve, solvers.cpp:135-145, 442-463): fp64 CG
// iterates, fp32 operator.  out[dot_pair_blocks()] = per-block partial sums.
void launch_cg_update(double* x, double* r, const double* p, const float* ap, double a,
                      size_t count, double* out, cudaStream_t s);
void launch_cg_direction(double* p, const double* r, double beta, float* p32, size_t count,
                         cudaStream_t s);
void launch_cg_dot(const double* p, const float* ap, size_t count, double* out, cudaStream_t s);
void launch_x_update(float* x, float* x_old, const double* d, double inv_alpha, size_t count,
                     int* flag, cudaStream_t s);

// empirical_mask (circulant.cpp:98-140) on half spectra [batch][n/2+1][n]:
// out[batch][dot_pair_blocks()] partial sums of the full-spectrum |F v|^2;
// sum / hits accumulate F(Av)/F(v) where |F v| >= cutoff[b].
void launch_spec_norm(const float2* spec, int n, int batch, double* out, cudaStream_t s);
void launch_mask_accumulate(const float2* fv, const float2* fav, const double* cutoff, int batch,
                            size_t total, double2* sum, int* hits, cudaStream_t s);
}  // namespace ncsg
