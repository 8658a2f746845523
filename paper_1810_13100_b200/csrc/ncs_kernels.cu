// Streaming kernels of the NCS step: the fused dual update (extrapolation +
// conjugate proxes + ax cache + finiteness flag), the objective reduction,
// stand-alone D / D^T, and small vector helpers.  All HBM-bound; each element
// of u, ax and b crosses HBM once per step.
#include <cuda_runtime.h>

#include <algorithm>

#include "ncs_device.cuh"
#include "ncs_kernels.cuh"

namespace ncsg {

namespace {

int grid_for(size_t total, int block, int cap = 148 * 8) {
  size_t g = (total + block - 1) / block;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(g, cap)));
}

// w * (D x)_e with D the forward difference of grad.cpp:53-64.
__device__ __forceinline__ float grad_at(const float* x, int n, size_t e) {
  const size_t half = static_cast<size_t>(n) * (n - 1);
  if (e < half) {
    const size_t i = e / (n - 1), j = e - i * (n - 1);
    const float* p = x + i * n + j;
    return p[0] - p[1];
  }
  const size_t e2 = e - half;
  const size_t i = e2 / n, j = e2 - i * n;
  const float* p = x + i * n + j;
  return p[0] - p[n];
}

// Engine::step dual half (solvers.cpp:148-156) for every block:
//   r = u + alpha (2 ax_new - ax_old - b);  u = prox_{alpha g*}(r)
// with QuadraticConj (prox.cpp:21-24), ScaledL1Conj (prox.cpp:36-38, bound
// lambda*alpha/beta) and NonnegConj (prox.cpp:103-105); CT data rays also
// sum the projector's strip partials into ax_new and store it as the new ax.
// Orbit-interleaved copy of the sinogram dual for bp_gather_kernel.
__device__ __forceinline__ void put_u4(const DualArgs& a, int b, size_t i, float v) {
  const int t = static_cast<int>(i / a.det);
  const int sl = a.slot[t];
  if (sl < 0) return;
  const size_t d = i - static_cast<size_t>(t) * a.det;
  a.u4[b * a.u4_stride + ((static_cast<size_t>(sl >> 2) * a.u4_row + a.u4_pad + d) << 2) + (sl & 3)] = v;
}

__global__ void dual_update_kernel(DualArgs a) {
  pdl_wait();
  const int b = blockIdx.z;
  const int section = blockIdx.y;
  const float alpha = a.alpha;
  const size_t nn = static_cast<size_t>(a.n) * a.n;
  const float* x = a.x + b * nn;
  const float* xo = a.x_old + b * nn;
  bool bad = false;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t i0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (section == 0) {
    if (a.kind == NCSG_CT) {
      const float* part = a.fp_part + b * a.n_strips * a.m;
      float* us = a.u0 + b * a.u_stride;
      float* ax = a.axs + b * a.m;
      const float* bb = a.b + b * a.m;
      if (a.orb_t) {
        // orbit-major: a block item is (orbit o, 64 detectors); thread
        // (member k, detector d) updates ray t_k*det + d (coalesced along d),
        // then the four members of each detector leave as one 16-byte u4 cell
        __shared__ float sh[4][64];
        const int nch = (a.det + 63) / 64;
        const size_t items = static_cast<size_t>(a.n_orb) * nch;
        float4* u4b = reinterpret_cast<float4*>(a.u4 + b * a.u4_stride);
        const int k = threadIdx.x >> 6, dl = threadIdx.x & 63;
        for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
          const int o = static_cast<int>(it / nch);
          const int d = static_cast<int>(it - static_cast<size_t>(o) * nch) * 64 + dl;
          const int t = __ldg(reinterpret_cast<const int*>(a.orb_t + o) + k);
          float un = 0.f;
          if (t >= 0 && d < a.det) {
            const size_t i = static_cast<size_t>(t) * a.det + d;
            float rx = 0.f;
            for (int q = 0; q < a.n_strips; ++q) rx += part[q * a.m + i];
            un = (us[i] + alpha * (2.f * rx - ax[i] - bb[i])) * a.s_quad;
            us[i] = un;
            ax[i] = rx;
            bad |= isnan(un);
          }
          sh[k][dl] = un;
          __syncthreads();
          if (threadIdx.x < 64 && d < a.det)
            u4b[static_cast<size_t>(o) * a.u4_row + a.u4_pad + d] =
                make_float4(sh[0][dl], sh[1][dl], sh[2][dl], sh[3][dl]);
          __syncthreads();
        }
      } else if (!a.own && ((a.m | a.m_begin | a.m_end | a.u_stride) & 3) == 0) {
        // four rays per thread, float4 loads of every partial slot
        for (size_t i = a.m_begin + 4 * i0; i < a.m_end; i += 4 * stride) {
          float4 rx = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int k = 0; k < a.n_strips; ++k) {
            const float4 q = *reinterpret_cast<const float4*>(part + k * a.m + i);
            rx.x += q.x, rx.y += q.y, rx.z += q.z, rx.w += q.w;
          }
          const float4 uo = *reinterpret_cast<const float4*>(us + i);
          const float4 ao = *reinterpret_cast<const float4*>(ax + i);
          const float4 bo = *reinterpret_cast<const float4*>(bb + i);
          float4 un;
          un.x = (uo.x + alpha * (2.f * rx.x - ao.x - bo.x)) * a.s_quad;
          un.y = (uo.y + alpha * (2.f * rx.y - ao.y - bo.y)) * a.s_quad;
          un.z = (uo.z + alpha * (2.f * rx.z - ao.z - bo.z)) * a.s_quad;
          un.w = (uo.w + alpha * (2.f * rx.w - ao.w - bo.w)) * a.s_quad;
          *reinterpret_cast<float4*>(us + i) = un;
          *reinterpret_cast<float4*>(ax + i) = rx;
          bad |= isnan(un.x) || isnan(un.y) || isnan(un.z) || isnan(un.w);
          if (a.u4) {
            put_u4(a, b, i, un.x);
            put_u4(a, b, i + 1, un.y);
            put_u4(a, b, i + 2, un.z);
            put_u4(a, b, i + 3, un.w);
          }
        }
      } else {
        for (size_t i = a.m_begin + i0; i < a.m_end; i += stride) {
          if (a.own && !a.own[i / a.det]) continue;  // another shard's orbit
          float rx = 0.f;
          for (int k = 0; k < a.n_strips; ++k) rx += part[k * a.m + i];
          const float r = us[i] + alpha * (2.f * rx - ax[i] - bb[i]);
          const float un = r * a.s_quad;
          us[i] = un;
          ax[i] = rx;
          bad |= isnan(un);
          if (a.u4) put_u4(a, b, i, un);
        }
      }
    } else if (a.kind == NCSG_PET) {
      // PoissonConj block (pipeline.cpp:86-88): offset 0, counts in b,
      // u = prox_conj_poisson(r, alpha * counts) (prox.cpp:9-13, 56-60) in the
      // cancellation-free form 1 + (d - sqrt(d^2 + 4c)) / 2 = 1 - 2c / (d + sqrt(...)).
      const float* part = a.fp_part + b * a.n_strips * a.m;
      float* us = a.u0 + b * a.u_stride;
      float* ax = a.axs + b * a.m;
      const float* cnt = a.b + b * a.m;
      for (size_t i = a.m_begin + i0; i < a.m_end; i += stride) {
        if (a.own && !a.own[i / a.det]) continue;  // another shard's orbit
        float rx = 0.f;
        for (int k = 0; k < a.n_strips; ++k) rx += part[k * a.m + i];
        const double r = static_cast<double>(us[i]) + alpha * (2.f * rx - ax[i]);
        const double c = static_cast<double>(alpha) * cnt[i];
        const double d = r - 1.0;
        const double sq = sqrt(d * d + 4.0 * c);
        const double un = d > 0.0 ? 1.0 - 2.0 * c / (d + sq) : 1.0 + 0.5 * (d - sq);
        us[i] = static_cast<float>(un);
        ax[i] = rx;
        bad |= isnan(un);
        if (a.u4) put_u4(a, b, i, static_cast<float>(un));
      }
    } else {
      float* ud = a.u0 + b * a.u_stride;
      const float* bb = a.b + b * nn;
      if (((nn | a.u_stride) & 3) == 0) {  // four pixels per thread, float4
        for (size_t i = 4 * i0; i < nn; i += 4 * stride) {
          const float4 u0 = *reinterpret_cast<const float4*>(ud + i);
          const float4 x4 = *reinterpret_cast<const float4*>(x + i);
          const float4 o4 = *reinterpret_cast<const float4*>(xo + i);
          const float4 b4 = *reinterpret_cast<const float4*>(bb + i);
          float4 un;
          un.x = (u0.x + alpha * (2.f * x4.x - o4.x - b4.x)) * a.s_quad;
          un.y = (u0.y + alpha * (2.f * x4.y - o4.y - b4.y)) * a.s_quad;
          un.z = (u0.z + alpha * (2.f * x4.z - o4.z - b4.z)) * a.s_quad;
          un.w = (u0.w + alpha * (2.f * x4.w - o4.w - b4.w)) * a.s_quad;
          *reinterpret_cast<float4*>(ud + i) = un;
          bad |= isnan(un.x) || isnan(un.y) || isnan(un.z) || isnan(un.w);
        }
      } else {
        for (size_t i = i0; i < nn; i += stride) {
          const float r = ud[i] + alpha * (2.f * x[i] - xo[i] - bb[i]);
          const float un = r * a.s_quad;
          ud[i] = un;
          bad |= isnan(un);
        }
      }
    }
  } else if (section == 1) {
    float* ug = a.ug + b * a.u_stride;
    const size_t g = 2 * static_cast<size_t>(a.n) * (a.n - 1);
    const float wd = a.wd, bd = a.bound;
    if (((a.ug - a.u0) & 3) == 0 && (a.u_stride & 3) == 0 && (g & 3) == 0) {
      // four edges per thread: the dual as float4, the differences per edge
      for (size_t e = 4 * i0; e < g; e += 4 * stride) {
        const float4 u4v = *reinterpret_cast<const float4*>(ug + e);
        const float uo[4] = {u4v.x, u4v.y, u4v.z, u4v.w};
        float un[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float an = wd * grad_at(x, a.n, e + q);
          const float ao = wd * grad_at(xo, a.n, e + q);
          const float z = uo[q] + alpha * (2.f * an - ao - 0.f);
          un[q] = z < -bd ? -bd : (z > bd ? bd : z);
          bad |= isnan(z);
        }
        *reinterpret_cast<float4*>(ug + e) = make_float4(un[0], un[1], un[2], un[3]);
      }
    } else {
      for (size_t e = i0; e < g; e += stride) {
        const float an = wd * grad_at(x, a.n, e);
        const float ao = wd * grad_at(xo, a.n, e);
        const float z = ug[e] + alpha * (2.f * an - ao - 0.f);
        const float un = z < -bd ? -bd : (z > bd ? bd : z);
        ug[e] = un;
        bad |= isnan(z);
      }
    }
  } else {
    float* up = a.up + b * a.u_stride;
    for (size_t i = i0; i < nn; i += stride) {
      const float z = up[i] + alpha * (2.f * x[i] - xo[i]);
      up[i] = z < 0.f ? z : 0.f;
      bad |= isnan(z);
    }
  }
  // dual NaN (check_finite's second test, solvers.cpp:252-254): flag word 2
  if (a.flag && __syncthreads_or(bad) && threadIdx.x == 0)
    atomicMin(a.flag + 2, *(volatile int*)(a.flag + 1));
}

__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (blockDim.x >> 5); ++k) s += sh[k];
  return s;
}

__device__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (blockDim.x >> 5); ++k) s = fmax(s, sh[k]);
  return s;
}

// Per-block fp64 partial sums of objective_from_ax (solvers.cpp:362-381):
// [0] sum (ax_data - b)^2, [1] sum |w D x|, [2] max |x| (positivity),
// [3] min x (positivity).
__global__ void objective_kernel(ObjArgs a) {
  __shared__ double sh[32];
  const int b = blockIdx.y;
  const size_t nn = static_cast<size_t>(a.n) * a.n;
  const float* x = a.x + b * nn;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t i0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  double q = 0.0, l1 = 0.0, mx = 0.0, mn = 0.0;
  if (a.kind == NCSG_CT) {
    const float* ax = a.axs + b * a.m;
    const float* bb = a.b + b * a.m;
    for (size_t i = a.m_begin + i0; i < a.m_end; i += stride) {
      if (a.own && !a.own[i / a.det]) continue;
      const double z = static_cast<double>(ax[i]) - static_cast<double>(bb[i]);
      q += z * z;
    }
  } else if (a.kind == NCSG_PET) {
    // PoissonConj::objective (prox.cpp:62-74): sum y - c log y, +inf outside the domain
    const float* ax = a.axs + b * a.m;
    const float* cnt = a.b + b * a.m;
    for (size_t i = a.m_begin + i0; i < a.m_end; i += stride) {
      if (a.own && !a.own[i / a.det]) continue;
      const double y = ax[i], c = cnt[i];
      if (c > 0.0)
        q += y <= 0.0 ? INFINITY : y - c * log(y);
      else
        q += y < 0.0 ? INFINITY : y;
    }
  } else {
    const float* bb = a.b + b * nn;
    for (size_t i = i0; i < nn; i += stride) {
      const double z = static_cast<double>(x[i]) - static_cast<double>(bb[i]);
      q += z * z;
    }
  }
  if (a.with_grad) {
    const size_t g = 2 * static_cast<size_t>(a.n) * (a.n - 1);
    for (size_t e = i0; e < g; e += stride)
      l1 += fabs(static_cast<double>(a.wd * grad_at(x, a.n, e)));
  }
  if (a.positivity) {
    for (size_t i = i0; i < nn; i += stride) {
      mx = fmax(mx, fabs(static_cast<double>(x[i])));
      mn = fmin(mn, static_cast<double>(x[i]));
    }
  }
  double* out = a.out + (static_cast<size_t>(b) * gridDim.x + blockIdx.x) * 4;
  const double s0 = block_sum(q, sh);
  if (threadIdx.x == 0) out[0] = s0;
  const double s1 = block_sum(l1, sh);
  if (threadIdx.x == 0) out[1] = s1;
  const double s2 = block_max(mx, sh);
  if (threadIdx.x == 0) out[2] = s2;
  const double s3 = -block_max(-mn, sh);
  if (threadIdx.x == 0) out[3] = s3;
}

__global__ void grad_forward_kernel(const float* x, float* out, int n, int batch) {
  const size_t g = 2 * static_cast<size_t>(n) * (n - 1);
  const size_t nn = static_cast<size_t>(n) * n;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < g * batch;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t b = i / g, e = i - b * g;
    out[i] = grad_at(x + b * nn, n, e);
  }
}

__global__ void grad_adjoint_kernel(const float* gbuf, float* out, int n, int batch) {
  const size_t g = 2 * static_cast<size_t>(n) * (n - 1);
  const size_t nn = static_cast<size_t>(n) * n;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nn * batch;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t b = i / nn, p = i - b * nn;
    const int y = static_cast<int>(p / n), x = static_cast<int>(p - static_cast<size_t>(y) * n);
    const float* hb = gbuf + b * g;
    const float* vb = hb + static_cast<size_t>(n) * (n - 1);
    float d = 0.f;
    if (x < n - 1) d += hb[static_cast<size_t>(y) * (n - 1) + x];
    if (x > 0) d -= hb[static_cast<size_t>(y) * (n - 1) + x - 1];
    if (y < n - 1) d += vb[static_cast<size_t>(y) * n + x];
    if (y > 0) d -= vb[static_cast<size_t>(y - 1) * n + x];
    out[i] = d;
  }
}

__global__ void transpose_kernel(const float* in, float* out, int n, int batch) {
  __shared__ float t[32][33];
  const size_t nn = static_cast<size_t>(n) * n;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = by + k, x = bx + threadIdx.x;
    if (y < n && x < n) t[k][threadIdx.x] = in[b * nn + static_cast<size_t>(y) * n + x];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = bx + k, x = by + threadIdx.x;
    if (y < n && x < n) out[b * nn + static_cast<size_t>(y) * n + x] = t[threadIdx.x][k];
  }
}

__global__ void f64_to_f32_kernel(const double* in, float* out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}

__global__ void f32_to_f64_kernel(const float* in, double* out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}

// out = a - b (fp32), used for the seminorm step differences.
__global__ void sub_kernel(const float* a, const float* b, float* out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] - b[i];
}

// Seminorm partial sums (solvers.cpp:166-177), per block:
//   [0] sum (du - alpha adx)^2   [1] sum adx^2   [2] sum dx * mdx
__global__ void seminorm_kernel(SemArgs a) {
  __shared__ double sh[32];
  const int b = blockIdx.y;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t i0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const float* du = a.du + b * a.range;
  const float* adx = a.adx + b * a.range;
  double t1 = 0.0, aq = 0.0, mq = 0.0;
  for (size_t i = i0; i < a.range; i += stride) {
    const bool mine = i < a.m0 ? (i >= a.m_begin && i < a.m_end && (!a.own || a.own[i / a.det]))
                               : a.rank0 != 0;
    if (mine && i >= a.r_begin && i < a.r_end) {
      const double d = static_cast<double>(du[i]) - a.alpha * static_cast<double>(adx[i]);
      t1 += d * d;
      aq += static_cast<double>(adx[i]) * adx[i];
    }
  }
  const size_t nn = static_cast<size_t>(a.n) * a.n;
  if (a.rank0) {
    const float* dx = a.dx + b * nn;
    const float* w = a.mdx ? a.mdx + b * nn : nullptr;  // F^-1 (h F dx) (Engine::apply_m)
    for (size_t i = i0; i < nn; i += stride) {
      const double d = dx[i];
      mq += d * (a.gamma * d + (w ? a.alpha * static_cast<double>(w[i]) : 0.0));
    }
  }
  double* out = a.out + (static_cast<size_t>(b) * gridDim.x + blockIdx.x) * 3;
  const double s0 = block_sum(t1, sh);
  if (threadIdx.x == 0) out[0] = s0;
  const double s1 = block_sum(aq, sh);
  if (threadIdx.x == 0) out[1] = s1;
  const double s2 = block_sum(mq, sh);
  if (threadIdx.x == 0) out[2] = s2;
}

// Stacked forward of dx for the seminorm: data block (strip sum or identity),
// D block (weighted) and positivity identity, into adx[batch][range].
__global__ void stacked_rest_kernel(StackArgs a) {
  const int b = blockIdx.y;
  const size_t nn = static_cast<size_t>(a.n) * a.n;
  const size_t g = 2 * static_cast<size_t>(a.n) * (a.n - 1);
  const float* x = a.x + b * nn;
  float* out = a.out + b * a.range;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < a.range;
       i += stride) {
    float v;
    if (i < a.m0) {
      if (a.kind != NCSG_DENOISE) {
        const float* part = a.fp_part + b * a.n_strips * a.m0 + i;
        v = 0.f;
        for (int k = 0; k < a.n_strips; ++k) v += part[k * a.m0];
      } else {
        v = x[i];
      }
    } else if (i < a.m0 + g) {
      v = a.wd * grad_at(x, a.n, i - a.m0);
    } else {
      v = x[i - a.m0 - g];
    }
    out[i] = v;
  }
}

}  // namespace

#ifndef NCSG_DUAL_WAVES
#define NCSG_DUAL_WAVES 8
#endif
void launch_dual_update(const DualArgs& a, int batch, cudaStream_t s) {
  size_t big = std::max<size_t>(a.m_end - a.m_begin, 2 * static_cast<size_t>(a.n) * a.n);
  if (a.data_only) big = a.m_end - a.m_begin;
  dim3 grid(grid_for(big, 256, 148 * NCSG_DUAL_WAVES), a.data_only ? 1 : (a.positivity ? 3 : 2),
            batch);
  launch_pdl(dual_update_kernel, grid, dim3(256), 0, s, a);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

// u4 from u for every owned sinogram ray (after the state was set from
// outside the dual update).
__global__ void u4_pack_kernel(DualArgs a) {
  const int b = blockIdx.y;
  const float* us = a.u0 + b * a.u_stride;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < a.m;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    put_u4(a, b, i, us[i]);
}

void launch_u4_pack(const DualArgs& a, int batch, cudaStream_t s) {
  dim3 grid(grid_for(a.m, 256, 148 * 4), batch);
  u4_pack_kernel<<<grid, 256, 0, s>>>(a);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

int objective_blocks() { return 148; }

void launch_objective(const ObjArgs& a, int batch, cudaStream_t s) {
  dim3 grid(objective_blocks(), batch);
  objective_kernel<<<grid, 256, 0, s>>>(a);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_grad_forward(const float* x, float* out, int n, int batch, cudaStream_t s) {
  size_t total = 2 * static_cast<size_t>(n) * (n - 1) * batch;
  grad_forward_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, out, n, batch);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_grad_adjoint(const float* g, float* out, int n, int batch, cudaStream_t s) {
  size_t total = static_cast<size_t>(n) * n * batch;
  grad_adjoint_kernel<<<grid_for(total, 256), 256, 0, s>>>(g, out, n, batch);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_transpose(const float* in, float* out, int n, int batch, cudaStream_t s) {
  dim3 grid((n + 31) / 32, (n + 31) / 32, batch);
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, out, n, batch);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_f64_to_f32(const double* in, float* out, size_t count, cudaStream_t s) {
  f64_to_f32_kernel<<<grid_for(count, 256), 256, 0, s>>>(in, out, count);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_f32_to_f64(const float* in, double* out, size_t count, cudaStream_t s) {
  f32_to_f64_kernel<<<grid_for(count, 256), 256, 0, s>>>(in, out, count);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_sub(const float* a, const float* b, float* out, size_t count, cudaStream_t s) {
  sub_kernel<<<grid_for(count, 256), 256, 0, s>>>(a, b, out, count);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_seminorm(const SemArgs& a, int batch, cudaStream_t s) {
  dim3 grid(objective_blocks(), batch);
  seminorm_kernel<<<grid, 256, 0, s>>>(a);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_stacked_rest(const StackArgs& a, int batch, cudaStream_t s) {
  dim3 grid(grid_for(a.range, 256), batch);
  stacked_rest_kernel<<<grid, 256, 0, s>>>(a);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

}  // namespace ncsg

namespace ncsg {
namespace {
__global__ void sum_partials_kernel(const float* part, int nV, int nH, float* out, int n) {
  __shared__ float t[32][33];
  const size_t nn = static_cast<size_t>(n) * n;
  const int b = blockIdx.z;
  const float* pb = part + static_cast<size_t>(b) * (nV + nH) * nn;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  // class-H partials are stored transposed: stage them through shared memory
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = bx + k, x = by + threadIdx.x;  // transposed coordinates
    float v = 0.f;
    if (y < n && x < n)
      for (int c = 0; c < nH; ++c) v += pb[(nV + c) * nn + static_cast<size_t>(y) * n + x];
    t[k][threadIdx.x] = v;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = by + k, x = bx + threadIdx.x;
    if (y >= n || x >= n) continue;
    float v = 0.f;
    for (int c = 0; c < nV; ++c) v += pb[c * nn + static_cast<size_t>(y) * n + x];
    out[b * nn + static_cast<size_t>(y) * n + x] = v + t[threadIdx.x][k];
  }
}
}  // namespace

void launch_sum_partials(const float* part, int nV, int nH, float* out, int n, int batch,
                         cudaStream_t s) {
  dim3 grid((n + 31) / 32, (n + 31) / 32, batch);
  sum_partials_kernel<<<grid, dim3(32, 8), 0, s>>>(part, nV, nH, out, n);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}
}  // namespace ncsg

namespace ncsg {
namespace {
// A^T u as one image: class-V partials + transposed class-H partials (through
// a shared-memory tile) + identity blocks + w D^T u_g (linear_map.cpp:47-55).
// Per-block partial sums [sum a*b, sum c*d] in fp64 for the setup path
// (power_method dots, calibrate_scale sums); block partials are added on the
// host in block order, so results are deterministic.
__global__ void dot_pair_kernel(const float* a, const float* b, const float* c, const float* d,
                                size_t count, double* out) {
  __shared__ double sh[32];
  const size_t off = static_cast<size_t>(blockIdx.y) * count;
  double s0 = 0.0, s1 = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    s0 += static_cast<double>(a[off + i]) * b[off + i];
    s1 += static_cast<double>(c[off + i]) * d[off + i];
  }
  double* o = out + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 2;
  const double t0 = block_sum(s0, sh);
  if (threadIdx.x == 0) o[0] = t0;
  const double t1 = block_sum(s1, sh);
  if (threadIdx.x == 0) o[1] = t1;
}

// The shifted screen operator (solvers.cpp:228-237):
//   w = alpha * A^T A v - M v + shift * v,  M v = gamma v + alpha * (C v).
__global__ void screen_combine_kernel(const float* v, const float* atav, const float* cv,
                                      float alpha, float gamma, float shift, float* w,
                                      size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float mv = gamma * v[i] + (cv ? alpha * cv[i] : 0.f);
    w[i] = alpha * atav[i] - mv + shift * v[i];
  }
}

// CG step of cg (solvers.cpp:456-459) with fp64 iterates (the operator runs
// in fp32): x += a p; r -= a ap; per-block partial sums of r.r into out[block].
__global__ void cg_update_kernel(double* x, double* r, const double* p, const float* ap,
                                 double a, size_t count, double* out) {
  __shared__ double sh[32];
  double rr = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    x[i] += a * p[i];
    const double ri = r[i] - a * static_cast<double>(ap[i]);
    r[i] = ri;
    rr += ri * ri;
  }
  const double t = block_sum(rr, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = t;
}

// p = r + beta p (solvers.cpp:461), plus the fp32 copy the operator reads.
__global__ void cg_direction_kernel(double* p, const double* r, double beta, float* p32,
                                    size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double v = r[i] + beta * p[i];
    p[i] = v;
    p32[i] = static_cast<float>(v);
  }
}

// p.ap with fp64 p (power of the CG denominator) -- per-block partials.
__global__ void cg_dot_kernel(const double* p, const float* ap, size_t count, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    acc += p[i] * static_cast<double>(ap[i]);
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = t;
}

// ADMM-CG x update (solvers.cpp:138-145): x_old = x; x -= inv_alpha * d; the
// check_finite flag (solvers.cpp:248-255) and the step counter like c2r.
__global__ void x_update_kernel(float* x, float* x_old, const double* d, double inv_alpha,
                                size_t count, int* flag) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && flag) atomicAdd(flag + 1, 1);
  int bad = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float xo = x[i];
    x_old[i] = xo;
    const float xn = static_cast<float>(xo - inv_alpha * d[i]);
    x[i] = xn;
    bad |= !isfinite(xn);
  }
  if (flag && __syncthreads_or(bad) && threadIdx.x == 0)
    atomicMin(flag, *(volatile int*)(flag + 1));
}

// empirical_mask (circulant.cpp:119-127) on the half spectrum specT[k][j]:
// per-block partial sums of sum |F v|^2 over the FULL spectrum (columns
// 0 < k < n/2 stand for two bins each).
__global__ void spec_norm_kernel(const float2* spec, int n, double* out) {
  __shared__ double sh[32];
  const int nk = n / 2 + 1;
  const size_t total = static_cast<size_t>(nk) * n;
  const float2* sb = spec + blockIdx.y * total;
  double acc = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / n);
    const double w = (k == 0 || 2 * k == n) ? 1.0 : 2.0;  // self-conjugate columns count once
    const double a = sb[i].x, b = sb[i].y;
    acc += w * (a * a + b * b);
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// sum += F(Av) / F(v), hits += 1 where |F v| >= cutoff[b] (fp64 division).
__global__ void mask_accumulate_kernel(const float2* fv, const float2* fav, const double* cutoff,
                                       int batch, size_t total, double2* sum, int* hits) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double2 s = sum[i];
    int h = hits[i];
    for (int b = 0; b < batch; ++b) {
      const double a = fv[b * total + i].x, c0 = fv[b * total + i].y;
      if (hypot(a, c0) < cutoff[b]) continue;
      const double c = fav[b * total + i].x, d = fav[b * total + i].y;
      const double den = a * a + c0 * c0;
      s.x += (c * a + d * c0) / den;
      s.y += (d * a - c * c0) / den;
      ++h;
    }
    sum[i] = s;
    hits[i] = h;
  }
}

__global__ void scale_kernel(const float* in, float s, float* out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = s * in[i];
}

__global__ void atu_assemble_kernel(AtuTerms T, float* out) {
  __shared__ float t[32][33];
  const int n = T.n;
  const size_t nn = static_cast<size_t>(n) * n;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const float* ph = T.bp_part ? T.bp_part + b * T.part_stride + T.nV * nn : nullptr;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = bx + k, x = by + threadIdx.x;  // transposed coordinates
    float v = 0.f;
    if (ph && y < n && x < n)
      for (int c = 0; c < T.nH; ++c) v += ph[c * nn + static_cast<size_t>(y) * n + x];
    t[k][threadIdx.x] = v;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = by + k, x = bx + threadIdx.x;
    if (y >= n || x >= n) continue;
    out[b * nn + static_cast<size_t>(y) * n + x] = atu_rowmajor(T, b, y, x) + t[threadIdx.x][k];
  }
}
// The fused P2P reduce-scatter: this rank's A^T u (partials summed as in
// atu_assemble_kernel), row y stored straight into its owner rank q = y / R's
// receive slots at [src rank][y - q R][x] over peer memory (NVLink).  The
// owner sums its P slots in rank order (deterministic).
__global__ void atu_assemble_scatter_kernel(AtuTerms T, PeerPtrs slots, int R, int rank) {
  __shared__ float t[32][33];
  const int n = T.n;
  const size_t nn = static_cast<size_t>(n) * n;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const float* ph = T.bp_part ? T.bp_part + T.nV * nn : nullptr;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = bx + k, x = by + threadIdx.x;  // transposed coordinates
    float v = 0.f;
    if (ph && y < n && x < n)
      for (int c = 0; c < T.nH; ++c) v += ph[c * nn + static_cast<size_t>(y) * n + x];
    t[k][threadIdx.x] = v;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int y = by + k, x = bx + threadIdx.x;
    if (y >= n || x >= n) continue;
    const int q = y / R;
    float* dst = static_cast<float*>(slots.p[q]) +
                 (static_cast<size_t>(rank) * R + (y - q * R)) * n + x;
    *dst = atu_rowmajor(T, 0, y, x) + t[threadIdx.x][k];
  }
}
}  // namespace

void launch_atu_assemble_scatter(const AtuTerms& T, const PeerPtrs& slots, int R, int rank,
                                 cudaStream_t s) {
  dim3 grid((T.n + 31) / 32, (T.n + 31) / 32, 1);
  atu_assemble_scatter_kernel<<<grid, dim3(32, 8), 0, s>>>(T, slots, R, rank);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_atu_assemble(const AtuTerms& T, float* out, int batch, cudaStream_t s) {
  dim3 grid((T.n + 31) / 32, (T.n + 31) / 32, batch);
  atu_assemble_kernel<<<grid, dim3(32, 8), 0, s>>>(T, out);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}
int dot_pair_blocks() { return 148; }

void launch_dot_pair(const float* a, const float* b, const float* c, const float* d, size_t count,
                     int batch, double* out, cudaStream_t s) {
  dim3 grid(dot_pair_blocks(), batch);
  dot_pair_kernel<<<grid, 256, 0, s>>>(a, b, c, d, count, out);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_screen_combine(const float* v, const float* atav, const float* cv, float alpha,
                           float gamma, float shift, float* w, size_t count, cudaStream_t s) {
  screen_combine_kernel<<<grid_for(count, 256), 256, 0, s>>>(v, atav, cv, alpha, gamma, shift, w,
                                                             count);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_scale(const float* in, float sc, float* out, size_t count, cudaStream_t s) {
  scale_kernel<<<grid_for(count, 256), 256, 0, s>>>(in, sc, out, count);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_cg_update(double* x, double* r, const double* p, const float* ap, double a,
                      size_t count, double* out, cudaStream_t s) {
  cg_update_kernel<<<dot_pair_blocks(), 256, 0, s>>>(x, r, p, ap, a, count, out);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_cg_direction(double* p, const double* r, double beta, float* p32, size_t count,
                         cudaStream_t s) {
  cg_direction_kernel<<<grid_for(count, 256), 256, 0, s>>>(p, r, beta, p32, count);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_cg_dot(const double* p, const float* ap, size_t count, double* out, cudaStream_t s) {
  cg_dot_kernel<<<dot_pair_blocks(), 256, 0, s>>>(p, ap, count, out);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_x_update(float* x, float* x_old, const double* d, double inv_alpha, size_t count,
                     int* flag, cudaStream_t s) {
  x_update_kernel<<<grid_for(count, 256), 256, 0, s>>>(x, x_old, d, inv_alpha, count, flag);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_spec_norm(const float2* spec, int n, int batch, double* out, cudaStream_t s) {
  spec_norm_kernel<<<dim3(dot_pair_blocks(), batch), 256, 0, s>>>(spec, n, out);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_mask_accumulate(const float2* fv, const float2* fav, const double* cutoff, int batch,
                            size_t total, double2* sum, int* hits, cudaStream_t s) {
  mask_accumulate_kernel<<<grid_for(total, 256), 256, 0, s>>>(fv, fav, cutoff, batch, total, sum,
                                                              hits);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

}  // namespace ncsg
