/* ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * Plain-C fp64 restatement of the reference's NCS hot path (arXiv 1810.13100,
 * `ncstomo`), used by tests/ as the parity checker, by __graft_entry__.smoke()
 * and by bench.py's cpu_baseline leg.  Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).
 *
 * Pinning: tests/test_oracle_pin.py checks this file against the reference's
 * own sources compiled unchanged (oracle/_ref/libncsref.so, see Makefile) --
 * bitwise for the serial paths -- and against the reference tests' known-answer
 * vectors (test_ops.cpp, test_circulant.cpp, test_prox.cpp, test_solvers.cpp).
 *
 * Threading: `nthreads == 1` reproduces the reference's serial summation order
 * exactly.  With more threads the forward projector stays bitwise identical
 * (rays are independent) while the adjoint sums per-thread partial images in a
 * fixed order, so it is deterministic and agrees with the serial order to
 * ~1e-15 relative (SURVEY.md §7 "Oracle runtime").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "fft_core.h"

static const double kPi = 3.14159265358979323846;
static const double kSqrt2 = 1.41421356237309504880;

static void set_threads(int nthreads) {
#ifdef _OPENMP
  omp_set_num_threads(nthreads > 0 ? nthreads : 1);
#else
  (void)nthreads;
#endif
}

/* ---------------------------------------------------------------- rng.cpp */
/* splitmix64_mix (rng.cpp:9-14) */
static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t state;
  double cached;
  int have;
} Rng;

/* RngStream(seed, stream_id) (rng.cpp:16-17) */
static Rng rng_make(uint64_t seed, uint64_t stream) {
  Rng r;
  r.state = mix64(mix64(seed) + stream);
  r.cached = 0.0;
  r.have = 0;
  return r;
}

/* next_u64 (rng.cpp:19-25) */
static uint64_t rng_u64(Rng* r) {
  r->state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = r->state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* next_double (rng.cpp:27-31) */
static double rng_double(Rng* r) {
  uint64_t bits = rng_u64(r) >> 11;
  if (bits == 0) bits = 1;
  return (double)bits * 0x1.0p-53;
}

/* next_normal, Box-Muller with cached pair (rng.cpp:33-45) */
static double rng_normal(Rng* r) {
  if (r->have) {
    r->have = 0;
    return r->cached;
  }
  double u1 = rng_double(r);
  double u2 = rng_double(r);
  double rad = sqrt(-2.0 * log(u1));
  double t = 2.0 * kPi * u2;
  r->cached = rad * sin(t);
  r->have = 1;
  return rad * cos(t);
}

void orc_rng_normals(uint64_t seed, uint64_t stream, int count, double* out) {
  Rng r = rng_make(seed, stream);
  for (int i = 0; i < count; ++i) out[i] = rng_normal(&r);
}

/* -------------------------------------------------------------- radon.cpp */
/* default_detector_count (radon.cpp:10-13) */
int orc_default_detector_count(int n) {
  int d = (int)ceil(kSqrt2 * n + 1.0);
  return d % 2 == 0 ? d + 1 : d;
}

typedef struct {
  double px0, py0, dpx, dpy;
  int count;
} Ray;

/* axis_interval (radon.cpp:22-31) */
static void axis_interval(double a, double b, double lo, double hi, double* t_lo, double* t_hi) {
  if (b == 0.0) {
    if (a >= lo && a <= hi) {
      *t_lo = -1e30;
      *t_hi = 1e30;
    } else {
      *t_lo = 1.0;
      *t_hi = 0.0;
    }
    return;
  }
  double t0 = (lo - a) / b;
  double t1 = (hi - a) / b;
  if (t0 > t1) {
    double t = t0;
    t0 = t1;
    t1 = t;
  }
  *t_lo = t0;
  *t_hi = t1;
}

/* RadonMap::RadonMap geometry checks (radon.cpp:35-42); returns 0 on success. */
int orc_radon_check(int n, int n_angles, int n_det) {
  if (n < 2) return 1;
  if (n_angles < 1) return 2;
  if (n_det % 2 == 0) return 3;
  int min_det = (int)ceil(kSqrt2 * n);
  if (min_det % 2 == 0) ++min_det;
  if (n_det < min_det) return 4;
  return 0;
}

/* Ray table (radon.cpp:43-71). */
static Ray* radon_rays(int n, int n_angles, int n_det) {
  Ray* rays = (Ray*)malloc(sizeof(Ray) * (size_t)n_angles * n_det);
  double c = 0.5 * (n - 1);
  double s_mid = 0.5 * (n_det - 1);
  for (int t = 0; t < n_angles; ++t) {
    double theta = kPi * t / n_angles;
    double ct = cos(theta);
    double st = sin(theta);
    for (int d = 0; d < n_det; ++d) {
      double s = d - s_mid;
      double ixl, ixh, iyl, iyh;
      axis_interval(s * ct + c, -st, 0.0, n - 1, &ixl, &ixh);
      axis_interval(c - s * st, -ct, 0.0, n - 1, &iyl, &iyh);
      double lo = ixl > iyl ? ixl : iyl;
      double hi = ixh < iyh ? ixh : iyh;
      Ray ray = {0.0, 0.0, -st, -ct, 0};
      if (lo <= hi) {
        double k0 = ceil(lo);
        double k1 = floor(hi);
        if (k0 <= k1) {
          ray.px0 = s * ct - k0 * st + c;
          ray.py0 = c - s * st - k0 * ct;
          ray.count = (int)(k1 - k0) + 1;
        }
      }
      rays[(size_t)t * n_det + d] = ray;
    }
  }
  return rays;
}

/* One ray of RadonMap::forward (radon.cpp:85-100). */
static double ray_sum(const Ray* ray, int n, const double* x) {
  double edge = n - 1;
  double acc = 0.0;
  for (int k = 0; k < ray->count; ++k) {
    double px = ray->px0 + k * ray->dpx;
    double py = ray->py0 + k * ray->dpy;
    if (px < 0.0 || px > edge || py < 0.0 || py > edge) continue;
    int ix = (int)px;
    if (ix > n - 2) ix = n - 2;
    int iy = (int)py;
    if (iy > n - 2) iy = n - 2;
    double fx = px - ix;
    double fy = py - iy;
    const double* p = x + (size_t)iy * n + ix;
    acc += (1.0 - fy) * ((1.0 - fx) * p[0] + fx * p[1]) + fy * ((1.0 - fx) * p[n] + fx * p[n + 1]);
  }
  return acc;
}

/* RadonMap::forward (radon.cpp:82-102); rays are independent, so the
 * OpenMP split is bitwise identical to the serial loop. */
int orc_radon_forward(int n, int n_angles, int n_det, const double* x, double* out,
                      int nthreads) {
  if (orc_radon_check(n, n_angles, n_det)) return 2;
  Ray* rays = radon_rays(n, n_angles, n_det);
  long long m = (long long)n_angles * n_det;
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256)
  for (long long r = 0; r < m; ++r) out[r] = ray_sum(&rays[r], n, x);
  free(rays);
  return 0;
}

/* Forward restricted to a subset of rays (for C4-sized spot checks). */
int orc_radon_forward_rays(int n, int n_angles, int n_det, const double* x, int count,
                           const int64_t* ray_idx, double* out, int nthreads) {
  if (orc_radon_check(n, n_angles, n_det)) return 2;
  Ray* rays = radon_rays(n, n_angles, n_det);
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
  for (int i = 0; i < count; ++i) out[i] = ray_sum(&rays[ray_idx[i]], n, x);
  free(rays);
  return 0;
}

/* Scatter of one ray (radon.cpp:108-126). */
static void ray_scatter(const Ray* ray, int n, double w, double* out) {
  double edge = n - 1;
  for (int k = 0; k < ray->count; ++k) {
    double px = ray->px0 + k * ray->dpx;
    double py = ray->py0 + k * ray->dpy;
    if (px < 0.0 || px > edge || py < 0.0 || py > edge) continue;
    int ix = (int)px;
    if (ix > n - 2) ix = n - 2;
    int iy = (int)py;
    if (iy > n - 2) iy = n - 2;
    double fx = px - ix;
    double fy = py - iy;
    double* p = out + (size_t)iy * n + ix;
    p[0] += w * (1.0 - fy) * (1.0 - fx);
    p[1] += w * (1.0 - fy) * fx;
    p[n] += w * fy * (1.0 - fx);
    p[n + 1] += w * fy * fx;
  }
}

/* RadonMap::adjoint (radon.cpp:104-127).  nthreads == 1: exact serial order.
 * Otherwise contiguous ray blocks go to per-thread partial images that are
 * summed in thread order (deterministic, ~1e-15 from the serial order). */
int orc_radon_adjoint(int n, int n_angles, int n_det, const double* u, double* out,
                      int nthreads) {
  if (orc_radon_check(n, n_angles, n_det)) return 2;
  Ray* rays = radon_rays(n, n_angles, n_det);
  size_t nn = (size_t)n * n;
  long long m = (long long)n_angles * n_det;
  memset(out, 0, sizeof(double) * nn);
  if (nthreads <= 1) {
    for (long long r = 0; r < m; ++r) {
      double w = u[r];
      if (w == 0.0) continue;
      ray_scatter(&rays[r], n, w, out);
    }
    free(rays);
    return 0;
  }
  int nt = nthreads;
  double* parts = (double*)calloc(nn * (size_t)nt, sizeof(double));
  set_threads(nt);
#pragma omp parallel num_threads(nt)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    long long lo = m * tid / nt, hi = m * (tid + 1) / nt;
    double* part = parts + nn * (size_t)tid;
    for (long long r = lo; r < hi; ++r) {
      double w = u[r];
      if (w == 0.0) continue;
      ray_scatter(&rays[r], n, w, part);
    }
  }
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)nn; ++i) {
    double acc = 0.0;
    for (int t = 0; t < nt; ++t) acc += parts[nn * (size_t)t + i];
    out[i] = acc;
  }
  free(parts);
  free(rays);
  return 0;
}

/* Number of samples with a valid box check per ray, i.e. R(1) exactly as an
 * integer count (radon.cpp:88-98 with x == 1). */
int orc_radon_valid_counts(int n, int n_angles, int n_det, int32_t* out) {
  if (orc_radon_check(n, n_angles, n_det)) return 2;
  Ray* rays = radon_rays(n, n_angles, n_det);
  long long m = (long long)n_angles * n_det;
  double edge = n - 1;
  for (long long r = 0; r < m; ++r) {
    int c = 0;
    for (int k = 0; k < rays[r].count; ++k) {
      double px = rays[r].px0 + k * rays[r].dpx;
      double py = rays[r].py0 + k * rays[r].dpy;
      if (px < 0.0 || px > edge || py < 0.0 || py > edge) continue;
      ++c;
    }
    out[r] = c;
  }
  free(rays);
  return 0;
}

/* --------------------------------------------------------------- grad.cpp */
/* GradMap::forward (grad.cpp:53-64): h block N x (N-1) then v block (N-1) x N */
void orc_grad_forward(int n, const double* x, double* out) {
  size_t half = (size_t)n * (n - 1);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j + 1 < n; ++j)
      out[(size_t)i * (n - 1) + j] = x[(size_t)i * n + j] - x[(size_t)i * n + j + 1];
  for (int i = 0; i + 1 < n; ++i)
    for (int j = 0; j < n; ++j)
      out[half + (size_t)i * n + j] = x[(size_t)i * n + j] - x[(size_t)(i + 1) * n + j];
}

/* GradMap::adjoint (grad.cpp:66-84) */
void orc_grad_adjoint(int n, const double* u, double* out) {
  size_t half = (size_t)n * (n - 1);
  memset(out, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j + 1 < n; ++j) {
      double w = u[(size_t)i * (n - 1) + j];
      out[(size_t)i * n + j] += w;
      out[(size_t)i * n + j + 1] -= w;
    }
  for (int i = 0; i + 1 < n; ++i)
    for (int j = 0; j < n; ++j) {
      double w = u[half + (size_t)i * n + j];
      out[(size_t)i * n + j] += w;
      out[(size_t)(i + 1) * n + j] -= w;
    }
}

/* ---------------------------------------------------------- circulant.cpp */
/* MaskApplier::apply (circulant.cpp:27-37) via Fft2D (fft.cpp:37-48):
 * out = Re(F^-1 (h .* F x)); the inverse carries the 1/N^2 (fft.cpp:46-47). */
void orc_mask_apply(int n, const double* h, const double* x, double* out) {
  size_t nn = (size_t)n * n;
  double* work = (double*)malloc(sizeof(double) * 2 * nn);
  double* spec = (double*)malloc(sizeof(double) * 2 * nn);
  for (size_t i = 0; i < nn; ++i) {
    work[2 * i] = x[i];
    work[2 * i + 1] = 0.0;
  }
  ncs_fft2d(work, spec, n, n, -1);
  for (size_t i = 0; i < nn; ++i) {
    /* std::complex<double> operator*= (libstdc++ without -ffast-math keeps the
     * textbook formula for finite values) */
    double ar = spec[2 * i], ai = spec[2 * i + 1];
    double br = h[2 * i], bi = h[2 * i + 1];
    spec[2 * i] = ar * br - ai * bi;
    spec[2 * i + 1] = ar * bi + ai * br;
  }
  ncs_fft2d(spec, work, n, n, +1);
  double scale = 1.0 / (double)nn;
  for (size_t i = 0; i < nn; ++i) out[i] = work[2 * i] * scale;
  free(work);
  free(spec);
}

/* pinv_mask (circulant.cpp:47-55) */
void orc_pinv_mask(int n, const double* h, double rel_tol, double* out) {
  size_t nn = (size_t)n * n;
  double hmax = 0.0;
  for (size_t i = 0; i < nn; ++i) {
    double a = hypot(h[2 * i], h[2 * i + 1]);
    if (a > hmax) hmax = a;
  }
  double cutoff = rel_tol * hmax;
  for (size_t i = 0; i < nn; ++i) {
    double re = h[2 * i], im = h[2 * i + 1];
    if (hypot(re, im) > cutoff) {
      if (im == 0.0) {
        out[2 * i] = 1.0 / re;
        out[2 * i + 1] = 0.0;
      } else {
        double d = re * re + im * im;
        out[2 * i] = re / d;
        out[2 * i + 1] = -im / d;
      }
    } else {
      out[2 * i] = 0.0;
      out[2 * i + 1] = 0.0;
    }
  }
}

/* laplacian_mask_2d (circulant.cpp:57-68) */
void orc_laplacian_mask(int n, double* out) {
  double* s2 = (double*)malloc(sizeof(double) * n);
  for (int j = 0; j < n; ++j) {
    double s = sin(kPi * j / n);
    s2[j] = s * s;
  }
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      out[2 * ((size_t)j * n + k)] = 4.0 * (s2[j] + s2[k]);
      out[2 * ((size_t)j * n + k) + 1] = 0.0;
    }
  free(s2);
}

/* radon_mask (circulant.cpp:70-84) */
void orc_radon_mask(int n, double scale, double dc, double* out) {
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      double mj = j < n - j ? j : n - j;
      double mk = k < n - k ? k : n - k;
      double v = (j == 0 && k == 0) ? dc : scale / sqrt(mj * mj + mk * mk);
      out[2 * ((size_t)j * n + k)] = v;
      out[2 * ((size_t)j * n + k) + 1] = 0.0;
    }
}

/* calibrate_scale(NormalMap(R), radon_mask(N,1,1), samples, seed)
 * (circulant.cpp:142-169, probes circulant.cpp:89-94, pipeline.cpp:100-110) */
int orc_calibrate_scale(int n, int n_angles, int n_det, int samples, uint64_t seed,
                        int nthreads, double* result) {
  if (orc_radon_check(n, n_angles, n_det)) return 2;
  size_t nn = (size_t)n * n;
  size_t m = (size_t)n_angles * n_det;
  double* tmpl = (double*)malloc(sizeof(double) * 2 * nn);
  orc_radon_mask(n, 1.0, 1.0, tmpl);
  double* v = (double*)malloc(sizeof(double) * nn);
  double* av = (double*)malloc(sizeof(double) * nn);
  double* mid = (double*)malloc(sizeof(double) * m);
  double* cin = (double*)malloc(sizeof(double) * 2 * nn);
  double* fv = (double*)malloc(sizeof(double) * 2 * nn);
  double* fav = (double*)malloc(sizeof(double) * 2 * nn);
  double num = 0.0, den = 0.0;
  for (int s = 0; s < samples; ++s) {
    Rng r = rng_make(seed, (uint64_t)s);
    for (size_t i = 0; i < nn; ++i) v[i] = rng_normal(&r);
    for (size_t i = 0; i < nn; ++i) {
      cin[2 * i] = v[i];
      cin[2 * i + 1] = 0.0;
    }
    ncs_fft2d(cin, fv, n, n, -1);
    orc_radon_forward(n, n_angles, n_det, v, mid, nthreads);
    orc_radon_adjoint(n, n_angles, n_det, mid, av, nthreads);
    for (size_t i = 0; i < nn; ++i) {
      cin[2 * i] = av[i];
      cin[2 * i + 1] = 0.0;
    }
    ncs_fft2d(cin, fav, n, n, -1);
    for (size_t i = 1; i < nn; ++i) {
      double tr = tmpl[2 * i] * fv[2 * i] - tmpl[2 * i + 1] * fv[2 * i + 1];
      double ti = tmpl[2 * i] * fv[2 * i + 1] + tmpl[2 * i + 1] * fv[2 * i];
      num += tr * fav[2 * i] + ti * fav[2 * i + 1];
      den += tr * tr + ti * ti;
    }
  }
  free(tmpl);
  free(v);
  free(av);
  free(mid);
  free(cin);
  free(fv);
  free(fav);
  if (den == 0.0) return 2;
  *result = num / den;
  return 0;
}

/* ------------------------------------------------------------ phantom.cpp */
/* make_phantom (phantom.cpp:29-51); ellipses: {intensity,x0,y0,a,b,rot_deg} */
int orc_make_phantom(int n, int count, const double* ell, double* out) {
  if (n < 1) return 2;
  for (int e = 0; e < count; ++e)
    if (ell[6 * e + 3] <= 0.0 || ell[6 * e + 4] <= 0.0) return 2;
  memset(out, 0, sizeof(double) * (size_t)n * n);
  for (int e = 0; e < count; ++e) {
    const double* E = ell + 6 * e;
    double phi = E[5] * kPi / 180.0;
    double c = cos(phi), s = sin(phi);
    for (int i = 0; i < n; ++i) {
      double v = (n - 1.0 - 2.0 * i) / n;
      for (int j = 0; j < n; ++j) {
        double u = (2.0 * j - (n - 1.0)) / n;
        double du = u - E[1], dv = v - E[2];
        double xi = (c * du + s * dv) / E[3];
        double eta = (-s * du + c * dv) / E[4];
        if (xi * xi + eta * eta <= 1.0) out[(size_t)i * n + j] += E[0];
      }
    }
  }
  return 0;
}

/* simulate_ct (phantom.cpp:53-63): b_i = (R x)_i + sigma * RngStream(seed,i).normal */
int orc_simulate_ct(int n, int n_angles, int n_det, const double* x, double sigma,
                    uint64_t seed, double* out, int nthreads) {
  if (sigma < 0.0) return 2;
  int rc = orc_radon_forward(n, n_angles, n_det, x, out, nthreads);
  if (rc) return rc;
  size_t m = (size_t)n_angles * n_det;
  for (size_t i = 0; i < m; ++i) {
    Rng r = rng_make(seed, (uint64_t)i);
    out[i] = out[i] + sigma * rng_normal(&r);
  }
  return 0;
}

/* ------------------------------------------------ fan beam (SparseMap) */
/* CSR system matrix with its stored transpose (SparseMap, sparse.cpp:9-45). */
typedef struct {
  int n, views, rays;
  double radius, fan;
  size_t rows, cols, nnz;
  size_t *row_ptr, *col_idx, *t_row_ptr, *t_col_idx;
  double *val, *t_val;
} Csr;

static double g_fan_radius = 0.0, g_fan_angle = 0.0; /* orc_set_fan */
static Csr g_fan_csr = {0};                          /* single-entry cache */

void orc_set_fan(double source_radius, double fan_angle) {
  g_fan_radius = source_radius;
  g_fan_angle = fan_angle;
}

/* FanBeamGeometry::defaults (fanbeam.cpp:10-17) */
void orc_fan_defaults(int n, double* source_radius, double* fan_angle) {
  *source_radius = n;
  *fan_angle = 2.0 * asin(sqrt(2.0) * n / (2.0 * (double)n));
}

/* clip_axis (fanbeam.cpp:27-38) */
static void clip_axis(double s0, double d, double h, double* enter, double* exit_, int* hit) {
  if (d == 0.0) {
    if (s0 < -h || s0 > h) *hit = 0;
    return;
  }
  double t0 = (-h - s0) / d, t1 = (h - s0) / d;
  if (t0 > t1) {
    double t = t0;
    t0 = t1;
    t1 = t;
  }
  if (t0 > *enter) *enter = t0;
  if (t1 < *exit_) *exit_ = t1;
  if (*enter >= *exit_) *hit = 0;
}

/* build_fanbeam (fanbeam.cpp:43-111): Siddon intersection lengths, triplets
 * in ray order; then SparseMap's CSR + counting-sort transpose. */
static int fan_build(int n, int views, int rays, double R, double fan, Csr* A) {
  if (n < 2 || views < 1 || rays < 1) return 2;
  double h = 0.5 * n;
  if (R <= h * sqrt(2.0)) return 2;
  if (fan <= 0.0 || fan >= kPi) return 2;
  size_t cap = (size_t)views * rays * 2 * n + 16, cnt = 0;
  int64_t* tr = (int64_t*)malloc(sizeof(int64_t) * cap);
  int64_t* tc = (int64_t*)malloc(sizeof(int64_t) * cap);
  double* tv = (double*)malloc(sizeof(double) * cap);
  double dpsi = rays > 1 ? fan / (rays - 1) : 0.0;
  double psi0 = -0.5 * fan;
  int64_t ray_index = 0;
  for (int v = 0; v < views; ++v) {
    double phi = 2.0 * kPi * v / views;
    double sx = R * cos(phi), sy = R * sin(phi);
    double cx = -cos(phi), cy = -sin(phi);
    for (int r = 0; r < rays; ++r, ++ray_index) {
      double psi = rays > 1 ? psi0 + r * dpsi : 0.0;
      double cp = cos(psi), sp = sin(psi);
      double dx = cp * cx - sp * cy;
      double dy = sp * cx + cp * cy;
      double enter = 0.0, exit_ = INFINITY;
      int hit = 1;
      clip_axis(sx, dx, h, &enter, &exit_, &hit);
      clip_axis(sy, dy, h, &enter, &exit_, &hit);
      if (!hit) continue;
      double t = enter;
      double px = sx + t * dx, py = sy + t * dy;
      int ix = (int)floor(px + h), iy = (int)floor(py + h);
      ix = ix < 0 ? 0 : (ix > n - 1 ? n - 1 : ix);
      iy = iy < 0 ? 0 : (iy > n - 1 ? n - 1 : iy);
      int step_x = dx > 0.0 ? 1 : -1, step_y = dy > 0.0 ? 1 : -1;
      while (t < exit_ - 1e-12) {
        double tx = dx != 0.0 ? ((ix + (step_x > 0 ? 1 : 0)) - h - sx) / dx : INFINITY;
        double ty = dy != 0.0 ? ((iy + (step_y > 0 ? 1 : 0)) - h - sy) / dy : INFINITY;
        double m = tx < ty ? tx : ty;
        if (exit_ < m) m = exit_;
        double t_next = m > t ? m : t;
        double len = t_next - t;
        if (len > 0.0) {
          if (cnt == cap) {
            cap *= 2;
            tr = (int64_t*)realloc(tr, sizeof(int64_t) * cap);
            tc = (int64_t*)realloc(tc, sizeof(int64_t) * cap);
            tv = (double*)realloc(tv, sizeof(double) * cap);
          }
          tr[cnt] = ray_index;
          tc[cnt] = (int64_t)(n - 1 - iy) * n + ix;
          tv[cnt] = len;
          ++cnt;
        }
        t = t_next;
        if (t >= exit_ - 1e-12) break;
        if (tx <= ty) {
          ix += step_x;
          if (ix < 0 || ix >= n) break;
        } else {
          iy += step_y;
          if (iy < 0 || iy >= n) break;
        }
      }
    }
  }
  A->n = n;
  A->views = views;
  A->rays = rays;
  A->radius = R;
  A->fan = fan;
  A->rows = (size_t)views * rays;
  A->cols = (size_t)n * n;
  A->nnz = cnt;
  /* rows are generated in increasing order, so the stable sort by row is the
   * identity (sparse.cpp:19-20) */
  A->row_ptr = (size_t*)calloc(A->rows + 1, sizeof(size_t));
  A->col_idx = (size_t*)malloc(sizeof(size_t) * (cnt ? cnt : 1));
  A->val = (double*)malloc(sizeof(double) * (cnt ? cnt : 1));
  for (size_t i = 0; i < cnt; ++i) ++A->row_ptr[tr[i] + 1];
  for (size_t r = 0; r < A->rows; ++r) A->row_ptr[r + 1] += A->row_ptr[r];
  for (size_t i = 0; i < cnt; ++i) {
    A->col_idx[i] = (size_t)tc[i];
    A->val[i] = tv[i];
  }
  A->t_row_ptr = (size_t*)calloc(A->cols + 1, sizeof(size_t));
  A->t_col_idx = (size_t*)malloc(sizeof(size_t) * (cnt ? cnt : 1));
  A->t_val = (double*)malloc(sizeof(double) * (cnt ? cnt : 1));
  for (size_t i = 0; i < cnt; ++i) ++A->t_row_ptr[A->col_idx[i] + 1];
  for (size_t c = 0; c < A->cols; ++c) A->t_row_ptr[c + 1] += A->t_row_ptr[c];
  size_t* cursor = (size_t*)malloc(sizeof(size_t) * (A->cols + 1));
  memcpy(cursor, A->t_row_ptr, sizeof(size_t) * A->cols);
  for (size_t r = 0; r < A->rows; ++r)
    for (size_t i = A->row_ptr[r]; i < A->row_ptr[r + 1]; ++i) {
      size_t dst = cursor[A->col_idx[i]]++;
      A->t_col_idx[dst] = r;
      A->t_val[dst] = A->val[i];
    }
  free(cursor);
  free(tr);
  free(tc);
  free(tv);
  return 0;
}

static void csr_free(Csr* A) {
  free(A->row_ptr);
  free(A->col_idx);
  free(A->val);
  free(A->t_row_ptr);
  free(A->t_col_idx);
  free(A->t_val);
  memset(A, 0, sizeof(*A));
}

/* the cached fan-beam matrix for (n, views, rays) and the current orc_set_fan */
static Csr* fan_matrix(int n, int views, int rays) {
  Csr* A = &g_fan_csr;
  if (A->row_ptr && A->n == n && A->views == views && A->rays == rays &&
      A->radius == g_fan_radius && A->fan == g_fan_angle)
    return A;
  csr_free(A);
  if (fan_build(n, views, rays, g_fan_radius, g_fan_angle, A)) return NULL;
  return A;
}

/* SparseMap::forward (sparse.cpp:55-62); rows independent -> OpenMP-exact */
static void csr_forward(const Csr* A, const double* x, double* out, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(static)
  for (long long r = 0; r < (long long)A->rows; ++r) {
    double acc = 0.0;
    for (size_t i = A->row_ptr[r]; i < A->row_ptr[r + 1]; ++i) acc += A->val[i] * x[A->col_idx[i]];
    out[r] = acc;
  }
}

/* SparseMap::adjoint with the stored transpose (sparse.cpp:64-71) */
static void csr_adjoint(const Csr* A, const double* u, double* out, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(static)
  for (long long c = 0; c < (long long)A->cols; ++c) {
    double acc = 0.0;
    for (size_t i = A->t_row_ptr[c]; i < A->t_row_ptr[c + 1]; ++i)
      acc += A->t_val[i] * u[A->t_col_idx[i]];
    out[c] = acc;
  }
}

int orc_fanbeam_triplets(int n, int views, int rays, double R, double fan, int64_t cap,
                         int64_t* nnz, int64_t* row, int64_t* col, double* val) {
  Csr A;
  memset(&A, 0, sizeof(A));
  if (fan_build(n, views, rays, R, fan, &A)) return 2;
  *nnz = (int64_t)A.nnz;
  if (cap >= (int64_t)A.nnz)
    for (size_t r = 0; r < A.rows; ++r)
      for (size_t i = A.row_ptr[r]; i < A.row_ptr[r + 1]; ++i) {
        row[i] = (int64_t)r;
        col[i] = (int64_t)A.col_idx[i];
        val[i] = A.val[i];
      }
  csr_free(&A);
  return 0;
}

/* empirical_mask (circulant.cpp:98-140) of NormalMap(fan-beam SparseMap):
 * per bin the mean of F(A^T A v)/F(v) over the probes whose |F v| clears
 * 1e-12 * ||F v||; dead bins (never cleared) stay 0. */
int orc_fanbeam_empirical_mask(int n, int views, int rays, double R, double fan, int samples,
                               uint64_t seed, int nthreads, double* mask, int* n_dead) {
  Csr A;
  memset(&A, 0, sizeof(A));
  if (samples < 1 || fan_build(n, views, rays, R, fan, &A)) return 2;
  size_t nn = (size_t)n * n;
  double* v = (double*)malloc(sizeof(double) * nn);
  double* av = (double*)malloc(sizeof(double) * nn);
  double* mid = (double*)malloc(sizeof(double) * A.rows);
  double* cin = (double*)malloc(sizeof(double) * 2 * nn);
  double* fv = (double*)malloc(sizeof(double) * 2 * nn);
  double* fav = (double*)malloc(sizeof(double) * 2 * nn);
  double* sum = (double*)calloc(2 * nn, sizeof(double));
  int* hits = (int*)calloc(nn, sizeof(int));
  for (int s = 0; s < samples; ++s) {
    Rng r = rng_make(seed, (uint64_t)s);
    for (size_t i = 0; i < nn; ++i) v[i] = rng_normal(&r);
    for (size_t i = 0; i < nn; ++i) {
      cin[2 * i] = v[i];
      cin[2 * i + 1] = 0.0;
    }
    ncs_fft2d(cin, fv, n, n, -1);
    csr_forward(&A, v, mid, nthreads);
    csr_adjoint(&A, mid, av, nthreads);
    for (size_t i = 0; i < nn; ++i) {
      cin[2 * i] = av[i];
      cin[2 * i + 1] = 0.0;
    }
    ncs_fft2d(cin, fav, n, n, -1);
    double norm = 0.0;
    for (size_t i = 0; i < nn; ++i) norm += fv[2 * i] * fv[2 * i] + fv[2 * i + 1] * fv[2 * i + 1];
    norm = sqrt(norm);
    double cutoff = 1e-12 * norm;
    for (size_t i = 0; i < nn; ++i) {
      double a = fv[2 * i], b = fv[2 * i + 1];
      if (hypot(a, b) < cutoff) continue;
      /* complex division fav / fv as std::complex<double> does (libstdc++) */
      double c = fav[2 * i], d = fav[2 * i + 1];
      double den = a * a + b * b;
      sum[2 * i] += (c * a + d * b) / den;
      sum[2 * i + 1] += (d * a - c * b) / den;
      ++hits[i];
    }
  }
  int dead = 0;
  for (size_t i = 0; i < nn; ++i) {
    if (hits[i] == 0) {
      mask[2 * i] = mask[2 * i + 1] = 0.0;
      ++dead;
      continue;
    }
    mask[2 * i] = sum[2 * i] / (double)hits[i];
    mask[2 * i + 1] = sum[2 * i + 1] / (double)hits[i];
  }
  *n_dead = dead;
  free(v);
  free(av);
  free(mid);
  free(cin);
  free(fv);
  free(fav);
  free(sum);
  free(hits);
  csr_free(&A);
  return 0;
}

int orc_fanbeam_apply(int n, int views, int rays, double R, double fan, int adjoint,
                      const double* in, double* out, int nthreads) {
  Csr A;
  memset(&A, 0, sizeof(A));
  if (fan_build(n, views, rays, R, fan, &A)) return 2;
  if (adjoint)
    csr_adjoint(&A, in, out, nthreads);
  else
    csr_forward(&A, in, out, nthreads);
  csr_free(&A);
  return 0;
}

/* ------------------------------------------------------- solvers.cpp NCS */
/* Problem layouts of the hot path:
 *   kind 0  CT-TV:    blocks {1, R, QuadraticConj, b}, {beta/alpha, D,
 *                     ScaledL1Conj(lambda*alpha/beta)} [+ {1, I, NonnegConj}]
 *                     -- assemble_problem (pipeline.cpp:84-97)
 *   kind 1  denoise:  blocks {1, I, QuadraticConj, b}, {beta/alpha, D, ...}
 *                     [+ {1, I, NonnegConj}] (test_solvers.cpp:646-664).
 *   kind 2  PET-TV:   kind 0 with {1, R, PoissonConj(b, alpha), 0}.
 *   kind 3  fan-beam CT-TV: kind 0 on build_fanbeam's SparseMap (angles =
 *                     views, det = rays; geometry from orc_set_fan). */
typedef struct {
  int kind, n, angles, det, positivity, nthreads;
  double alpha, beta, lambda;
  size_t nn, m0, g, range;
  double w_d, bound;
  const double* b; /* block-0 offset, length m0 */
  const Csr* fanA; /* kind 3 */
} Prob;

static void prob_init(Prob* p, int kind, int n, int angles, int det, double alpha, double beta,
                      double lambda, int positivity, const double* b, int nthreads) {
  p->kind = kind;
  p->n = n;
  p->angles = angles;
  p->det = det;
  p->positivity = positivity;
  p->nthreads = nthreads;
  p->alpha = alpha;
  p->beta = beta;
  p->lambda = lambda;
  p->nn = (size_t)n * n;
  p->m0 = kind != 1 ? (size_t)angles * det : p->nn; /* CT (0) and PET (2) project */
  p->g = 2 * (size_t)n * (n - 1);
  p->range = p->m0 + p->g + (positivity ? p->nn : 0);
  p->w_d = beta / alpha;
  p->bound = lambda * alpha / beta;
  p->b = b;
  p->fanA = kind == 3 ? fan_matrix(n, angles, det) : NULL;
}

/* StackedMap::forward (linear_map.cpp:39-45) */
static void stacked_forward(const Prob* p, const double* x, double* out) {
  if (p->kind == 3)
    csr_forward(p->fanA, x, out, p->nthreads);
  else if (p->kind != 1)
    orc_radon_forward(p->n, p->angles, p->det, x, out, p->nthreads);
  else
    memcpy(out, x, sizeof(double) * p->nn);
  for (size_t i = 0; i < p->m0; ++i) out[i] *= 1.0;
  double* g = out + p->m0;
  orc_grad_forward(p->n, x, g);
  for (size_t i = 0; i < p->g; ++i) g[i] *= p->w_d;
  if (p->positivity) {
    double* q = out + p->m0 + p->g;
    memcpy(q, x, sizeof(double) * p->nn);
    for (size_t i = 0; i < p->nn; ++i) q[i] *= 1.0;
  }
}

/* StackedMap::adjoint (linear_map.cpp:47-55) */
static void stacked_adjoint(const Prob* p, const double* u, double* out, double* tmp) {
  memset(out, 0, sizeof(double) * p->nn);
  if (p->kind == 3)
    csr_adjoint(p->fanA, u, tmp, p->nthreads);
  else if (p->kind != 1)
    orc_radon_adjoint(p->n, p->angles, p->det, u, tmp, p->nthreads);
  else
    memcpy(tmp, u, sizeof(double) * p->nn);
  for (size_t j = 0; j < p->nn; ++j) out[j] += 1.0 * tmp[j];
  orc_grad_adjoint(p->n, u + p->m0, tmp);
  for (size_t j = 0; j < p->nn; ++j) out[j] += p->w_d * tmp[j];
  if (p->positivity) {
    memcpy(tmp, u + p->m0 + p->g, sizeof(double) * p->nn);
    for (size_t j = 0; j < p->nn; ++j) out[j] += 1.0 * tmp[j];
  }
}

/* SplitProblem::objective_from_ax (solvers.cpp:362-381) with
 * QuadraticConj::objective (prox.cpp:26-30), ScaledL1Conj::objective
 * (prox.cpp:40-44), NonnegConj::objective (prox.cpp:107-114). */
static double objective_from_ax(const Prob* p, const double* ax) {
  double total = 0.0;
  double acc = 0.0;
  if (p->kind == 2) {
    /* PoissonConj::objective (prox.cpp:62-74), counts in b */
    for (size_t j = 0; j < p->m0; ++j) {
      double y = ax[j], c = p->b[j];
      if (c > 0.0) {
        if (y <= 0.0) return INFINITY;
        acc += y - c * log(y);
      } else {
        if (y < 0.0) return INFINITY;
        acc += y;
      }
    }
    total += acc;
  } else {
    for (size_t j = 0; j < p->m0; ++j) {
      double z = ax[j] - p->b[j];
      acc += z * z;
    }
    total += 0.5 * acc;
  }
  acc = 0.0;
  const double* g = ax + p->m0;
  for (size_t j = 0; j < p->g; ++j) acc += fabs(g[j]);
  total += p->bound * acc;
  if (isinf(total)) return INFINITY;
  if (p->positivity) {
    const double* q = ax + p->m0 + p->g;
    double hi = 0.0;
    for (size_t j = 0; j < p->nn; ++j)
      if (fabs(q[j]) > hi) hi = fabs(q[j]);
    double tol = 1e-9 * (hi > 1.0 ? hi : 1.0);
    for (size_t j = 0; j < p->nn; ++j)
      if (q[j] < -tol) return INFINITY;
    total += 0.0;
  }
  return total;
}

/* prox evaluate per block (solvers.cpp:151-156; prox.cpp:21-44,103-105) */
/* prox_conj_poisson (prox.cpp:9-13) */
static double prox_conj_poisson(double u, double c) {
  double d = u - 1.0;
  return 1.0 + 0.5 * (d - sqrt(d * d + 4.0 * c));
}

static void prox_all(const Prob* p, double* r) {
  if (p->kind == 2) {
    /* PoissonConj::evaluate (prox.cpp:56-60): c = alpha * counts */
    for (size_t j = 0; j < p->m0; ++j) r[j] = prox_conj_poisson(r[j], p->alpha * p->b[j]);
  } else {
    double s = 1.0 / (1.0 + p->alpha);
    for (size_t j = 0; j < p->m0; ++j) r[j] *= s;
  }
  double* g = r + p->m0;
  double bd = p->bound;
  for (size_t j = 0; j < p->g; ++j) {
    double z = g[j];
    g[j] = z < -bd ? -bd : (z > bd ? bd : z);
  }
  if (p->positivity) {
    double* q = r + p->m0 + p->g;
    for (size_t j = 0; j < p->nn; ++j) q[j] = q[j] < 0.0 ? q[j] : 0.0;
  }
}

typedef struct {
  Prob* p;
  double alpha, gamma;
  int n_cg;           /* > 0: admm_cg x-update (XMode::Cg) */
  const double* mask; /* cfg.mask (nullable) */
  double* m_pinv;     /* pinv(gamma + alpha*mask) */
  double *ax, *ax_new, *r, *atu, *w, *adx, *mdx, *tmp;
} Engine;

/* Engine::Engine mask setup (solvers.cpp:86-116) */
static void engine_init(Engine* e, Prob* p, double alpha, double gamma, const double* mask) {
  e->p = p;
  e->alpha = alpha;
  e->gamma = gamma;
  e->n_cg = 0;
  e->mask = mask;
  e->m_pinv = NULL;
  if (mask) {
    size_t nn = p->nn;
    double* m = (double*)malloc(sizeof(double) * 2 * nn);
    for (size_t i = 0; i < nn; ++i) {
      /* m.h[i] = gamma + alpha * c.h[i] (complex<double> arithmetic) */
      m[2 * i] = gamma + alpha * mask[2 * i];
      m[2 * i + 1] = 0.0 + alpha * mask[2 * i + 1];
    }
    e->m_pinv = (double*)malloc(sizeof(double) * 2 * nn);
    orc_pinv_mask(p->n, m, 1e-12, e->m_pinv);
    free(m);
  }
  e->ax = (double*)calloc(p->range, sizeof(double));
  e->ax_new = (double*)calloc(p->range, sizeof(double));
  e->r = (double*)calloc(p->range, sizeof(double));
  e->adx = (double*)calloc(p->range, sizeof(double));
  e->atu = (double*)calloc(p->nn, sizeof(double));
  e->w = (double*)calloc(p->nn, sizeof(double));
  e->mdx = (double*)calloc(p->nn, sizeof(double));
  e->tmp = (double*)calloc(p->nn, sizeof(double));
}

static void engine_free(Engine* e) {
  free(e->m_pinv);
  free(e->ax);
  free(e->ax_new);
  free(e->r);
  free(e->adx);
  free(e->atu);
  free(e->w);
  free(e->mdx);
  free(e->tmp);
}

/* check_finite (solvers.cpp:248-255): 0 ok, 1 diverged */
static int check_finite(const Prob* p, const double* x, const double* u) {
  for (size_t j = 0; j < p->nn; ++j)
    if (isnan(x[j]) || fabs(x[j]) > 1e150) return 1;
  for (size_t j = 0; j < p->range; ++j)
    if (isnan(u[j])) return 1;
  return 0;
}

static double dotd(const double* a, const double* b, size_t n);

/* cg (solvers.cpp:442-463) on NormalMap(stacked) (linear_map.cpp:57-61):
 * n_iters conjugate-gradient steps from x = 0 for A^T A x = rhs. */
static void cg_normal(Prob* p, const double* rhs, int n_iters, double* x, double* tmp) {
  size_t n = p->nn;
  double* r = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  double* ap = (double*)malloc(sizeof(double) * n);
  double* mid = (double*)malloc(sizeof(double) * p->range);
  memset(x, 0, sizeof(double) * n);
  memcpy(r, rhs, sizeof(double) * n);
  memcpy(q, rhs, sizeof(double) * n);
  double rs = dotd(r, r, n);
  for (int it = 0; it < n_iters; ++it) {
    if (rs == 0.0) break;
    stacked_forward(p, q, mid);
    stacked_adjoint(p, mid, ap, tmp);
    double pap = dotd(q, ap, n);
    if (pap <= 0.0) break;
    double a = rs / pap;
    for (size_t j = 0; j < n; ++j) x[j] += a * q[j];
    for (size_t j = 0; j < n; ++j) r[j] -= a * ap[j];
    double rs_new = dotd(r, r, n);
    double beta = rs_new / rs;
    for (size_t j = 0; j < n; ++j) q[j] = r[j] + beta * q[j];
    rs = rs_new;
  }
  free(r);
  free(q);
  free(ap);
  free(mid);
}

/* Engine::step (solvers.cpp:124-161) in mask (NCS), scaled (PDHG) or Cg
 * (ADMM-CG) mode.  Returns 0 or 1 on divergence.  (u, r swap handled by
 * copying back.) */
static int engine_step(Engine* e, double* x, double* u) {
  Prob* p = e->p;
  stacked_adjoint(p, u, e->atu, e->tmp);
  if (e->n_cg > 0) {
    cg_normal(p, e->atu, e->n_cg, e->w, e->tmp);
    double inv = 1.0 / e->alpha;
    for (size_t j = 0; j < p->nn; ++j) e->w[j] = inv * e->w[j];
  } else if (e->m_pinv) {
    orc_mask_apply(p->n, e->m_pinv, e->atu, e->w);
  } else {
    double inv = 1.0 / e->gamma;
    for (size_t j = 0; j < p->nn; ++j) e->w[j] = inv * e->atu[j];
  }
  for (size_t j = 0; j < p->nn; ++j) x[j] -= e->w[j];
  stacked_forward(p, x, e->ax_new);
  for (size_t i = 0; i < p->range; ++i) {
    double bi = (i < p->m0 && p->kind != 2) ? p->b[i] : 0.0; /* PET block: offset {} */
    e->r[i] = u[i] + e->alpha * (2.0 * e->ax_new[i] - e->ax[i] - bi);
  }
  prox_all(p, e->r);
  memcpy(u, e->r, sizeof(double) * p->range);
  double* t = e->ax;
  e->ax = e->ax_new;
  e->ax_new = t;
  return check_finite(p, x, u);
}

static double dotd(const double* a, const double* b, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

/* Engine::apply_m (solvers.cpp:179-202) */
static void engine_apply_m(Engine* e, const double* dx, double* out) {
  Prob* p = e->p;
  if (e->mask) {
    orc_mask_apply(p->n, e->mask, dx, out);
    for (size_t j = 0; j < p->nn; ++j) out[j] = e->gamma * dx[j] + e->alpha * out[j];
  } else {
    for (size_t j = 0; j < p->nn; ++j) out[j] = e->gamma * dx[j];
  }
}

/* Engine::step_seminorm + seminorm_from (solvers.cpp:35-50,166-177).
 * Returns NaN when the radicand is negative beyond roundoff (the solve loop
 * turns the reference's exception into a NaN row, solvers.cpp:305-316). */
static double engine_seminorm(Engine* e, const double* dx, const double* du) {
  Prob* p = e->p;
  stacked_forward(p, dx, e->adx);
  double t1 = 0.0;
  for (size_t i = 0; i < p->range; ++i) {
    double d = du[i] - e->alpha * e->adx[i];
    t1 += d * d;
  }
  double a_quad = e->alpha * e->alpha * dotd(e->adx, e->adx, p->range);
  double m_quad;
  if (e->n_cg > 0) {
    m_quad = a_quad; /* M = alpha A^T A (solvers.cpp:174) */
  } else {
    engine_apply_m(e, dx, e->mdx);
    m_quad = e->alpha * dotd(dx, e->mdx, p->nn);
  }
  double rad = t1 + m_quad - a_quad;
  if (rad < 0.0) {
    double mag = t1 + fabs(m_quad) + a_quad;
    if (mag < 1.0) mag = 1.0;
    if (rad < -1e-10 * mag) return NAN;
    rad = 0.0;
  }
  return sqrt(rad);
}

/* power_method (solvers.cpp:465-484) on the shifted screen operator
 * alpha A^T A - M + shift I (solvers.cpp:206-245).  Returns the estimate of
 * lambda_max(alpha A^T A - M) (the quantity the screen compares to zero). */
static double engine_screen(Engine* e, int iters, uint64_t seed) {
  Prob* p = e->p;
  size_t nn = p->nn;
  double shift;
  if (e->mask) {
    double hmax = 0.0;
    for (size_t i = 0; i < nn; ++i) {
      double a = hypot(e->mask[2 * i], e->mask[2 * i + 1]);
      if (a > hmax) hmax = a;
    }
    shift = e->gamma + e->alpha * hmax;
  } else {
    shift = e->gamma;
  }
  double* v = (double*)malloc(sizeof(double) * nn);
  double* w = (double*)malloc(sizeof(double) * nn);
  double* mx = (double*)malloc(sizeof(double) * nn);
  double* mid = (double*)malloc(sizeof(double) * p->range);
  Rng r = rng_make(seed, 0);
  for (size_t j = 0; j < nn; ++j) v[j] = rng_normal(&r);
  double nv = sqrt(dotd(v, v, nn));
  double lambda = 0.0;
  if (nv != 0.0) {
    for (size_t j = 0; j < nn; ++j) v[j] /= nv;
    for (int it = 0; it < iters; ++it) {
      stacked_forward(p, v, mid);
      stacked_adjoint(p, mid, w, e->tmp);
      engine_apply_m(e, v, mx);
      for (size_t j = 0; j < nn; ++j) w[j] = e->alpha * w[j] - mx[j] + shift * v[j];
      lambda = dotd(v, w, nn);
      double nw = sqrt(dotd(w, w, nn));
      if (nw == 0.0) {
        lambda = 0.0;
        break;
      }
      for (size_t j = 0; j < nn; ++j) v[j] = w[j] / nw;
    }
  }
  free(v);
  free(w);
  free(mx);
  free(mid);
  return lambda - shift;
}

int orc_screen(int kind, int n, int angles, int det, double alpha, double beta, double lambda,
               int positivity, const double* b, double gamma, const double* mask, int iters,
               uint64_t seed, int nthreads, double* est) {
  Prob p;
  prob_init(&p, kind, n, angles, det, alpha, beta, lambda, positivity, b, nthreads);
  Engine e;
  engine_init(&e, &p, alpha, gamma, mask);
  *est = engine_screen(&e, iters, seed);
  engine_free(&e);
  return 0;
}

/* solve_template (solvers.cpp:267-337) for ncs_solve (mask) / pdhg_solve
 * (mask == NULL).  rows: {iter, objective, rel_subopt, seminorm, wall_ms=0}.
 * Returns 0, 2 (bad input) or 4 (DivergenceError; *div_iter set). */
int orc_solve_ex(int kind, int n, int angles, int det, double alpha, double beta,
                 double lambda, int positivity, const double* b, double gamma,
                 const double* mask, int n_cg, int max_iters, int record_every,
                 const double* x0, const double* u0, double* x_out, double* u_out, double* rows,
                 int max_rows, int* n_rows, double* objective, int64_t* div_iter, int nthreads) {
  if (max_iters < 0 || record_every < 1 || alpha <= 0.0) return 2;
  if (!mask && n_cg <= 0 && gamma <= 0.0) return 2;
  if (n_cg > 0 && mask) return 2; /* admm_cg uses M = alpha A^T A (solvers.cpp:437-438) */
  if ((kind == 0 || kind == 2) && orc_radon_check(n, angles, det)) return 2;
  if (kind == 3 && !fan_matrix(n, angles, det)) return 2;
  Prob p;
  prob_init(&p, kind, n, angles, det, alpha, beta, lambda, positivity, b, nthreads);
  Engine e;
  engine_init(&e, &p, alpha, gamma, mask);
  e.n_cg = n_cg;
  const int64_t axis_scale = n_cg > 0 ? n_cg : 1; /* solvers.cpp:279 */
  double* x = x_out;
  double* u = u_out;
  if (x0)
    memcpy(x, x0, sizeof(double) * p.nn);
  else
    memset(x, 0, sizeof(double) * p.nn);
  if (u0)
    memcpy(u, u0, sizeof(double) * p.range);
  else
    memset(u, 0, sizeof(double) * p.range);
  stacked_forward(&p, x, e.ax); /* Engine::init */
  int k_rows = 0;
#define EMIT(K, SEM)                                          \
  do {                                                        \
    if (k_rows < max_rows) {                                  \
      double* o = rows + 5 * k_rows;                          \
      o[0] = (double)((K) * axis_scale);                      \
      o[1] = objective_from_ax(&p, e.ax);                     \
      o[2] = 0.0;                                             \
      o[3] = (SEM);                                           \
      o[4] = 0.0;                                             \
      ++k_rows;                                               \
    }                                                         \
  } while (0)
  EMIT(0, 0.0);
  double* x_prev = (double*)malloc(sizeof(double) * p.nn);
  double* u_prev = (double*)malloc(sizeof(double) * p.range);
  double* dx = (double*)malloc(sizeof(double) * p.nn);
  double* du = (double*)malloc(sizeof(double) * p.range);
  int rc = 0;
  for (int k = 1; k <= max_iters; ++k) {
    int recorded = (k % record_every == 0) || k == max_iters;
    if (recorded) {
      memcpy(x_prev, x, sizeof(double) * p.nn);
      memcpy(u_prev, u, sizeof(double) * p.range);
    }
    if (engine_step(&e, x, u)) {
      if (div_iter) *div_iter = k;
      rc = 4;
      break;
    }
    if (recorded) {
      for (size_t j = 0; j < p.nn; ++j) dx[j] = x[j] - x_prev[j];
      for (size_t i = 0; i < p.range; ++i) du[i] = u[i] - u_prev[i];
      double sem = engine_seminorm(&e, dx, du);
      EMIT(k, sem);
    }
  }
#undef EMIT
  if (rc == 0) {
    double f_ref = INFINITY;
    for (int i = 0; i < k_rows; ++i)
      if (rows[5 * i + 1] < f_ref) f_ref = rows[5 * i + 1];
    for (int i = 0; i < k_rows; ++i) {
      double a = fabs(f_ref) > 1.0 ? fabs(f_ref) : 1.0;
      rows[5 * i + 2] = isfinite(f_ref) ? (rows[5 * i + 1] - f_ref) / a : 0.0;
    }
    *objective = rows[5 * (k_rows - 1) + 1];
  }
  *n_rows = k_rows;
  free(x_prev);
  free(u_prev);
  free(dx);
  free(du);
  engine_free(&e);
  return rc;
}

int orc_solve(int kind, int n, int angles, int det, double alpha, double beta, double lambda,
              int positivity, const double* b, double gamma, const double* mask, int max_iters,
              int record_every, const double* x0, const double* u0, double* x_out,
              double* u_out, double* rows, int max_rows, int* n_rows, double* objective,
              int64_t* div_iter, int nthreads) {
  return orc_solve_ex(kind, n, angles, det, alpha, beta, lambda, positivity, b, gamma, mask, 0,
                      max_iters, record_every, x0, u0, x_out, u_out, rows, max_rows, n_rows,
                      objective, div_iter, nthreads);
}

/* ncs_step (solvers.cpp:417-421): fresh Engine + init + one step, `steps` times. */
int orc_ncs_step(int kind, int n, int angles, int det, double alpha, double beta,
                 double lambda, int positivity, const double* b, double gamma,
                 const double* mask, double* x, double* u, int steps, int nthreads) {
  Prob p;
  prob_init(&p, kind, n, angles, det, alpha, beta, lambda, positivity, b, nthreads);
  for (int k = 0; k < steps; ++k) {
    Engine e;
    engine_init(&e, &p, alpha, gamma, mask);
    stacked_forward(&p, x, e.ax);
    int rc = engine_step(&e, x, u);
    engine_free(&e);
    if (rc) return 4;
  }
  return 0;
}

/* SplitProblem::objective (solvers.cpp:383-387) */
int orc_objective(int kind, int n, int angles, int det, double alpha, double beta,
                  double lambda, int positivity, const double* b, const double* x,
                  int nthreads, double* f) {
  Prob p;
  prob_init(&p, kind, n, angles, det, alpha, beta, lambda, positivity, b, nthreads);
  double* ax = (double*)malloc(sizeof(double) * p.range);
  stacked_forward(&p, x, ax);
  *f = objective_from_ax(&p, ax);
  free(ax);
  return 0;
}

/* Stacked forward / adjoint of the problem (for per-operator parity). */
int orc_stacked_forward(int kind, int n, int angles, int det, double alpha, double beta,
                        int positivity, const double* x, double* out, int nthreads) {
  Prob p;
  prob_init(&p, kind, n, angles, det, alpha, beta, 1.0, positivity, NULL, nthreads);
  stacked_forward(&p, x, out);
  return 0;
}

int orc_stacked_adjoint(int kind, int n, int angles, int det, double alpha, double beta,
                        int positivity, const double* u, double* out, int nthreads) {
  Prob p;
  prob_init(&p, kind, n, angles, det, alpha, beta, 1.0, positivity, NULL, nthreads);
  double* tmp = (double*)malloc(sizeof(double) * p.nn);
  stacked_adjoint(&p, u, out, tmp);
  free(tmp);
  return 0;
}
