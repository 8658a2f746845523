// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// extern "C" harness around the *reference's own* ncstomo sources, compiled
// unchanged from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libncsref.so.  Python tests and golden-vector generation
// (oracle/gen_golden.py) call it through ctypes; bench.py --impl reference
// times its ncs_solve.  Nothing here re-implements the algorithm: every entry
// forwards to the reference symbol named in its comment.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "ncstomo/circulant.hpp"
#include "ncstomo/fanbeam.hpp"
#include "ncstomo/grad.hpp"
#include "ncstomo/linear_map.hpp"
#include "ncstomo/phantom.hpp"
#include "ncstomo/pipeline.hpp"
#include "ncstomo/prox.hpp"
#include "ncstomo/radon.hpp"
#include "ncstomo/rng.hpp"
#include "ncstomo/solvers.hpp"
#include "ncstomo/sparse.hpp"

using namespace ncstomo;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

SpectralMask mask_from(int n, const double* h) {
  SpectralMask m(n);
  for (std::size_t i = 0; i < m.h.size(); ++i) m.h[i] = {h[2 * i], h[2 * i + 1]};
  return m;
}

void mask_to(const SpectralMask& m, double* out) {
  for (std::size_t i = 0; i < m.h.size(); ++i) {
    out[2 * i] = m.h[i].real();
    out[2 * i + 1] = m.h[i].imag();
  }
}

// Problem kinds of the hot path: 0 = CT-TV via
// assemble_problem (pipeline.cpp:69-98), 1 = TV denoise A=[I;D] built with
// the SplitProblem API as test_solvers.cpp:646-664 does.
struct Desc {
  int kind, n, angles, det;
  double alpha, beta, lambda;
  int positivity;
};

// Fan-beam geometry used by kind 3 (fan-beam CT-TV through SparseMap): set by
// ref_set_fan before building problems (test infrastructure, not thread-safe).
FanBeamGeometry g_fan{};

SplitProblem build_problem(const Desc& d, const double* b) {
  if (d.kind == 3) {  // CT-TV on build_fanbeam's SparseMap (fanbeam.cpp, sparse.cpp)
    FanBeamGeometry g = g_fan;
    g.n_views = d.angles;
    g.n_rays = d.det;
    auto geom = std::make_shared<SparseMap>(build_fanbeam(d.n, g));
    Sinogram s(d.angles, d.det);
    std::memcpy(s.v.data(), b, sizeof(double) * s.v.size());
    ModelParams p;
    p.model = "ct";
    p.alpha = d.alpha;
    p.beta = d.beta;
    p.lambda = d.lambda;
    p.positivity = d.positivity != 0;
    return assemble_problem(s, geom, p);
  }
  if (d.kind == 0 || d.kind == 2) {  // CT-TV or PET-TV (assemble_problem, pipeline.cpp:69-98)
    auto geom = std::make_shared<RadonMap>(d.n, d.angles, d.det);
    Sinogram s(d.angles, d.det);
    std::memcpy(s.v.data(), b, sizeof(double) * s.v.size());
    ModelParams p;
    p.model = d.kind == 2 ? "pet" : "ct";
    p.alpha = d.alpha;
    p.beta = d.beta;
    p.lambda = d.lambda;
    p.positivity = d.positivity != 0;
    return assemble_problem(s, geom, p);
  }
  std::size_t nn = static_cast<std::size_t>(d.n) * d.n;
  std::vector<SplitBlock> blocks;
  blocks.push_back({1.0, std::make_shared<IdentityMap>(nn), std::make_shared<QuadraticConj>(),
                    std::vector<double>(b, b + nn)});
  blocks.push_back({d.beta / d.alpha, std::make_shared<GradMap>(d.n),
                    std::make_shared<ScaledL1Conj>(d.lambda * d.alpha / d.beta),
                    {}});
  if (d.positivity)
    blocks.push_back({1.0, std::make_shared<IdentityMap>(nn), std::make_shared<NonnegConj>(),
                      {}});
  return SplitProblem(d.n, std::move(blocks));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Fan-beam geometry (fanbeam.hpp FanBeamGeometry) for kind 3 problems.
void ref_set_fan(double source_radius, double fan_angle) {
  g_fan.source_radius = source_radius;
  g_fan.fan_angle = fan_angle;
}

// FanBeamGeometry::defaults (fanbeam.cpp:10-17): radius and fan angle.
void ref_fan_defaults(int n, double* source_radius, double* fan_angle) {
  FanBeamGeometry g = FanBeamGeometry::defaults(n, 1, 1);
  *source_radius = g.source_radius;
  *fan_angle = g.fan_angle;
}

// build_fanbeam (fanbeam.cpp:43-111) as CSR-ordered triplets (to_triplets,
// sparse.cpp:73-80).  Call with cap = 0 to get *nnz only.
int ref_fanbeam_triplets(int n, int views, int rays, double source_radius, double fan_angle,
                         int64_t cap, int64_t* nnz, int64_t* row, int64_t* col, double* val) {
  return guard([&] {
    FanBeamGeometry g{views, rays, source_radius, fan_angle};
    SparseMap m = build_fanbeam(n, g);
    auto t = m.to_triplets();
    *nnz = static_cast<int64_t>(t.size());
    if (cap >= static_cast<int64_t>(t.size()))
      for (std::size_t i = 0; i < t.size(); ++i) {
        row[i] = t[i].row;
        col[i] = t[i].col;
        val[i] = t[i].value;
      }
  });
}

// measurement_mask for a non-parallel geometry = empirical_mask(NormalMap(A),
// n, samples, seed).mask (pipeline.cpp:100-110, circulant.cpp:98-140) on the
// fan-beam SparseMap; *n_dead = number of dead bins.
int ref_fanbeam_empirical_mask(int n, int views, int rays, double source_radius,
                               double fan_angle, int samples, uint64_t seed, double* mask_out,
                               int* n_dead) {
  return guard([&] {
    FanBeamGeometry g{views, rays, source_radius, fan_angle};
    auto A = std::make_shared<SparseMap>(build_fanbeam(n, g));
    NormalMap normal(A);
    EmpiricalMask e = empirical_mask(normal, n, samples, seed);
    mask_to(e.mask, mask_out);
    *n_dead = static_cast<int>(e.dead_bins.size());
  });
}

// SparseMap::forward / adjoint (sparse.cpp:55-71) of the fan-beam matrix.
int ref_fanbeam_apply(int n, int views, int rays, double source_radius, double fan_angle,
                      int adjoint, const double* in, double* out) {
  return guard([&] {
    FanBeamGeometry g{views, rays, source_radius, fan_angle};
    SparseMap m = build_fanbeam(n, g);
    if (adjoint)
      m.adjoint({in, m.range_size()}, {out, m.domain_size()});
    else
      m.forward({in, m.domain_size()}, {out, m.range_size()});
  });
}

int ref_default_detector_count(int n) { return default_detector_count(n); }

// RadonMap::forward / adjoint (radon.cpp:82-127)
int ref_radon_forward(int n, int angles, int det, const double* x, double* out) {
  return guard([&] {
    RadonMap m(n, angles, det);
    m.forward({x, m.domain_size()}, {out, m.range_size()});
  });
}
int ref_radon_adjoint(int n, int angles, int det, const double* u, double* out) {
  return guard([&] {
    RadonMap m(n, angles, det);
    m.adjoint({u, m.range_size()}, {out, m.domain_size()});
  });
}

// GradMap::forward / adjoint (grad.cpp:53-84)
int ref_grad_forward(int n, const double* x, double* out) {
  return guard([&] {
    GradMap m(n);
    m.forward({x, m.domain_size()}, {out, m.range_size()});
  });
}
int ref_grad_adjoint(int n, const double* g, double* out) {
  return guard([&] {
    GradMap m(n);
    m.adjoint({g, m.range_size()}, {out, m.domain_size()});
  });
}

// MaskApplier::apply (circulant.cpp:27-37); mask is interleaved complex N*N.
int ref_mask_apply(int n, const double* mask, const double* x, double* out) {
  return guard([&] {
    MaskApplier a(n);
    std::size_t nn = static_cast<std::size_t>(n) * n;
    a.apply(mask_from(n, mask), {x, nn}, {out, nn});
  });
}

int ref_pinv_mask(int n, const double* mask, double rel_tol, double* out) {
  return guard([&] { mask_to(pinv_mask(mask_from(n, mask), rel_tol), out); });
}
int ref_laplacian_mask(int n, double* out) {
  return guard([&] { mask_to(laplacian_mask_2d(n), out); });
}
int ref_radon_mask(int n, double scale, double dc, double* out) {
  return guard([&] { mask_to(radon_mask(n, scale, dc), out); });
}

// calibrate_scale(NormalMap(R), radon_mask(N,1,1), samples, seed) -- the
// inner call of measurement_mask for parallel beam (pipeline.cpp:100-110).
int ref_calibrate_scale(int n, int angles, int det, int samples, uint64_t seed, double* out) {
  return guard([&] {
    auto r = std::make_shared<RadonMap>(n, angles, det);
    NormalMap normal(r);
    *out = calibrate_scale(normal, radon_mask(n, 1.0, 1.0), samples, seed);
  });
}

// measurement_mask + metric_mask (pipeline.cpp:100-118), CT parallel beam.
int ref_ct_metric_mask(int n, int angles, int det, double alpha, double beta, double dc,
                       int samples, uint64_t seed, int positivity, double* out) {
  return guard([&] {
    GeometrySpec spec;
    spec.kind = "parallel";
    spec.image_size = n;
    spec.angles = angles;
    spec.detectors = det;
    RadonMap r(n, angles, det);
    SpectralMask meas = measurement_mask(spec, r, dc, samples, seed);
    ModelParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.positivity = positivity != 0;
    mask_to(metric_mask(meas, p), out);
  });
}

// metric_mask on an explicit measurement mask (pipeline.cpp:112-118).
int ref_metric_mask(int n, const double* meas, double alpha, double beta, int positivity,
                    double* out) {
  return guard([&] {
    ModelParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.positivity = positivity != 0;
    mask_to(metric_mask(mask_from(n, meas), p), out);
  });
}

// make_phantom (phantom.cpp:29-51); ellipses: 6 doubles each
// {intensity, x0, y0, a, b, rot_deg}.
int ref_make_phantom(int n, int count, const double* ell, double* out) {
  return guard([&] {
    PhantomSpec spec;
    spec.n = n;
    for (int i = 0; i < count; ++i) {
      const double* e = ell + 6 * i;
      spec.ellipses.push_back({e[0], e[1], e[2], e[3], e[4], e[5]});
    }
    ImageGrid img = make_phantom(spec);
    std::memcpy(out, img.v.data(), sizeof(double) * img.v.size());
  });
}

// simulate_ct (phantom.cpp:53-63)
int ref_simulate_ct(int n, int angles, int det, const double* x, double sigma, uint64_t seed,
                    double* out) {
  return guard([&] {
    RadonMap r(n, angles, det);
    ImageGrid img(n);
    std::memcpy(img.v.data(), x, sizeof(double) * img.v.size());
    Sinogram s = simulate_ct(img, r, sigma, seed);
    std::memcpy(out, s.v.data(), sizeof(double) * s.v.size());
  });
}

int ref_rng_normals(uint64_t seed, uint64_t stream, int count, double* out) {
  return guard([&] {
    RngStream rng(seed, stream);
    for (int i = 0; i < count; ++i) out[i] = rng.next_normal();
  });
}

int ref_problem_sizes(int kind, int n, int angles, int det, int positivity, int64_t* range) {
  return guard([&] {
    Desc d{kind, n, angles, det, 1.0, 1.0, 1.0, positivity};
    std::size_t m = kind != 1 ? static_cast<std::size_t>(angles) * det
                              : static_cast<std::size_t>(n) * n;
    std::vector<double> b(m, 0.0);
    SplitProblem p = build_problem(d, b.data());
    *range = static_cast<int64_t>(p.range_size());
  });
}

// ncs_solve / pdhg_solve (solvers.cpp:423-432) with optional init state.
// rows: up to max_rows of {iter, objective, rel_subopt, seminorm, wall_ms}.
int ref_solve(int kind, int n, int angles, int det, double alpha, double beta, double lambda,
              int positivity, const double* b, double gamma, const double* mask /*nullable*/,
              int max_iters, int record_every, int check_step, const double* x0 /*nullable*/,
              const double* u0 /*nullable*/, int use_pdhg, double* x_out, double* u_out,
              double* rows, int max_rows, int* n_rows, double* objective) {
  return guard([&] {
    Desc d{kind, n, angles, det, alpha, beta, lambda, positivity};
    SplitProblem prob = build_problem(d, b);
    SolverConfig cfg;
    cfg.alpha = alpha;
    cfg.gamma = gamma;
    if (mask) cfg.mask = mask_from(n, mask);
    cfg.max_iters = max_iters;
    cfg.record_every = record_every;
    cfg.check_step_condition = check_step != 0;
    SolverState init = make_state(prob);
    if (x0) std::memcpy(init.x.v.data(), x0, sizeof(double) * init.x.v.size());
    if (u0) std::memcpy(init.u.data(), u0, sizeof(double) * init.u.size());
    SolveResult res = use_pdhg ? pdhg_solve(prob, cfg, nullptr, &init)
                               : ncs_solve(prob, cfg, nullptr, &init);
    std::memcpy(x_out, res.state.x.v.data(), sizeof(double) * res.state.x.v.size());
    std::memcpy(u_out, res.state.u.data(), sizeof(double) * res.state.u.size());
    int k = 0;
    for (const RecordRow& r : res.record.rows) {
      if (k >= max_rows) break;
      double* o = rows + 5 * k;
      o[0] = static_cast<double>(r.iter);
      o[1] = r.objective;
      o[2] = r.rel_subopt;
      o[3] = r.seminorm_step;
      o[4] = r.wall_ms;
      ++k;
    }
    *n_rows = k;
    *objective = res.objective;
  });
}

// admm_cg_solve (solvers.cpp:435-440): the same engine with the x-update
// w = (1/alpha) CG(A^T A, A^T u, n_cg); no mask.
int ref_admm_cg_solve(int kind, int n, int angles, int det, double alpha, double beta,
                      double lambda, int positivity, const double* b, double gamma, int n_cg,
                      int max_iters, int record_every, double* x_out, double* u_out,
                      double* rows, int max_rows, int* n_rows, double* objective) {
  return guard([&] {
    Desc d{kind, n, angles, det, alpha, beta, lambda, positivity};
    SplitProblem prob = build_problem(d, b);
    SolverConfig cfg;
    cfg.alpha = alpha;
    cfg.gamma = gamma;
    cfg.max_iters = max_iters;
    cfg.record_every = record_every;
    cfg.check_step_condition = false;
    SolveResult res = admm_cg_solve(prob, cfg, n_cg);
    std::memcpy(x_out, res.state.x.v.data(), sizeof(double) * res.state.x.v.size());
    std::memcpy(u_out, res.state.u.data(), sizeof(double) * res.state.u.size());
    int k = 0;
    for (const RecordRow& r : res.record.rows) {
      if (k >= max_rows) break;
      double* o = rows + 5 * k;
      o[0] = static_cast<double>(r.iter);
      o[1] = r.objective;
      o[2] = r.rel_subopt;
      o[3] = r.seminorm_step;
      o[4] = r.wall_ms;
      ++k;
    }
    *n_rows = k;
    *objective = res.objective;
  });
}

// ncs_step (solvers.cpp:417-421): fresh Engine per call, in place on (x, u).
int ref_ncs_step(int kind, int n, int angles, int det, double alpha, double beta, double lambda,
                 int positivity, const double* b, double gamma, const double* mask, double* x,
                 double* u, int steps) {
  return guard([&] {
    Desc d{kind, n, angles, det, alpha, beta, lambda, positivity};
    SplitProblem prob = build_problem(d, b);
    SolverConfig cfg;
    cfg.alpha = alpha;
    cfg.gamma = gamma;
    if (mask) cfg.mask = mask_from(n, mask);
    SolverState s = make_state(prob);
    std::memcpy(s.x.v.data(), x, sizeof(double) * s.x.v.size());
    std::memcpy(s.u.data(), u, sizeof(double) * s.u.size());
    for (int k = 0; k < steps; ++k) ncs_step(s, prob, cfg);
    std::memcpy(x, s.x.v.data(), sizeof(double) * s.x.v.size());
    std::memcpy(u, s.u.data(), sizeof(double) * s.u.size());
  });
}

// SplitProblem::objective (solvers.cpp:383-387)
int ref_objective(int kind, int n, int angles, int det, double alpha, double beta,
                  double lambda, int positivity, const double* b, const double* x, double* f) {
  return guard([&] {
    Desc d{kind, n, angles, det, alpha, beta, lambda, positivity};
    SplitProblem prob = build_problem(d, b);
    *f = prob.objective({x, prob.domain_size()});
  });
}

}  // extern "C"
