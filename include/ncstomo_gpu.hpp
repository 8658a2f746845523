// ncstomo_gpu.hpp -- C++20 mirror of the reference's operator/solver API for
// the NCS hot path, implemented over the C ABI in ncsg.h (libncsg.so).
//
// Same names, argument meaning and error behaviour as the reference headers
// (paths relative to /root/reference/proj/include/ncstomo):
//   RadonMap, GradMap, IdentityMap ........ radon.hpp:16-36, grad.hpp:17-28,
//                                           linear_map.hpp:25-35
//   SpectralMask, MaskApplier, pinv_mask,
//   laplacian_mask_2d, radon_mask ......... circulant.hpp:16-66
//   ModelParams, assemble_problem,
//   metric_mask ........................... pipeline.hpp:38-71
//   SolverConfig, SolverState, RecordRow,
//   SolveResult, DivergenceError,
//   ncs_step, ncs_solve, pdhg_solve, admm_cg_solve ... solvers.hpp:59-121
// Exceptions: std::invalid_argument for validation failures, DivergenceError
// (a std::runtime_error with .iter) for divergence, std::runtime_error for
// device failures (there is no CPU fallback).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <memory>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ncsg.h"

namespace ncstomo_gpu {

namespace detail {
inline void check(ncsg_status st) {
  if (st == NCSG_OK) return;
  std::string msg = ncsg_last_error();
  if (st == NCSG_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

inline int default_detector_count(int n) { return ncsg_default_detector_count(n); }

/// Matrix-free operator with exact adjoint (linear_map.hpp:13-20).
class LinearMap {
 public:
  virtual ~LinearMap() = default;
  virtual std::size_t domain_size() const = 0;
  virtual std::size_t range_size() const = 0;
  virtual void forward(std::span<const double> x, std::span<double> out) const = 0;
  virtual void adjoint(std::span<const double> u, std::span<double> out) const = 0;
};

class ProjectionMap : public LinearMap {
 public:
  virtual int n_angles() const = 0;
  virtual int n_detectors() const = 0;
};

/// Ray-driven parallel-beam projector (radon.hpp:16-36) on the GPU.
class RadonMap final : public ProjectionMap {
 public:
  RadonMap(int n, int n_angles, int n_det, int device = 0)
      : n_(n), n_angles_(n_angles), n_det_(n_det) {
    ncsg_radon* h = nullptr;
    detail::check(ncsg_radon_create(n, n_angles, n_det, device, &h));
    h_.reset(h, [](ncsg_radon* p) { ncsg_radon_destroy(p); });
  }
  std::size_t domain_size() const override { return static_cast<std::size_t>(n_) * n_; }
  std::size_t range_size() const override {
    return static_cast<std::size_t>(n_angles_) * n_det_;
  }
  void forward(std::span<const double> x, std::span<double> out) const override {
    if (x.size() != domain_size() || out.size() != range_size())
      throw std::invalid_argument("RadonMap::forward size mismatch");
    detail::check(ncsg_radon_forward_host(h_.get(), x.data(), out.data(), 1));
  }
  void adjoint(std::span<const double> u, std::span<double> out) const override {
    if (u.size() != range_size() || out.size() != domain_size())
      throw std::invalid_argument("RadonMap::adjoint size mismatch");
    detail::check(ncsg_radon_adjoint_host(h_.get(), u.data(), out.data(), 1));
  }
  int n_angles() const override { return n_angles_; }
  int n_detectors() const override { return n_det_; }
  int n() const { return n_; }
  /// Valid bilinear samples per application (the reference's sum of R(1)).
  std::int64_t sample_count() const { return ncsg_radon_sample_count(h_.get()); }
  const ncsg_radon* handle() const { return h_.get(); }

 private:
  int n_, n_angles_, n_det_;
  std::shared_ptr<ncsg_radon> h_;
};

/// Explicit sparse projector (sparse.hpp:21-43) on the GPU: CSR rows over
/// sinogram bins plus the stored transpose for the adjoint.
class SparseMap final : public ProjectionMap {
 public:
  SparseMap(int n_image, int n_angles, int n_det, const std::vector<std::int64_t>& rows,
            const std::vector<std::int64_t>& cols, const std::vector<double>& vals,
            int device = 0)
      : n_(n_image), n_angles_(n_angles), n_det_(n_det) {
    if (rows.size() != cols.size() || rows.size() != vals.size())
      throw std::invalid_argument("sparse triplet arrays differ in length");
    ncsg_sparse* h = nullptr;
    detail::check(ncsg_sparse_create(n_image, n_angles, n_det,
                                     static_cast<std::int64_t>(rows.size()), rows.data(),
                                     cols.data(), vals.data(), device, &h));
    h_.reset(h, [](ncsg_sparse* q) { ncsg_sparse_destroy(q); });
  }
  SparseMap(std::shared_ptr<ncsg_sparse> h, int n, int n_angles, int n_det)
      : n_(n), n_angles_(n_angles), n_det_(n_det), h_(std::move(h)) {}
  std::size_t domain_size() const override { return static_cast<std::size_t>(n_) * n_; }
  std::size_t range_size() const override {
    return static_cast<std::size_t>(n_angles_) * n_det_;
  }
  void forward(std::span<const double> x, std::span<double> out) const override {
    if (x.size() != domain_size() || out.size() != range_size())
      throw std::invalid_argument("SparseMap::forward size mismatch");
    detail::check(ncsg_sparse_forward_host(h_.get(), x.data(), out.data(), 1));
  }
  void adjoint(std::span<const double> u, std::span<double> out) const override {
    if (u.size() != range_size() || out.size() != domain_size())
      throw std::invalid_argument("SparseMap::adjoint size mismatch");
    detail::check(ncsg_sparse_adjoint_host(h_.get(), u.data(), out.data(), 1));
  }
  int n_angles() const override { return n_angles_; }
  int n_detectors() const override { return n_det_; }
  int n() const { return n_; }
  std::int64_t nnz() const { return ncsg_sparse_nnz(h_.get()); }
  const std::shared_ptr<ncsg_sparse>& handle() const { return h_; }

 private:
  int n_, n_angles_, n_det_;
  std::shared_ptr<ncsg_sparse> h_;
};

/// FanBeamGeometry (fanbeam.hpp:8-19).
struct FanBeamGeometry {
  int n_views = 0;
  int n_rays = 0;
  double source_radius = 0.0;
  double fan_angle = 0.0;
  static FanBeamGeometry defaults(int n, int n_views, int n_rays) {
    FanBeamGeometry g;
    g.n_views = n_views;
    g.n_rays = n_rays;
    detail::check(ncsg_fan_defaults(n, &g.source_radius, &g.fan_angle));
    return g;
  }
};

/// build_fanbeam (fanbeam.cpp:43-111): the Siddon system matrix as a SparseMap.
inline SparseMap build_fanbeam(int n, const FanBeamGeometry& g, int device = 0) {
  ncsg_sparse* h = nullptr;
  detail::check(
      ncsg_fanbeam_create(n, g.n_views, g.n_rays, g.source_radius, g.fan_angle, device, &h));
  return SparseMap(std::shared_ptr<ncsg_sparse>(h, [](ncsg_sparse* q) { ncsg_sparse_destroy(q); }),
                   n, g.n_views, g.n_rays);
}

/// Forward differences with Neumann boundaries (grad.hpp:17-28).
class GradMap final : public LinearMap {
 public:
  explicit GradMap(int n) : n_(n) {
    if (n < 2) throw std::invalid_argument("grad needs N >= 2");
  }
  std::size_t domain_size() const override { return static_cast<std::size_t>(n_) * n_; }
  std::size_t range_size() const override { return 2 * static_cast<std::size_t>(n_) * (n_ - 1); }
  void forward(std::span<const double> x, std::span<double> out) const override {
    detail::check(ncsg_grad_forward_host(n_, x.data(), out.data(), 1));
  }
  void adjoint(std::span<const double> u, std::span<double> out) const override {
    detail::check(ncsg_grad_adjoint_host(n_, u.data(), out.data(), 1));
  }
  int n() const { return n_; }

 private:
  int n_;
};

/// Eigenvalue grid of a block-circulant operator (circulant.hpp:16-25).
struct SpectralMask {
  int n = 0;
  std::vector<std::complex<double>> h;
  SpectralMask() = default;
  explicit SpectralMask(int n_) : n(n_), h(static_cast<std::size_t>(n_) * n_, 0.0) {}
  std::complex<double>& at(int j, int k) { return h[static_cast<std::size_t>(j) * n + k]; }
  std::complex<double> at(int j, int k) const { return h[static_cast<std::size_t>(j) * n + k]; }
};

inline SpectralMask operator+(const SpectralMask& a, const SpectralMask& b) {
  if (a.n != b.n) throw std::invalid_argument("mask size mismatch");
  SpectralMask out(a.n);
  for (std::size_t i = 0; i < out.h.size(); ++i) out.h[i] = a.h[i] + b.h[i];
  return out;
}
inline SpectralMask operator*(double c, const SpectralMask& m) {
  SpectralMask out(m.n);
  for (std::size_t i = 0; i < out.h.size(); ++i) out.h[i] = c * m.h[i];
  return out;
}

/// laplacian_mask_2d (circulant.cpp:57-68).
inline SpectralMask laplacian_mask_2d(int n) {
  if (n < 1) throw std::invalid_argument("mask size must be positive");
  SpectralMask out(n);
  std::vector<double> s2(n);
  for (int j = 0; j < n; ++j) {
    double s = std::sin(3.14159265358979323846 * j / n);
    s2[j] = s * s;
  }
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) out.at(j, k) = 4.0 * (s2[j] + s2[k]);
  return out;
}

/// radon_mask (circulant.cpp:70-84).
inline SpectralMask radon_mask(int n, double scale, double dc_value) {
  if (n < 1) throw std::invalid_argument("mask size must be positive");
  if (dc_value < 0.0) throw std::invalid_argument("dc_value must be nonnegative");
  SpectralMask out(n);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      double mj = std::min(j, n - j), mk = std::min(k, n - k);
      out.at(j, k) = (j == 0 && k == 0) ? dc_value : scale / std::sqrt(mj * mj + mk * mk);
    }
  return out;
}

/// pinv_mask (circulant.cpp:47-55).
inline SpectralMask pinv_mask(const SpectralMask& mask, double rel_tol = 1e-12) {
  double hmax = 0.0;
  for (const auto& z : mask.h) hmax = std::max(hmax, std::abs(z));
  SpectralMask out(mask.n);
  for (std::size_t i = 0; i < mask.h.size(); ++i)
    out.h[i] = std::abs(mask.h[i]) > rel_tol * hmax ? 1.0 / mask.h[i] : 0.0;
  return out;
}

/// Reusable FFT workspace (circulant.hpp:31-42): out = Re(F^-1 (h .* F x)).
class MaskApplier {
 public:
  explicit MaskApplier(int n, int device = 0) : n_(n), device_(device) {}
  void apply(const SpectralMask& mask, std::span<const double> x, std::span<double> out) const {
    if (mask.n != n_) throw std::invalid_argument("mask size mismatch");
    std::size_t nn = static_cast<std::size_t>(n_) * n_;
    if (x.size() != nn || out.size() != nn) throw std::invalid_argument("image size mismatch");
    detail::check(ncsg_mask_apply_host(n_, reinterpret_cast<const double*>(mask.h.data()),
                                       x.data(), out.data(), 1, device_));
  }

 private:
  int n_, device_;
};

/// ModelParams (pipeline.hpp:38-47), CT defaults.
struct ModelParams {
  std::string model = "ct";
  double alpha = 1e-2;
  double beta = 1e-2;
  double gamma = 1.0;
  double lambda = 1.0;
  double dc = 1e-1;
  bool positivity = false;
};

/// default_model_params (pipeline.cpp:54-67).
inline ModelParams default_model_params(const std::string& model) {
  ModelParams p;
  p.model = model;
  if (model == "ct") return p;
  if (model == "pet") {
    p.alpha = 1e-3;
    p.beta = 1e-3;
    p.gamma = 1e-4;
    p.lambda = 1e-3;
    p.dc = 1e-2;
    return p;
  }
  throw std::invalid_argument("unknown model \"" + model + "\"");
}

/// calibrate_scale(NormalMap(geometry), radon_mask(n, 1, 1), n_samples, seed)
/// (circulant.cpp:142-169), computed on the GPU.
inline double calibrate_scale(const RadonMap& geometry, int n_samples, std::uint64_t seed) {
  double scale = 0.0;
  detail::check(ncsg_calibrate_scale(geometry.handle(), n_samples, seed, &scale));
  return scale;
}

/// <1, R^T R 1> / N^2, the dc value the configs pin for radon_mask.
inline double dc_response(const RadonMap& geometry) {
  double dc = 0.0;
  detail::check(ncsg_radon_dc_response(geometry.handle(), &dc));
  return dc;
}

/// measurement_mask for parallel-beam geometry (pipeline.cpp:100-110).
inline SpectralMask measurement_mask(const RadonMap& geometry, double dc, int samples,
                                     std::uint64_t seed) {
  if (samples < 1) throw std::invalid_argument("mask estimation needs samples >= 1");
  return radon_mask(geometry.n(), calibrate_scale(geometry, samples, seed), dc);
}

/// measurement_mask for a non-parallel geometry (pipeline.cpp:100-110):
/// empirical_mask(NormalMap(geometry), n, samples, seed).mask
/// (circulant.cpp:98-140); `dc` is unused there, as in the reference.
inline SpectralMask measurement_mask(const SparseMap& geometry, double /*dc*/, int samples,
                                     std::uint64_t seed) {
  if (samples < 1) throw std::invalid_argument("mask estimation needs samples >= 1");
  SpectralMask m(geometry.n());
  detail::check(ncsg_sparse_empirical_mask(geometry.handle().get(), samples, seed,
                                           reinterpret_cast<double*>(m.h.data()), nullptr));
  return m;
}

/// metric_mask (pipeline.cpp:112-118).
inline SpectralMask metric_mask(const SpectralMask& measurement, const ModelParams& p) {
  double w = p.beta / p.alpha;
  SpectralMask mask = measurement + (w * w) * laplacian_mask_2d(measurement.n);
  if (p.positivity)
    for (auto& h : mask.h) h += 1.0;
  return mask;
}

/// The two SplitProblem shapes of the hot path: CT-TV as assemble_problem
/// builds it (pipeline.cpp:84-97) and TV denoising {I, D} (the SplitProblem of
/// test_solvers.cpp:646-664).
struct SplitProblem {
  ncsg_kind kind = NCSG_CT;
  int n = 0, n_angles = 0, n_det = 0;
  double alpha = 1.0, beta = 1.0, lambda = 1.0;
  bool positivity = false;
  std::vector<double> offset;  // b (sinogram or noisy image; PET: counts)
  std::shared_ptr<ncsg_sparse> sparse;  // SparseMap geometry (fan beam), else RadonMap
  std::size_t domain_size() const { return static_cast<std::size_t>(n) * n; }
  std::size_t range_size() const {
    std::size_t nn = domain_size();
    std::size_t m = kind != NCSG_DENOISE ? static_cast<std::size_t>(n_angles) * n_det : nn;
    return m + 2 * static_cast<std::size_t>(n) * (n - 1) + (positivity ? nn : 0);
  }
};

namespace detail {
inline SplitProblem assemble_problem_common(std::span<const double> sino, int n, int n_angles,
                                            int n_det, std::size_t range, const ModelParams& p) {
  if (p.model != "ct" && p.model != "pet")
    throw std::invalid_argument("unknown model \"" + p.model + "\"");
  if (p.alpha <= 0.0 || p.beta <= 0.0)
    throw std::invalid_argument("alpha and beta must be positive");
  if (p.lambda < 0.0) throw std::invalid_argument("lambda must be nonnegative");
  if (range != sino.size())
    throw std::invalid_argument("sinogram shape does not match the geometry");
  SplitProblem s;
  // ct: {1, A, QuadraticConj, sino}; pet: {1, A, PoissonConj(sino, alpha), 0}
  // (pipeline.cpp:84-89) -- the counts travel in the offset slot
  s.kind = p.model == "pet" ? NCSG_PET : NCSG_CT;
  if (s.kind == NCSG_PET)
    for (double c : sino)
      if (c < 0.0) throw std::invalid_argument("Poisson counts must be nonnegative");
  s.n = n;
  s.n_angles = n_angles;
  s.n_det = n_det;
  s.alpha = p.alpha;
  s.beta = p.beta;
  s.lambda = p.lambda;
  s.positivity = p.positivity;
  s.offset.assign(sino.begin(), sino.end());
  return s;
}
}  // namespace detail

/// assemble_problem (pipeline.cpp:69-98) on the parallel-beam RadonMap.
inline SplitProblem assemble_problem(std::span<const double> sino, const RadonMap& geometry,
                                     const ModelParams& p) {
  return detail::assemble_problem_common(sino, geometry.n(), geometry.n_angles(),
                                         geometry.n_detectors(), geometry.range_size(), p);
}

/// assemble_problem on a SparseMap geometry (fan beam): same blocks as for
/// RadonMap (pipeline.cpp:69-98), the data block projecting with the matrix.
inline SplitProblem assemble_problem(std::span<const double> sino, const SparseMap& geometry,
                                     const ModelParams& p) {
  SplitProblem s = detail::assemble_problem_common(sino, geometry.n(), geometry.n_angles(),
                                           geometry.n_detectors(), geometry.range_size(), p);
  s.sparse = geometry.handle();
  return s;
}

inline SplitProblem denoise_problem(std::span<const double> noisy, int n, const ModelParams& p) {
  if (noisy.size() != static_cast<std::size_t>(n) * n)
    throw std::invalid_argument("image size mismatch");
  SplitProblem s;
  s.kind = NCSG_DENOISE;
  s.n = n;
  s.alpha = p.alpha;
  s.beta = p.beta;
  s.lambda = p.lambda;
  s.positivity = p.positivity;
  s.offset.assign(noisy.begin(), noisy.end());
  return s;
}

/// SolverConfig (solvers.hpp:59-72).
struct SolverConfig {
  double alpha = 1.0;
  double gamma = 0.0;
  std::optional<SpectralMask> mask;
  int max_iters = 100;
  int record_every = 1;
  double pinv_rel_tol = 1e-12;
  std::uint64_t seed = 0;
  /// Power-method screen of M >= alpha A^T A at solve start (solvers.hpp:67-69);
  /// a violation becomes a warning in the record, as in the reference.
  bool check_step_condition = true;
  int device = 0;
};

struct SolverState {
  int n = 0;
  std::vector<double> x;  // row-major N*N
  std::vector<double> u;  // stacked dual
  std::int64_t iter = 0;
};

inline SolverState make_state(const SplitProblem& prob) {
  SolverState s;
  s.n = prob.n;
  s.x.assign(prob.domain_size(), 0.0);
  s.u.assign(prob.range_size(), 0.0);
  return s;
}

struct RecordRow {
  std::int64_t iter = 0;
  double objective = 0.0, rel_subopt = 0.0, seminorm_step = 0.0, wall_ms = 0.0;
};
struct ConvergenceRecord {
  std::vector<RecordRow> rows;
  std::vector<std::string> warnings;
};
struct SolveResult {
  SolverState state;
  ConvergenceRecord record;
  double objective = 0.0;
};

class DivergenceError : public std::runtime_error {
 public:
  DivergenceError(std::int64_t it, const std::string& what)
      : std::runtime_error(what), iter(it) {}
  std::int64_t iter;
};

namespace detail {

/// Device-resident Engine for one (problem, config) pair.
class Engine {
 public:
  Engine(const SplitProblem& prob, const SolverConfig& cfg, bool pdhg, int n_cg = 0) {
    if (pdhg && cfg.mask) throw std::invalid_argument("pdhg uses M = gamma I; drop the mask");
    if (n_cg > 0 && cfg.mask)
      throw std::invalid_argument("admm_cg uses M = alpha A^T A; drop the mask/overrides");
    if (!(cfg.alpha > 0.0)) throw std::invalid_argument("alpha must be positive");
    if (cfg.mask && cfg.mask->n != prob.n)
      throw std::invalid_argument("mask/problem size mismatch");
    ncsg_problem_desc d{};
    d.kind = prob.kind;
    d.n = prob.n;
    d.n_angles = prob.n_angles;
    d.n_det = prob.n_det;
    d.batch = 1;
    d.positivity = prob.positivity ? 1 : 0;
    // the engine's alpha is the SolverConfig's (solvers.cpp:146-156); the
    // block weight beta/alpha and bound lambda*alpha/beta are the problem's
    d.alpha = cfg.alpha;
    d.beta = prob.beta * cfg.alpha / prob.alpha;
    d.lambda = prob.lambda;
    d.gamma = (n_cg > 0 && !(cfg.gamma > 0.0)) ? 1.0 : cfg.gamma;  // unused by the CG update
    d.pinv_rel_tol = cfg.pinv_rel_tol;
    d.mask = (!pdhg && cfg.mask) ? reinterpret_cast<const double*>(cfg.mask->h.data()) : nullptr;
    d.b = prob.offset.data();
    d.device = cfg.device;
    d.sparse = prob.sparse.get();
    ncsg_problem* h = nullptr;
    check(ncsg_problem_create(&d, &h));
    h_.reset(h, [](ncsg_problem* p) { ncsg_problem_destroy(p); });
    if (n_cg > 0) check(ncsg_set_cg(h, n_cg));
  }
  ncsg_problem* get() const { return h_.get(); }

 private:
  std::shared_ptr<ncsg_problem> h_;
};

inline void throw_divergence() {
  std::string msg = ncsg_last_error();
  std::int64_t it = -1;
  auto pos = msg.find("iteration ");
  if (pos != std::string::npos) it = std::stoll(msg.substr(pos + 10));
  throw DivergenceError(it, msg);
}

inline SolveResult solve(const SplitProblem& prob, const SolverConfig& cfg, bool pdhg,
                         const double* f_star, const SolverState* init, int n_cg = 0) {
  if (cfg.max_iters < 0) throw std::invalid_argument("max_iters must be nonnegative");
  if (cfg.record_every < 1) throw std::invalid_argument("record_every must be >= 1");
  if (n_cg < 0) throw std::invalid_argument("n_cg must be >= 1");
  Engine eng(prob, cfg, pdhg, n_cg);
  SolverState s = init ? *init : make_state(prob);
  check(ncsg_set_state(eng.get(), s.x.data(), s.u.data(), 0));
  int max_rows = cfg.max_iters / cfg.record_every + 3;
  std::vector<ncsg_record_row> rows(max_rows);
  int nr = 0;
  double est = 0.0;
  ncsg_status st = ncsg_solve(eng.get(), cfg.max_iters, cfg.record_every,
                              cfg.check_step_condition ? 1 : 0, cfg.seed, f_star, rows.data(),
                              max_rows, &nr, &est);
  if (st == NCSG_DIVERGED) throw_divergence();
  check(st);
  SolveResult res;
  if (cfg.check_step_condition && n_cg == 0) {  // screen_step_condition (solvers.cpp:207-244)
    double shift = cfg.gamma;
    if (!pdhg && cfg.mask) {
      double hmax = 0.0;
      for (const auto& z : cfg.mask->h) hmax = std::max(hmax, std::abs(z));
      shift = cfg.gamma + cfg.alpha * hmax;
    }
    if (est > 1e-8 * std::max(1.0, shift)) {
      std::ostringstream os;
      os << "step condition M >= alpha A^T A appears violated "
            "(largest eigenvalue of alpha A^T A - M is about " << est << ")";
      res.record.warnings.push_back(os.str());
    }
  }
  res.state = std::move(s);
  check(ncsg_get_state(eng.get(), res.state.x.data(), res.state.u.data(), nullptr));
  res.state.iter = 0;
  for (int i = 0; i < nr; ++i)
    res.record.rows.push_back({rows[i].iter, rows[i].objective, rows[i].rel_subopt,
                               rows[i].seminorm_step, rows[i].wall_ms});
  res.objective = res.record.rows.empty() ? 0.0 : res.record.rows.back().objective;
  return res;
}

}  // namespace detail

/// write_record_csv (io.cpp:203-215): the reference's convergence CSV, same
/// header and %.17g formatting.
inline void write_record_csv(const std::string& path, const ConvergenceRecord& record) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  out << "iter,objective,rel_subopt,seminorm_step,wall_ms\n";
  char buf[256];
  for (const auto& row : record.rows) {
    std::snprintf(buf, sizeof buf, "%lld,%.17g,%.17g,%.17g,%.17g\n",
                  static_cast<long long>(row.iter), row.objective, row.rel_subopt,
                  row.seminorm_step, row.wall_ms);
    out << buf;
  }
  if (!out) throw std::runtime_error("short write to " + path);
}

/// ncs_step (solvers.cpp:417-421): one splitting iteration in place.
inline void ncs_step(SolverState& state, const SplitProblem& prob, const SolverConfig& cfg) {
  detail::Engine eng(prob, cfg, false);
  detail::check(ncsg_set_state(eng.get(), state.x.data(), state.u.data(), state.iter));
  detail::check(ncsg_step(eng.get(), 1));
  std::int64_t div = -1;
  ncsg_status st = ncsg_sync(eng.get(), &div);
  if (st == NCSG_DIVERGED) throw DivergenceError(div, ncsg_last_error());  // absolute
  detail::check(st);
  detail::check(ncsg_get_state(eng.get(), state.x.data(), state.u.data(), nullptr));
  ++state.iter;
}

/// ncs_solve (solvers.cpp:423-426).
inline SolveResult ncs_solve(const SplitProblem& prob, const SolverConfig& cfg,
                             const double* f_star = nullptr, const SolverState* init = nullptr) {
  if (!cfg.mask) throw std::invalid_argument("ncs_solve needs cfg.mask (use pdhg_solve)");
  return detail::solve(prob, cfg, false, f_star, init);
}

/// pdhg_solve (solvers.cpp:428-433): same engine with M = gamma I.
inline SolveResult pdhg_solve(const SplitProblem& prob, const SolverConfig& cfg,
                              const double* f_star = nullptr,
                              const SolverState* init = nullptr) {
  return detail::solve(prob, cfg, true, f_star, init);
}

/// admm_cg_solve (solvers.cpp:435-440): x-update by n_cg conjugate-gradient
/// steps on A^T A (M = alpha A^T A); record iterations count CG steps.
inline SolveResult admm_cg_solve(const SplitProblem& prob, const SolverConfig& cfg, int n_cg,
                                 const double* f_star = nullptr,
                                 const SolverState* init = nullptr) {
  if (cfg.mask) throw std::invalid_argument("admm_cg uses M = alpha A^T A; drop the mask/overrides");
  if (n_cg < 1) throw std::invalid_argument("n_cg must be >= 1");
  return detail::solve(prob, cfg, true, f_star, init, n_cg);
}

}  // namespace ncstomo_gpu
