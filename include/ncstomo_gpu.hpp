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
//   ImageGrid, Sinogram ................... image.hpp:9-36
//   StackedMap, ProxConj, QuadraticConj,
//   ScaledL1Conj, PoissonConj, NonnegConj . linear_map.hpp:37-61, prox.hpp:9-95
//   SplitBlock, SplitProblem(n, blocks) ... solvers.hpp:17-52 (block lists the
//                                           device engine has kernels for)
//   SolverConfig (incl. m_pinv_override /
//   m_override as CirculantMap), SolverState, RecordRow,
//   SolveResult, DivergenceError,
//   ncs_step, ncs_solve, pdhg_solve, admm_cg_solve ... solvers.hpp:54-121
// Exceptions: std::invalid_argument for validation failures, DivergenceError
// (a std::runtime_error with .iter) for divergence, std::runtime_error for
// device failures (there is no CPU fallback).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
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

/// Square N x N image, row-major doubles (image.hpp:9-20).
struct ImageGrid {
  int n = 0;
  std::vector<double> v;
  ImageGrid() = default;
  explicit ImageGrid(int n_) : n(n_), v(static_cast<std::size_t>(n_) * n_, 0.0) {}
  double& at(int row, int col) { return v[static_cast<std::size_t>(row) * n + col]; }
  double at(int row, int col) const { return v[static_cast<std::size_t>(row) * n + col]; }
  std::size_t size() const { return v.size(); }
};

/// Projection data, angle-major (image.hpp:22-36).
struct Sinogram {
  int n_angles = 0, n_det = 0;
  std::vector<double> v;
  Sinogram() = default;
  Sinogram(int a, int d) : n_angles(a), n_det(d), v(static_cast<std::size_t>(a) * d, 0.0) {}
  double& at(int angle, int det) { return v[static_cast<std::size_t>(angle) * n_det + det]; }
  double at(int angle, int det) const { return v[static_cast<std::size_t>(angle) * n_det + det]; }
  std::size_t size() const { return v.size(); }
};

/// IdentityMap (linear_map.hpp:25-35).  On the device it is the identity
/// block of TV denoising or of the positivity constraint.
class IdentityMap final : public LinearMap {
 public:
  explicit IdentityMap(std::size_t n) : n_(n) {}
  std::size_t domain_size() const override { return n_; }
  std::size_t range_size() const override { return n_; }
  void forward(std::span<const double> x, std::span<double> out) const override {
    std::copy(x.begin(), x.end(), out.begin());
  }
  void adjoint(std::span<const double> u, std::span<double> out) const override {
    std::copy(u.begin(), u.end(), out.begin());
  }

 private:
  std::size_t n_;
};

/// StackedMap (linear_map.hpp:37-61): x -> (w_1 A_1 x, ..., w_m A_m x).
class StackedMap final : public LinearMap {
 public:
  struct Block {
    double weight = 1.0;
    std::shared_ptr<const LinearMap> map;
  };
  explicit StackedMap(std::vector<Block> blocks) : blocks_(std::move(blocks)) {
    if (blocks_.empty()) throw std::invalid_argument("StackedMap needs at least one block");
    domain_ = blocks_.front().map->domain_size();
    for (const auto& b : blocks_) {
      if (b.map->domain_size() != domain_)
        throw std::invalid_argument("StackedMap blocks must share a domain");
      offsets_.push_back(range_);
      range_ += b.map->range_size();
    }
  }
  std::size_t domain_size() const override { return domain_; }
  std::size_t range_size() const override { return range_; }
  std::size_t block_offset(std::size_t i) const { return offsets_.at(i); }
  const std::vector<Block>& blocks() const { return blocks_; }
  void forward(std::span<const double> x, std::span<double> out) const override {
    for (std::size_t i = 0; i < blocks_.size(); ++i) {
      auto seg = out.subspan(offsets_[i], blocks_[i].map->range_size());
      blocks_[i].map->forward(x, seg);
      for (double& s : seg) s *= blocks_[i].weight;
    }
  }
  void adjoint(std::span<const double> u, std::span<double> out) const override {
    std::fill(out.begin(), out.end(), 0.0);
    std::vector<double> tmp(domain_);
    for (std::size_t i = 0; i < blocks_.size(); ++i) {
      blocks_[i].map->adjoint(u.subspan(offsets_[i], blocks_[i].map->range_size()), tmp);
      for (std::size_t j = 0; j < domain_; ++j) out[j] += blocks_[i].weight * tmp[j];
    }
  }

 private:
  std::vector<Block> blocks_;
  std::vector<std::size_t> offsets_;
  std::size_t domain_ = 0, range_ = 0;
};

/// A circulant operator given by its eigenvalue grid: x -> Re(F^-1 (h .* F x))
/// (MaskApplier, circulant.hpp:31-42).  The GPU engine accepts
/// SolverConfig::m_pinv_override / m_override in this form.
class CirculantMap final : public LinearMap {
 public:
  explicit CirculantMap(SpectralMask mask, int device = 0)
      : mask_(std::move(mask)), device_(device) {}
  std::size_t domain_size() const override { return static_cast<std::size_t>(mask_.n) * mask_.n; }
  std::size_t range_size() const override { return domain_size(); }
  void forward(std::span<const double> x, std::span<double> out) const override {
    MaskApplier(mask_.n, device_).apply(mask_, x, out);
  }
  void adjoint(std::span<const double> u, std::span<double> out) const override {
    SpectralMask c(mask_.n);
    for (std::size_t i = 0; i < c.h.size(); ++i) c.h[i] = std::conj(mask_.h[i]);
    MaskApplier(mask_.n, device_).apply(c, u, out);
  }
  const SpectralMask& mask() const { return mask_; }

 private:
  SpectralMask mask_;
  int device_;
};

inline constexpr double kInf = std::numeric_limits<double>::infinity();

/// prox_{alpha g*} for g = 1/2 ||.||^2 and friends (prox.hpp:9-25).
inline double prox_conj_quadratic(double z, double alpha) { return z / (1.0 + alpha); }
inline double project_box(double z, double bound) {
  return z < -bound ? -bound : (z > bound ? bound : z);
}
inline double prox_conj_poisson(double u, double c) {
  if (c < 0.0) throw std::invalid_argument("prox_conj_poisson needs c >= 0");
  double d = u - 1.0;
  return 1.0 + 0.5 * (d - std::sqrt(d * d + 4.0 * c));
}
inline double prox_conj_nonneg(double u) { return u < 0.0 ? u : 0.0; }

/// Dual-block prox plus the matching primal objective term (prox.hpp:30-43).
/// The host evaluate/objective follow prox.cpp; the GPU engine recognises the
/// four concrete types below and runs their device kernels.
class ProxConj {
 public:
  virtual ~ProxConj() = default;
  virtual void evaluate(std::span<double> u, double alpha) const = 0;
  virtual double objective(std::span<const double> y) const = 0;
  virtual std::uint64_t param_hash() const = 0;
};

namespace detail {
inline std::uint64_t fnv1a(const void* data, std::size_t len, std::uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < len; ++i) h = (h ^ p[i]) * 0x100000001b3ULL;
  return h;
}
}  // namespace detail

/// g = 1/2 ||.||^2 (prox.cpp:21-30).
class QuadraticConj final : public ProxConj {
 public:
  void evaluate(std::span<double> u, double alpha) const override {
    double s = 1.0 / (1.0 + alpha);
    for (double& z : u) z *= s;
  }
  double objective(std::span<const double> y) const override {
    double acc = 0.0;
    for (double z : y) acc += z * z;
    return 0.5 * acc;
  }
  std::uint64_t param_hash() const override { return 0x9a0d; }
};

/// g = bound * ||.||_1 (prox.cpp:32-45).
class ScaledL1Conj final : public ProxConj {
 public:
  explicit ScaledL1Conj(double bound) : bound_(bound) {
    if (bound < 0.0) throw std::invalid_argument("l1 weight must be nonnegative");
  }
  void evaluate(std::span<double> u, double) const override {
    for (double& z : u) z = project_box(z, bound_);
  }
  double objective(std::span<const double> y) const override {
    double acc = 0.0;
    for (double z : y) acc += std::abs(z);
    return bound_ * acc;
  }
  std::uint64_t param_hash() const override {
    return detail::fnv1a(&bound_, sizeof bound_, 0x11);
  }
  double bound() const { return bound_; }

 private:
  double bound_;
};

/// Poisson log-likelihood, c = alpha * counts folded in (prox.cpp:47-74).
class PoissonConj final : public ProxConj {
 public:
  PoissonConj(std::vector<double> counts, double alpha) : counts_(std::move(counts)), alpha_(alpha) {
    if (alpha <= 0.0) throw std::invalid_argument("PoissonConj needs alpha > 0");
    for (double c : counts_)
      if (c < 0.0) throw std::invalid_argument("Poisson counts must be nonnegative");
  }
  void evaluate(std::span<double> u, double alpha) const override {
    if (u.size() != counts_.size()) throw std::invalid_argument("PoissonConj size mismatch");
    if (alpha != alpha_) throw std::invalid_argument("PoissonConj built for a different alpha");
    for (std::size_t i = 0; i < u.size(); ++i) u[i] = prox_conj_poisson(u[i], alpha_ * counts_[i]);
  }
  double objective(std::span<const double> y) const override {
    if (y.size() != counts_.size()) throw std::invalid_argument("PoissonConj size mismatch");
    double acc = 0.0;
    for (std::size_t i = 0; i < y.size(); ++i) {
      if (counts_[i] > 0.0) {
        if (y[i] <= 0.0) return kInf;
        acc += y[i] - counts_[i] * std::log(y[i]);
      } else {
        if (y[i] < 0.0) return kInf;
        acc += y[i];
      }
    }
    return acc;
  }
  std::uint64_t param_hash() const override {
    std::uint64_t h = detail::fnv1a(&alpha_, sizeof alpha_, 0x90155);
    return detail::fnv1a(counts_.data(), counts_.size() * sizeof(double), h);
  }
  const std::vector<double>& counts() const { return counts_; }
  double alpha() const { return alpha_; }

 private:
  std::vector<double> counts_;
  double alpha_;
};

/// g = indicator of the nonnegative orthant (prox.cpp:98-113).
class NonnegConj final : public ProxConj {
 public:
  void evaluate(std::span<double> u, double) const override {
    for (double& z : u) z = prox_conj_nonneg(z);
  }
  double objective(std::span<const double> y) const override {
    double hi = 0.0;
    for (double z : y) hi = std::max(hi, std::abs(z));
    double tol = 1e-9 * std::max(1.0, hi);
    for (double z : y)
      if (z < -tol) return kInf;
    return 0.0;
  }
  std::uint64_t param_hash() const override { return 0x20e6; }
};

/// One term of min_x sum_i g_i(w_i A_i x - o_i) (solvers.hpp:17-22).
struct SplitBlock {
  double weight = 1.0;
  std::shared_ptr<const LinearMap> map;
  std::shared_ptr<const ProxConj> prox;
  std::vector<double> offset;
};

/// SplitProblem(n, blocks) (solvers.hpp:24-52, solvers.cpp:341-360): same
/// validation and stacked layout.  The constructor also maps the block list
/// onto the device engine's problem kinds (ncsg.h):
///   {1, RadonMap|SparseMap, QuadraticConj, b}  + {w, GradMap, ScaledL1Conj(B)}  -> CT
///   {1, RadonMap|SparseMap, PoissonConj(c, a)} + {w, GradMap, ScaledL1Conj(B)}  -> PET
///   {1, IdentityMap(N^2), QuadraticConj, b}    + {w, GradMap, ScaledL1Conj(B)}  -> denoise
/// each optionally followed by {1, IdentityMap(N^2), NonnegConj} (positivity)
/// -- the shapes assemble_problem builds (pipeline.cpp:84-97) and the
/// denoising problem of test_solvers.cpp:646-664.  Any other list is valid
/// for the reference but has no device kernel: std::invalid_argument.
class SplitProblem {
 public:
  SplitProblem(int n, std::vector<SplitBlock> blocks) : n(n), blocks_(std::move(blocks)) {
    if (n < 1) throw std::invalid_argument("image size must be positive");
    std::vector<StackedMap::Block> stack;
    for (const auto& b : blocks_) {
      if (!b.map || !b.prox) throw std::invalid_argument("block needs a map and a prox");
      if (b.map->domain_size() != static_cast<std::size_t>(n) * n)
        throw std::invalid_argument("block domain does not match the image size");
      if (!b.offset.empty() && b.offset.size() != b.map->range_size())
        throw std::invalid_argument("block offset size mismatch");
      stack.push_back({b.weight, b.map});
    }
    stacked_ = std::make_shared<StackedMap>(std::move(stack));
    offsets_.assign(stacked_->range_size(), 0.0);
    for (std::size_t i = 0; i < blocks_.size(); ++i)
      if (!blocks_[i].offset.empty())
        std::copy(blocks_[i].offset.begin(), blocks_[i].offset.end(),
                  offsets_.begin() + stacked_->block_offset(i));
    classify();
  }

  std::size_t domain_size() const { return stacked_->domain_size(); }
  std::size_t range_size() const { return stacked_->range_size(); }
  const std::vector<SplitBlock>& blocks() const { return blocks_; }
  std::size_t block_offset(std::size_t i) const { return stacked_->block_offset(i); }
  const StackedMap& stacked() const { return *stacked_; }
  const std::vector<double>& offsets() const { return offsets_; }

  /// objective_from_ax / objective (solvers.cpp:362-388), on the host.
  double objective_from_ax(std::span<const double> ax) const {
    double total = 0.0;
    std::vector<double> tmp;
    for (std::size_t i = 0; i < blocks_.size(); ++i) {
      std::size_t off = block_offset(i), len = blocks_[i].map->range_size();
      std::span<const double> seg = ax.subspan(off, len);
      if (!blocks_[i].offset.empty()) {
        tmp.resize(len);
        for (std::size_t j = 0; j < len; ++j) tmp[j] = seg[j] - blocks_[i].offset[j];
        seg = tmp;
      }
      total += blocks_[i].prox->objective(seg);
      if (std::isinf(total)) return kInf;
    }
    return total;
  }
  double objective(std::span<const double> x) const {
    std::vector<double> ax(range_size());
    stacked_->forward(x, ax);
    return objective_from_ax(ax);
  }

  // ---- the device engine's view of the block list (set by classify) ----
  int n = 0;
  ncsg_kind kind = NCSG_CT;
  int n_angles = 0, n_det = 0;
  // engine parameters with the same block weights: D weight beta/alpha = w,
  // ScaledL1 bound lambda*alpha/beta = B (alpha = 1, beta = w, lambda = B w)
  double alpha = 1.0, beta = 1.0, lambda = 1.0;
  bool positivity = false;
  std::vector<double> offset;           // data-block offset b (PET: the counts)
  std::shared_ptr<ncsg_sparse> sparse;  // SparseMap data block (fan beam), else RadonMap
  double poisson_alpha = 0.0;           // PoissonConj's alpha (PET)

 private:
  void classify() {
    auto no_kernel = [](const std::string& why) {
      throw std::invalid_argument(
          "SplitProblem has no GPU kernel for this block list (" + why +
          "); the device engine runs {1, RadonMap|SparseMap|IdentityMap, Quadratic|Poisson} + "
          "{w, GradMap, ScaledL1Conj} [+ {1, IdentityMap, NonnegConj}] (pipeline.cpp:84-97)");
    };
    const std::size_t nn = static_cast<std::size_t>(n) * n;
    if (blocks_.size() < 2 || blocks_.size() > 3) no_kernel("2 or 3 blocks expected");
    const SplitBlock& d0 = blocks_[0];
    const SplitBlock& d1 = blocks_[1];
    if (d0.weight != 1.0) no_kernel("the data block weight must be 1");
    const auto* radon = dynamic_cast<const RadonMap*>(d0.map.get());
    const auto* sp = dynamic_cast<const SparseMap*>(d0.map.get());
    const auto* id0 = dynamic_cast<const IdentityMap*>(d0.map.get());
    const auto* quad = dynamic_cast<const QuadraticConj*>(d0.prox.get());
    const auto* pois = dynamic_cast<const PoissonConj*>(d0.prox.get());
    if (radon || sp) {
      n_angles = radon ? radon->n_angles() : sp->n_angles();
      n_det = radon ? radon->n_detectors() : sp->n_detectors();
      if (sp) sparse = sp->handle();
      if (quad) {
        kind = NCSG_CT;
        offset = d0.offset.empty() ? std::vector<double>(d0.map->range_size(), 0.0) : d0.offset;
      } else if (pois) {
        kind = NCSG_PET;
        for (double o : d0.offset)
          if (o != 0.0) no_kernel("a Poisson data block takes no offset");
        offset = pois->counts();
        poisson_alpha = pois->alpha();
      } else {
        no_kernel("the data block prox must be QuadraticConj or PoissonConj");
      }
    } else if (id0 && id0->domain_size() == nn && quad) {
      kind = NCSG_DENOISE;
      offset = d0.offset.empty() ? std::vector<double>(nn, 0.0) : d0.offset;
    } else {
      no_kernel("unsupported data-block map / prox");
    }
    const auto* grad = dynamic_cast<const GradMap*>(d1.map.get());
    const auto* l1 = dynamic_cast<const ScaledL1Conj*>(d1.prox.get());
    if (!grad || !l1 || grad->n() != n) no_kernel("the second block must be {w, GradMap(n), ScaledL1Conj}");
    if (!(d1.weight > 0.0)) no_kernel("the GradMap block weight must be positive");
    for (double o : d1.offset)
      if (o != 0.0) no_kernel("the GradMap block takes no offset");
    alpha = 1.0;
    beta = d1.weight;
    lambda = l1->bound() * d1.weight;
    positivity = false;
    if (blocks_.size() == 3) {
      const SplitBlock& d2 = blocks_[2];
      const auto* id2 = dynamic_cast<const IdentityMap*>(d2.map.get());
      if (!id2 || !dynamic_cast<const NonnegConj*>(d2.prox.get()) || d2.weight != 1.0)
        no_kernel("the third block must be {1, IdentityMap, NonnegConj}");
      for (double o : d2.offset)
        if (o != 0.0) no_kernel("the positivity block takes no offset");
      positivity = true;
    }
  }

  std::vector<SplitBlock> blocks_;
  std::shared_ptr<const StackedMap> stacked_;
  std::vector<double> offsets_;
};

/// assemble_problem (pipeline.cpp:69-98): the reference's block list on a
/// RadonMap or SparseMap geometry.
template <class Geometry>
inline SplitProblem assemble_problem(std::span<const double> sino,
                                     const std::shared_ptr<const Geometry>& geometry,
                                     const ModelParams& p) {
  if (p.model != "ct" && p.model != "pet")
    throw std::invalid_argument("unknown model \"" + p.model + "\"");
  if (p.alpha <= 0.0 || p.beta <= 0.0)
    throw std::invalid_argument("alpha and beta must be positive");
  if (p.lambda < 0.0) throw std::invalid_argument("lambda must be nonnegative");
  if (geometry->range_size() != sino.size())
    throw std::invalid_argument("sinogram shape does not match the geometry");
  const int n = geometry->n();
  std::vector<double> s(sino.begin(), sino.end());
  std::vector<SplitBlock> blocks;
  if (p.model == "ct")
    blocks.push_back({1.0, geometry, std::make_shared<QuadraticConj>(), s});
  else
    blocks.push_back({1.0, geometry, std::make_shared<PoissonConj>(s, p.alpha), {}});
  blocks.push_back({p.beta / p.alpha, std::make_shared<GradMap>(n),
                    std::make_shared<ScaledL1Conj>(p.lambda * p.alpha / p.beta), {}});
  if (p.positivity)
    blocks.push_back({1.0, std::make_shared<IdentityMap>(geometry->domain_size()),
                      std::make_shared<NonnegConj>(), {}});
  return SplitProblem(n, std::move(blocks));
}
inline SplitProblem assemble_problem(std::span<const double> sino, const RadonMap& geometry,
                                     const ModelParams& p) {
  return assemble_problem(sino, std::make_shared<const RadonMap>(geometry), p);
}
inline SplitProblem assemble_problem(std::span<const double> sino, const SparseMap& geometry,
                                     const ModelParams& p) {
  return assemble_problem(sino, std::make_shared<const SparseMap>(geometry), p);
}

/// TV denoising {1, I, QuadraticConj, noisy} + {beta/alpha, D, ScaledL1Conj}
/// (test_solvers.cpp:646-664).
inline SplitProblem denoise_problem(std::span<const double> noisy, int n, const ModelParams& p) {
  if (noisy.size() != static_cast<std::size_t>(n) * n)
    throw std::invalid_argument("image size mismatch");
  std::vector<SplitBlock> blocks;
  blocks.push_back({1.0, std::make_shared<IdentityMap>(noisy.size()),
                    std::make_shared<QuadraticConj>(),
                    std::vector<double>(noisy.begin(), noisy.end())});
  blocks.push_back({p.beta / p.alpha, std::make_shared<GradMap>(n),
                    std::make_shared<ScaledL1Conj>(p.lambda * p.alpha / p.beta), {}});
  if (p.positivity)
    blocks.push_back({1.0, std::make_shared<IdentityMap>(noisy.size()),
                      std::make_shared<NonnegConj>(), {}});
  return SplitProblem(n, std::move(blocks));
}

/// A rank's communicator for multi-GPU solves (ncsg_comm): one
/// process per GPU; the NCCL unique id is created on rank 0
/// (Communicator::unique_id) and shared by the caller (MPI, a file, ...).
class Communicator {
 public:
  static std::array<unsigned char, 128> unique_id() {
    std::array<unsigned char, 128> id{};
    detail::check(ncsg_nccl_unique_id(id.data()));
    return id;
  }
  /// NCCL communicator of rank `rank` of `nranks` on `device`.
  static std::shared_ptr<Communicator> nccl(const std::array<unsigned char, 128>& id, int rank,
                                            int nranks, int device) {
    ncsg_comm* c = nullptr;
    detail::check(ncsg_comm_create_nccl(id.data(), rank, nranks, device, &c));
    return std::shared_ptr<Communicator>(new Communicator(c, rank, nranks));
  }
  /// nranks communicators of one in-process group (one host thread per rank).
  static std::vector<std::shared_ptr<Communicator>> local_group(int nranks) {
    std::vector<ncsg_comm*> cs(nranks);
    detail::check(ncsg_comm_create_local(nranks, cs.data()));
    std::vector<std::shared_ptr<Communicator>> out;
    for (int r = 0; r < nranks; ++r)
      out.emplace_back(new Communicator(cs[r], r, nranks));
    return out;
  }
  ~Communicator() { ncsg_comm_destroy(c_); }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  ncsg_comm* get() const { return c_; }

 private:
  Communicator(ncsg_comm* c, int rank, int nranks) : c_(c), rank_(rank), nranks_(nranks) {}
  ncsg_comm* c_;
  int rank_, nranks_;
};

/// SolverConfig (solvers.hpp:54-72).  m_pinv_override / m_override are the
/// reference's explicit metric hooks; the device engine takes them as
/// CirculantMap (anything else: std::invalid_argument).
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
  std::shared_ptr<const LinearMap> m_pinv_override;
  std::shared_ptr<const LinearMap> m_override;
  int device = 0;
  /// Multi-GPU (no reference counterpart: the reference is serial): with a
  /// communicator of P > 1 ranks this rank solves its angle shard -- whole
  /// dihedral orbits when n_angles % 4 == 0, else a contiguous block -- and
  /// the exchange (slab FFT or all-reduce, ncsg.h) runs inside the library;
  /// the state's u then holds this rank's rays (x is replicated).
  std::shared_ptr<Communicator> comm;
  /// NCSG_XCHG_P2P (slab step, exchanges fused into the kernels over peer
  /// memory), NCSG_XCHG_SLAB (NCCL collectives) or NCSG_XCHG_ALLREDUCE.
  ncsg_exchange exchange = NCSG_XCHG_SLAB;
};

/// SolverState (solvers.hpp:74-78).
struct SolverState {
  ImageGrid x;
  std::vector<double> u;
  std::int64_t iter = 0;
};

/// make_state (solvers.cpp:406-411): zeros.
inline SolverState make_state(const SplitProblem& prob) {
  SolverState s;
  s.x = ImageGrid(prob.n);
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
    // pdhg_solve / admm_cg_solve preconditions (solvers.cpp:428-440)
    if (pdhg && (cfg.mask || cfg.m_pinv_override))
      throw std::invalid_argument("pdhg uses M = gamma I; drop the mask/overrides");
    if (n_cg > 0 && (cfg.mask || cfg.m_pinv_override))
      throw std::invalid_argument("admm_cg uses M = alpha A^T A; drop the mask/overrides");
    if (!(cfg.alpha > 0.0)) throw std::invalid_argument("alpha must be positive");
    // mode_from (solvers.cpp:75-79): Override > Mask > Scaled
    const bool override_mode = !pdhg && n_cg == 0 && cfg.m_pinv_override != nullptr;
    if (!override_mode && cfg.mask && cfg.mask->n != prob.n)
      throw std::invalid_argument("mask/problem size mismatch");
    if (prob.kind == NCSG_PET && prob.poisson_alpha != cfg.alpha)  // PoissonConj::evaluate
      throw std::invalid_argument("PoissonConj built for a different alpha");
    auto circulant = [&](const std::shared_ptr<const LinearMap>& m, const char* what) {
      const auto* c = dynamic_cast<const CirculantMap*>(m.get());
      if (!c)
        throw std::invalid_argument(std::string(what) +
                                    ": the GPU engine applies explicit metrics as circulants; "
                                    "pass a CirculantMap");
      if (c->mask().n != prob.n) throw std::invalid_argument("mask/problem size mismatch");
      return reinterpret_cast<const double*>(c->mask().h.data());
    };
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
    d.mask = (!pdhg && !override_mode && cfg.mask)
                 ? reinterpret_cast<const double*>(cfg.mask->h.data())
                 : nullptr;
    if (override_mode) {
      d.m_pinv = circulant(cfg.m_pinv_override, "m_pinv_override");
      if (cfg.m_override) d.m_symbol = circulant(cfg.m_override, "m_override");
    }
    d.b = prob.offset.data();
    d.device = cfg.device;
    d.sparse = prob.sparse.get();
    const int P = cfg.comm ? cfg.comm->nranks() : 1;
    if (P > 1) {
      if (prob.sparse) throw std::invalid_argument("sparse projectors are not angle-sharded");
      const int r = cfg.comm->rank();
      if (prob.n_angles % 4 == 0) {
        d.shard_rank = r;
        d.shard_count = P;
      } else {
        const int base = prob.n_angles / P, rem = prob.n_angles % P;
        d.angle_begin = r * base + std::min(r, rem);
        d.angle_end = d.angle_begin + base + (r < rem ? 1 : 0);
      }
    }
    ncsg_problem* h = nullptr;
    check(ncsg_problem_create(&d, &h));
    h_.reset(h, [](ncsg_problem* p) { ncsg_problem_destroy(p); });
    if (n_cg > 0) check(ncsg_set_cg(h, n_cg));
    if (P > 1) {
      comm_ = cfg.comm;
      check(ncsg_problem_set_comm(h, comm_->get(), cfg.exchange));
    }
  }
  ncsg_problem* get() const { return h_.get(); }

 private:
  std::shared_ptr<Communicator> comm_;  // outlives the problem's use of it
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
  s.iter = 0;  // solve_template (solvers.cpp:272)
  if (s.x.n != prob.n || s.u.size() != prob.range_size())  // Engine::init (solvers.cpp:118-121)
    throw std::invalid_argument("state does not match problem");
  check(ncsg_set_state(eng.get(), s.x.v.data(), s.u.data(), 0));
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
    auto hmax_of = [](const SpectralMask& m) {
      double hmax = 0.0;
      for (const auto& z : m.h) hmax = std::max(hmax, std::abs(z));
      return hmax;
    };
    if (!pdhg && cfg.m_pinv_override) {  // Override: 1.3 |lambda_max(M)| + 1 (solvers.cpp:219-226)
      const auto* c = dynamic_cast<const CirculantMap*>(cfg.m_override.get());
      shift = 1.3 * (c ? hmax_of(c->mask()) : 0.0) + 1.0;
    } else if (!pdhg && cfg.mask) {
      shift = cfg.gamma + cfg.alpha * hmax_of(*cfg.mask);
    }
    if (est > 1e-8 * std::max(1.0, shift)) {
      std::ostringstream os;
      os << "step condition M >= alpha A^T A appears violated "
            "(largest eigenvalue of alpha A^T A - M is about " << est << ")";
      res.record.warnings.push_back(os.str());
    }
  }
  res.state = std::move(s);
  check(ncsg_get_state(eng.get(), res.state.x.v.data(), res.state.u.data(), &res.state.iter));
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
  if (state.x.n != prob.n || state.u.size() != prob.range_size())
    throw std::invalid_argument("state does not match problem");
  detail::check(ncsg_set_state(eng.get(), state.x.v.data(), state.u.data(), state.iter));
  detail::check(ncsg_step(eng.get(), 1));
  std::int64_t div = -1;
  ncsg_status st = ncsg_sync(eng.get(), &div);
  if (st == NCSG_DIVERGED) throw DivergenceError(div, ncsg_last_error());  // absolute
  detail::check(st);
  detail::check(ncsg_get_state(eng.get(), state.x.v.data(), state.u.data(), nullptr));
  ++state.iter;
}

/// ncs_solve (solvers.cpp:423-426): the x-update mode follows mode_from
/// (solvers.cpp:75-79) -- m_pinv_override (a CirculantMap), else the mask's
/// pinv(gamma + alpha C), else M = gamma I (Scaled: the same iteration as
/// pdhg_solve).
inline SolveResult ncs_solve(const SplitProblem& prob, const SolverConfig& cfg,
                             const double* f_star = nullptr, const SolverState* init = nullptr) {
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
  if (cfg.mask || cfg.m_pinv_override)
    throw std::invalid_argument("admm_cg uses M = alpha A^T A; drop the mask/overrides");
  if (n_cg < 1) throw std::invalid_argument("n_cg must be >= 1");
  return detail::solve(prob, cfg, true, f_star, init, n_cg);
}

}  // namespace ncstomo_gpu
