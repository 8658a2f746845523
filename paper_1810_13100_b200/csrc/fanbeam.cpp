// Host-side fan-beam system matrix (fp64, setup only) for the SparseMap path.
//
// Restates build_fanbeam (fanbeam.cpp:43-111: Siddon ray/pixel-cell
// intersection lengths, view-major rows, pixel index (n-1-iy)*n + ix) and
// SparseMap's layout (sparse.cpp:9-45: CSR by row, rows stable-sorted, and the
// stored transpose by a counting sort over columns that keeps row order).
// Compiled with -ffp-contract=off so every length rounds like the
// reference's build; the device kernels consume the CSR arrays in fp32.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>

#include "ncsg_internal.cuh"

namespace ncsg {

namespace {

void clip_axis(double s, double d, double h, double& enter, double& exit_, bool& hit) {
  if (d == 0.0) {
    if (s < -h || s > h) hit = false;
    return;
  }
  double t0 = (-h - s) / d;
  double t1 = (h - s) / d;
  if (t0 > t1) std::swap(t0, t1);
  enter = std::max(enter, t0);
  exit_ = std::min(exit_, t1);
  if (enter >= exit_) hit = false;
}

}  // namespace

void fan_defaults(int n, double& source_radius, double& fan_angle) {
  // FanBeamGeometry::defaults (fanbeam.cpp:10-17)
  source_radius = n;
  fan_angle = 2.0 * std::asin(std::numbers::sqrt2 * n / (2.0 * source_radius));
}

SparseHost build_sparse(int n, int views, int rays, std::vector<int64_t> rows,
                        std::vector<int64_t> cols, std::vector<double> vals) {
  const size_t nr = static_cast<size_t>(views) * rays, nc = static_cast<size_t>(n) * n;
  for (size_t i = 0; i < rows.size(); ++i)
    if (rows[i] < 0 || rows[i] >= static_cast<int64_t>(nr) || cols[i] < 0 ||
        cols[i] >= static_cast<int64_t>(nc))
      throw Error{NCSG_INVALID, "sparse triplet out of range"};
  // stable sort by row (sparse.cpp:19-20)
  std::vector<size_t> order(rows.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return rows[a] < rows[b]; });
  SparseHost S;
  S.n = n;
  S.views = views;
  S.rays = rays;
  S.row_ptr.assign(nr + 1, 0);
  S.col.resize(order.size());
  S.val.resize(order.size());
  for (size_t i = 0; i < order.size(); ++i) ++S.row_ptr[rows[order[i]] + 1];
  for (size_t r = 0; r < nr; ++r) S.row_ptr[r + 1] += S.row_ptr[r];
  for (size_t i = 0; i < order.size(); ++i) {
    S.col[i] = static_cast<int>(cols[order[i]]);
    S.val[i] = vals[order[i]];
  }
  // stored transpose by counting sort over columns (sparse.cpp:31-44)
  S.t_row_ptr.assign(nc + 1, 0);
  S.t_col.resize(order.size());
  S.t_val.resize(order.size());
  for (size_t i = 0; i < S.col.size(); ++i) ++S.t_row_ptr[S.col[i] + 1];
  for (size_t c = 0; c < nc; ++c) S.t_row_ptr[c + 1] += S.t_row_ptr[c];
  std::vector<int64_t> cursor(S.t_row_ptr.begin(), S.t_row_ptr.end() - 1);
  for (size_t r = 0; r < nr; ++r)
    for (int64_t i = S.row_ptr[r]; i < S.row_ptr[r + 1]; ++i) {
      const int64_t dst = cursor[S.col[i]]++;
      S.t_col[dst] = static_cast<int>(r);
      S.t_val[dst] = S.val[i];
    }
  return S;
}

SparseHost build_fanbeam(int n, int views, int rays, double source_radius, double fan_angle) {
  // validation and messages of build_fanbeam (fanbeam.cpp:44-51)
  if (n < 2) throw Error{NCSG_INVALID, "image size must be >= 2"};
  if (views < 1 || rays < 1)
    throw Error{NCSG_INVALID, "fan-beam needs at least one view and one ray"};
  const double h = 0.5 * n;
  if (source_radius <= h * std::numbers::sqrt2)
    throw Error{NCSG_INVALID, "source must lie outside the image corner circle"};
  if (fan_angle <= 0.0 || fan_angle >= std::numbers::pi)
    throw Error{NCSG_INVALID, "fan angle must lie in (0, pi)"};
  std::vector<int64_t> tr, tc;
  std::vector<double> tv;
  tr.reserve(static_cast<size_t>(views) * rays * 2 * n);
  tc.reserve(tr.capacity());
  tv.reserve(tr.capacity());
  const double dpsi = rays > 1 ? fan_angle / (rays - 1) : 0.0;
  const double psi0 = -0.5 * fan_angle;
  int64_t ray_index = 0;
  for (int v = 0; v < views; ++v) {
    const double phi = 2.0 * std::numbers::pi * v / views;
    const double sx = source_radius * std::cos(phi), sy = source_radius * std::sin(phi);
    const double cx = -std::cos(phi), cy = -std::sin(phi);
    for (int r = 0; r < rays; ++r, ++ray_index) {
      const double psi = rays > 1 ? psi0 + r * dpsi : 0.0;
      const double cp = std::cos(psi), sp = std::sin(psi);
      const double dx = cp * cx - sp * cy;
      const double dy = sp * cx + cp * cy;
      double enter = 0.0, exit_ = std::numeric_limits<double>::infinity();
      bool hit = true;
      clip_axis(sx, dx, h, enter, exit_, hit);
      clip_axis(sy, dy, h, enter, exit_, hit);
      if (!hit) continue;
      double t = enter;
      const double px = sx + t * dx, py = sy + t * dy;
      int ix = std::clamp(static_cast<int>(std::floor(px + h)), 0, n - 1);
      int iy = std::clamp(static_cast<int>(std::floor(py + h)), 0, n - 1);
      const int step_x = dx > 0.0 ? 1 : -1, step_y = dy > 0.0 ? 1 : -1;
      while (t < exit_ - 1e-12) {
        const double tx = dx != 0.0 ? ((ix + (step_x > 0 ? 1 : 0)) - h - sx) / dx
                                    : std::numeric_limits<double>::infinity();
        const double ty = dy != 0.0 ? ((iy + (step_y > 0 ? 1 : 0)) - h - sy) / dy
                                    : std::numeric_limits<double>::infinity();
        const double t_next = std::max(std::min({tx, ty, exit_}), t);
        const double len = t_next - t;
        if (len > 0.0) {
          tr.push_back(ray_index);
          tc.push_back(static_cast<int64_t>(n - 1 - iy) * n + ix);
          tv.push_back(len);
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
  return build_sparse(n, views, rays, std::move(tr), std::move(tc), std::move(tv));
}

}  // namespace ncsg
