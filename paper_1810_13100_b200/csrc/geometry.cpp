// Host-side geometry of the parallel-beam projector (fp64, setup only).
//
// Replays the reference's ray table and per-sample box check so the device
// kernels visit exactly the reference's sample set, then derives the exact
// fixed-point lattice increments the kernels step with.  Compiled with
// -ffp-contract=off so the fp64 expressions round like the reference's
// (x86-64, no FMA) build.
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <numbers>
#include <thread>
#include <vector>

#include "ncsg_internal.cuh"

namespace ncsg {

namespace {

struct Interval {
  double lo, hi;
};

// axis_interval (radon.cpp:22-31): tau-interval where a + b*tau is in [lo, hi].
Interval axis_interval(double a, double b, double lo, double hi) {
  if (b == 0.0) {
    if (a >= lo && a <= hi) return {-1e30, 1e30};
    return {1.0, 0.0};
  }
  double t0 = (lo - a) / b;
  double t1 = (hi - a) / b;
  if (t0 > t1) std::swap(t0, t1);
  return {t0, t1};
}

long long q32(double v) { return std::llround(std::ldexp(v, 32)); }

// Shared-memory cost model of the adjoint scatter for one angle: lanes take
// rays `stride` apart, start y-aligned at a tile's top row and read-modify-
// write the 4 pixels of their sample.  Cost = average wavefronts per access
// (bank-conflict degree over the accumulator pitch) / fraction of useful
// lanes.  The stride with the lowest cost is used by bp_tile_kernel.
double scatter_cost(double aX, double aY, double bX, double bY, int stride, int W, int T,
                    int pitch) {
  const int rays = static_cast<int>(W * std::fabs(aX) + T * std::fabs(aY)) + 3;
  const int groups = (rays + 32 * stride - 1) / (32 * stride);
  const double util = static_cast<double>(rays) / (32.0 * stride * groups);
  double tot = 0.0;
  int cnt = 0;
  for (int trial = 0; trial < 8; ++trial) {
    const double x0 = 1.0 + 0.37 * trial, y0 = 2.0 + 0.11 * trial;
    for (int ph = 0; ph < stride; ++ph) {
      int nl = 0;
      double px[32], py[32];
      for (int l = 0; l < 32; ++l) {
        const int s = ph + stride * l;
        if (s >= rays) break;
        double x = x0 + s * aX, y = y0 + s * aY;
        const double k = std::ceil((y0 - y) / bY);
        px[nl] = x + k * bX;
        py[nl] = y + k * bY;
        ++nl;
      }
      if (!nl) continue;
      for (int step = 0; step < 3; ++step)
        for (int corner = 0; corner < 4; ++corner) {
          int bank_n[32] = {0};
          long addr[32];
          int worst = 0;
          // lanes' footprints are disjoint (stride >= 3), so addresses are distinct
          for (int l = 0; l < nl; ++l) {
            const long cy = static_cast<long>(std::floor(py[l] + step * bY)) + (corner >> 1);
            const long cx = static_cast<long>(std::floor(px[l] + step * bX)) + (corner & 1);
            addr[l] = cy * pitch + cx;
            worst = std::max(worst, ++bank_n[((addr[l] % 32) + 32) % 32]);
          }
          tot += worst;
          ++cnt;
        }
    }
  }
  return (tot / std::max(1, cnt)) / util;
}

}  // namespace

// Adjoint lane stride of every angle: the stride in 3..7 with the lowest
// scatter_cost, evaluated on all host cores (the model is ~1 ms per angle).
// Only the per-angle scatter (bp_tile_kernel) uses it, so RadonDev computes
// it on first use.
void choose_adjoint_strides(Geometry& g) {
  if (g.strides_ready) return;
  g.strides_ready = true;
  int bpW, bpT, bpP;
  bp_tile_shape(g.n, bpW, bpT, bpP);
  std::vector<AngleGeom*> all;
  for (auto& cls : g.cls)
    for (auto& a : cls) all.push_back(&a);
  auto work = [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      AngleGeom& a = *all[i];
      const double fax = std::ldexp(static_cast<double>(a.aX), -32);
      const double fay = std::ldexp(static_cast<double>(a.aY), -32);
      const double fbx = std::ldexp(static_cast<double>(a.dX), -32);
      const double fby = std::ldexp(static_cast<double>(a.dY), -32);
      double best = 1e300;
      a.bp_stride = 5;
      for (int st = 3; st <= 7; ++st) {
        const double cst = scatter_cost(fax, fay, fbx, fby, st, bpW, bpT, bpP);
        if (cst < best) best = cst, a.bp_stride = st;
      }
    }
  };
  const size_t nt = std::max<size_t>(1, std::min<size_t>(16, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  const size_t per = (all.size() + nt - 1) / nt;
  for (size_t t = 0; t < nt; ++t) {
    const size_t i0 = t * per, i1 = std::min(all.size(), i0 + per);
    if (i0 < i1) th.emplace_back(work, i0, i1);
  }
  for (auto& t : th) t.join();
}

Geometry build_geometry(int n, int n_angles, int n_det, int angle_begin, int angle_end,
                        int shard_rank, int shard_count) {
  // RadonMap::RadonMap validation (radon.cpp:37-42), same messages.
  if (n < 2) throw Error{NCSG_INVALID, "image size must be >= 2"};
  if (n_angles < 1) throw Error{NCSG_INVALID, "need at least one angle"};
  if (n_det % 2 == 0) throw Error{NCSG_INVALID, "detector count must be odd"};
  int min_det = static_cast<int>(std::ceil(std::numbers::sqrt2 * n));
  if (min_det % 2 == 0) ++min_det;
  if (n_det < min_det) throw Error{NCSG_INVALID, "detector row does not cover the image"};
  if (angle_end <= 0) {
    angle_begin = 0;
    angle_end = n_angles;
  }
  if (angle_begin < 0 || angle_end > n_angles || angle_begin >= angle_end)
    throw Error{NCSG_INVALID, "angle shard out of range"};
  const bool orbit_sharded = shard_count > 1;
  if (orbit_sharded) {
    if (n_angles % 4 != 0) throw Error{NCSG_INVALID, "orbit sharding needs a multiple of 4 angles"};
    if (shard_rank < 0 || shard_rank >= shard_count)
      throw Error{NCSG_INVALID, "shard rank out of range"};
    if (angle_begin != 0 || angle_end != n_angles)
      throw Error{NCSG_INVALID, "orbit sharding and angle ranges are exclusive"};
  }

  Geometry g;
  g.n = n;
  g.n_angles = n_angles;
  g.n_det = n_det;
  g.s_mid = (n_det - 1) / 2;
  g.P0 = static_cast<long long>(n - 1) << 31;  // c = (n-1)/2 in Q32
  g.rays.resize(static_cast<size_t>(n_angles) * n_det);
  g.orbit_sharded = orbit_sharded;
  g.own.assign(n_angles, 0);
  for (int t = 0; t < n_angles; ++t)
    g.own[t] = orbit_sharded ? (orbit_rep(t, n_angles) % shard_count == shard_rank)
                             : (t >= angle_begin && t < angle_end);

  const double c = 0.5 * (n - 1);
  const double s_mid = 0.5 * (n_det - 1);
  const double edge = n - 1;
  // Ray table replay, angle-parallel on the host cores (each angle writes its
  // own rows of g.rays and its own sample count).
  std::vector<int64_t> samples_t(n_angles, 0);
  auto replay = [&](int t0, int t1) {
    for (int t = t0; t < t1; ++t) {
      double theta = std::numbers::pi * t / n_angles;
      double ct = std::cos(theta);
      double st = std::sin(theta);
      for (int d = 0; d < n_det; ++d) {
        RayRange rr{1, 0};
        double s = d - s_mid;
        Interval ix = axis_interval(s * ct + c, -st, 0.0, n - 1);
        Interval iy = axis_interval(c - s * st, -ct, 0.0, n - 1);
        double lo = std::max(ix.lo, iy.lo);
        double hi = std::min(ix.hi, iy.hi);
        if (lo <= hi) {
          double k0 = std::ceil(lo);
          double k1 = std::floor(hi);
          if (k0 <= k1) {
            double px0 = s * ct - k0 * st + c;
            double py0 = c - s * st - k0 * ct;
            double dpx = -st, dpy = -ct;
            int count = static_cast<int>(k1 - k0) + 1;
            // per-sample box check (radon.cpp:88-90); valid samples of a ray
            // form one interval because px, py are monotone in k.
            auto valid = [&](int k) {
              double px = px0 + k * dpx;
              double py = py0 + k * dpy;
              return !(px < 0.0 || px > edge || py < 0.0 || py > edge);
            };
            int kf = 0;
            while (kf < count && !valid(kf)) ++kf;
            if (kf < count) {
              int kl = count - 1;
              while (kl > kf && !valid(kl)) --kl;
              int base = static_cast<int>(k0);
              rr.first = base + kf;
              rr.last = base + kl;
              samples_t[t] += kl - kf + 1;
            }
          }
        }
        g.rays[static_cast<size_t>(t) * n_det + d] = rr;
      }
    }
  };
  {
    const int nt = static_cast<int>(
        std::max<size_t>(1, std::min<size_t>(16, std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    const int per = (n_angles + nt - 1) / nt;
    for (int k = 0; k < nt; ++k) {
      const int t0 = k * per, t1 = std::min(n_angles, t0 + per);
      if (t0 < t1) th.emplace_back(replay, t0, t1);
    }
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < n_angles; ++t) {
    double theta = std::numbers::pi * t / n_angles;
    double ct = std::cos(theta);
    double st = std::sin(theta);
    bool own = g.own[t] != 0;
    if (own) g.samples += samples_t[t];
    if (!own) continue;

    AngleGeom a{};
    long long ax = q32(ct), ay = q32(-st), bx = q32(-st), by = q32(-ct);
    int cls = std::llabs(by) >= std::llabs(bx) ? 0 : 1;
    long long aX = cls == 0 ? ax : ay, aY = cls == 0 ? ay : ax;
    long long bX = cls == 0 ? bx : by, bY = cls == 0 ? by : bx;
    a.t = t;
    a.dir = bY > 0 ? 1 : -1;
    a.aX = aX;
    a.aY = aY;
    a.dX = a.dir * bX;
    a.dY = a.dir * bY;
    a.aXf = static_cast<float>(std::ldexp(static_cast<double>(aX), -32));
    a.aYf = static_cast<float>(std::ldexp(static_cast<double>(aY), -32));
    a.inv_dY16 = static_cast<float>(65536.0 / static_cast<double>(a.dY));
    a.inv_adX16 =
        a.dX == 0 ? 0.f : static_cast<float>(65536.0 / static_cast<double>(std::llabs(a.dX)));
    a.dXq = static_cast<int>(std::llround(std::ldexp(static_cast<double>(a.dX), -9)));
    a.bp_stride = 5;  // chosen on first use (choose_adjoint_strides)
    a.fp_rq = 8;      // orbit reps: chosen by RadonDev::upload (orbit_lane_rays)
    a.dYq = static_cast<int>(std::llround(std::ldexp(static_cast<double>(a.dY), -9)));
    g.cls[cls].push_back(a);
  }
  // Dihedral orbits (only for a full, unsharded angle set divisible by 4).
  if (n_angles % 4 == 0 && angle_begin == 0 && angle_end == n_angles) {  // full set or orbit shard
    const int q = n_angles / 4;
    for (const AngleGeom& a : g.cls[0]) {
      if (a.t > q) continue;  // reps: theta in [0, 45 deg]
      OrbitGeom o{};
      o.rep = a;
      o.t[0] = a.t;
      o.t[1] = a.t + 2 * q;
      o.t[2] = (a.t == 0 || a.t == q) ? -1 : n_angles - a.t;
      o.t[3] = (a.t == 0 || a.t == q) ? -1 : 2 * q - a.t;
      g.orbits.push_back(o);
    }
  }
  return g;
}

}  // namespace ncsg
