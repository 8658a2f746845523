// Host-side restatement of the reference's seeded stream generator
// (rng.cpp:9-46: SplitMix64 stream, 53-bit uniforms, Box-Muller normals with
// a cached second value), used to draw the probe images of calibrate_scale
// (circulant.cpp:89-94) and the power-method start vector
// (solvers.cpp:469-474) bit-for-bit as the reference does.
#pragma once

#include <cmath>
#include <cstdint>

namespace ncsg {

class HostRng {
 public:
  HostRng(uint64_t seed, uint64_t stream) : state_(mix(mix(seed) + stream)) {}

  uint64_t next_u64() {
    state_ += 0x9e3779b97f4a7c15ULL;
    return finalize(state_);
  }
  double next_double() {
    uint64_t bits = next_u64() >> 11;
    if (bits == 0) bits = 1;
    return static_cast<double>(bits) * 0x1.0p-53;
  }
  double next_normal() {
    if (cached_) {
      cached_ = false;
      return spare_;
    }
    const double u1 = next_double(), u2 = next_double();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * 3.141592653589793238462643383279502884 * u2;
    spare_ = r * std::sin(t);
    cached_ = true;
    return r * std::cos(t);
  }

 private:
  static uint64_t finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  static uint64_t mix(uint64_t z) { return finalize(z + 0x9e3779b97f4a7c15ULL); }
  uint64_t state_;
  bool cached_ = false;
  double spare_ = 0.0;
};

}  // namespace ncsg
