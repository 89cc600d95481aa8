// rng.hpp — seeded PCG32 (O'Neill's pcg32 "oneseq" variant) with a cached
// Box-Muller Gaussian, so seeded inputs are bit-identical to the reference's
// Rng (rng.hpp:13-48) on the same libm.
#pragma once

#include <cmath>
#include <cstdint>

namespace lrgw {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) {
    step();
    state_ += 0x853c49e6748fea9bULL ^ seed;
    step();
  }
  std::uint32_t next_u32() { return step(); }
  double uniform() { return (static_cast<double>(step()) + 1.0) / 4294967296.0; }  // (0, 1]
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double gaussian() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    const double u1 = uniform(), u2 = uniform();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    spare_ = rad * std::sin(ang);
    spare_ok_ = true;
    return rad * std::cos(ang);
  }

 private:
  std::uint32_t step() {
    const std::uint64_t s = state_;
    state_ = s * 6364136223846793005ULL + 1442695040888963407ULL;
    const std::uint32_t x = static_cast<std::uint32_t>(((s >> 18u) ^ s) >> 27u);
    const std::uint32_t rot = static_cast<std::uint32_t>(s >> 59u);
    return (x >> rot) | (x << ((32u - rot) & 31u));
  }
  std::uint64_t state_ = 0;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

}  // namespace lrgw
