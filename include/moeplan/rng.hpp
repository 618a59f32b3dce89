// B200 FSEP framework -- deterministic random streams shared with the planner.
// The stream definitions are part of the planner's observable behaviour (seeded
// perturbations, synthetic traces), so they follow the reference exactly:
// splitmix-style seed mixing and mt19937_64 with a 128-bit multiply-shift bounded
// draw, Box-Muller normals and Marsaglia-Tsang gammas
// (/root/reference/proj/include/moeplan/rng.hpp:24-85).
#pragma once
#include <cmath>
#include <cstdint>
#include <random>

namespace moeplan {

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b = 0) {
  constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
  constexpr std::uint64_t kSecond = 0x3c6ef372fe94f82bULL;
  std::uint64_t z = seed + kGolden * (a + 1) + kSecond * (b + 1);
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : mt_(seed) {}

  std::uint64_t next_u64() { return mt_(); }

  // [0, 1) with 53 random bits.
  double next_unit() { return static_cast<double>(mt_() >> 11) * (1.0 / 9007199254740992.0); }

  // [0, n) by multiply-shift (n > 0).
  std::uint64_t next_below(std::uint64_t n) {
    unsigned __int128 wide = static_cast<unsigned __int128>(mt_()) * n;
    return static_cast<std::uint64_t>(wide >> 64);
  }

  double next_normal() {
    const double u1 = 1.0 - next_unit();
    const double u2 = next_unit();
    constexpr double kTwoPi = 2.0 * 3.141592653589793238462643383279502884;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(kTwoPi * u2);
  }

  double next_gamma(double alpha) {
    if (alpha < 1.0) {
      const double u = 1.0 - next_unit();
      return next_gamma(alpha + 1.0) * std::pow(u, 1.0 / alpha);
    }
    const double d = alpha - 1.0 / 3.0;
    const double c = 1.0 / std::sqrt(9.0 * d);
    while (true) {
      const double x = next_normal();
      const double t = 1.0 + c * x;
      if (t <= 0.0) continue;
      const double v = t * t * t;
      const double u = 1.0 - next_unit();
      const double x2 = x * x;
      if (u < 1.0 - 0.0331 * x2 * x2) return d * v;
      if (std::log(u) < 0.5 * x2 + d * (1.0 - v + std::log(v))) return d * v;
    }
  }

 private:
  std::mt19937_64 mt_;
};

}  // namespace moeplan
