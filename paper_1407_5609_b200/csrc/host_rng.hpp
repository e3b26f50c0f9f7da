// host_rng.hpp — the reference's seeded sampling contract, host side.
//
// The reference draws every seeded value from std::mt19937_64 with hand
// samplers (core/include/pairscan/rng.hpp:14-41, core/src/rng.cpp:10-58) so
// that results are bit-exact across standard libraries.  The product needs
// the same stream for (a) the seeded reference choice of build_reference_set
// (refscan.cpp:41-42), and (b) the seeded synthetic datasets of the benchmark
// configs.  std::mt19937_64 itself is fully specified by the C++ standard.
#pragma once

#include <bit>
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <vector>

namespace psg {

class HostRng {
 public:
  explicit HostRng(uint64_t seed) : eng_(seed) {}
  uint64_t next() { return eng_(); }

  // Masked rejection (rng.cpp:10-20).
  uint64_t below(uint64_t bound) {
    if (bound == 0) throw std::invalid_argument("uniform_below: bound must be positive");
    if (bound == 1) return 0;
    const int width = 64 - std::countl_zero(bound - 1);
    const uint64_t mask = width == 64 ? ~0ull : ((1ull << width) - 1);
    for (;;) {
      const uint64_t v = eng_() & mask;
      if (v < bound) return v;
    }
  }
  // 53-bit unit real (rng.cpp:22-24).
  double unit() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  // Box-Muller, cosine branch, no cached spare (rng.cpp:26-32).
  double gauss(double mean, double sd) {
    const double u1 = 1.0 - unit();
    const double u2 = unit();
    const double r = std::sqrt(-2.0 * std::log(u1));
    return mean + sd * r * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
  // First k of a partial Fisher-Yates shuffle, selection order (rng.cpp:34-44).
  std::vector<uint64_t> choose(uint64_t n, uint64_t k) {
    if (k > n) throw std::invalid_argument("sample_without_replacement: k exceeds n");
    std::vector<uint64_t> pool(n);
    for (uint64_t i = 0; i < n; ++i) pool[i] = i;
    for (uint64_t i = 0; i < k; ++i) std::swap(pool[i], pool[i + below(n - i)]);
    pool.resize(k);
    return pool;
  }
  // The survey's float32 uniform: 24 high bits, exactly in [0,1).
  float u24() { return static_cast<float>(static_cast<double>(eng_() >> 40) * 0x1.0p-24); }

 private:
  std::mt19937_64 eng_;
};

// SplitMix64 finaliser and stream derivation (rng.cpp:46-58).
inline uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline uint64_t stream_seed(uint64_t base, uint64_t stream) { return splitmix(base ^ splitmix(stream + 1)); }

}  // namespace psg
