// SplitMix64 stream with the 53-bit unit mapping — bit-exact with
// /root/reference/proj/include/archetype/prng.hpp:11-30, so seeds recorded by
// either implementation replay identically in the other.
#pragma once

#include <cstdint>

namespace archetype {

class Prng {
 public:
  explicit Prng(std::uint64_t seed) : state_(seed) {}

  std::uint64_t next_u64() {
    state_ += kGolden;
    std::uint64_t z = state_;
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
  }

  /// Uniform in [0, 1): the top 53 bits times 2^-53.
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

 private:
  static constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
  static constexpr std::uint64_t kMix1 = 0xBF58476D1CE4E5B9ULL;
  static constexpr std::uint64_t kMix2 = 0x94D049BB133111EBULL;
  std::uint64_t state_;
};

}  // namespace archetype
