// ---------------------------------------------------------------------------
// eps/rng.hpp -- deterministic randomness on the decision path.
//
// Shard shuffles (redistribute) and the synthetic norm source must match the
// reference bit for bit (rng.hpp:11-43), so: splitmix64 with the published
// constants, modulo reduction for bounded draws, and the descending
// Fisher-Yates walk.  <random> distributions and std::shuffle are
// implementation-defined and never used on a decision path.
// ---------------------------------------------------------------------------
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

namespace eps {

class SplitMix64 {
 public:
  static constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;  // state increment

  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}

  std::uint64_t next() {  // Steele, Lea & Flood (2014) output function
    state_ += kGolden;
    std::uint64_t x = state_;
    x = (x ^ (x >> 30)) * kMulA;
    x = (x ^ (x >> 27)) * kMulB;
    return x ^ (x >> 31);
  }
  std::uint64_t next_below(std::uint64_t bound) {  // [0, bound), bound > 0, plain modulo
    return next() % bound;
  }
  double next_unit() {  // [0, 1) from the top 53 bits
    return static_cast<double>(next() >> 11) * 0x1.0p-53;
  }

 private:
  static constexpr std::uint64_t kMulA = 0xbf58476d1ce4e5b9ull;
  static constexpr std::uint64_t kMulB = 0x94d049bb133111ebull;
  std::uint64_t state_;
};

// a ^ (b + golden + (a << 6) + (a >> 2)): seeds per (run, epoch, node).
inline std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {
  return a ^ (b + SplitMix64::kGolden + (a << 6) + (a >> 2));
}

// Fisher-Yates from the back: slot n-1 swaps with next_below(n), n = size .. 2.
template <typename T>
void deterministic_shuffle(std::vector<T>& v, SplitMix64& rng) {
  for (std::size_t n = v.size(); n > 1; --n)
    std::swap(v[n - 1], v[static_cast<std::size_t>(rng.next_below(n))]);
}

}  // namespace eps
