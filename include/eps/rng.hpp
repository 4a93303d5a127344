// Deterministic randomness for the control plane.
//
// Drop-in for the reference's proj/include/eps/rng.hpp:11-43.  Shard
// shuffles (autodp redistribute) and the synthetic gradient-norm source must
// reproduce the reference bit for bit, so the generator is splitmix64 with
// the same constants, `next_below` is a plain modulo and the shuffle is the
// descending Fisher-Yates walk.  std::shuffle / <random> distributions are
// implementation-defined and therefore never used on a decision path.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

namespace eps {

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}

  // One splitmix64 step (Steele, Lea, Flood 2014; constants as in
  // rng.hpp:15-20).
  std::uint64_t next() {
    state_ += kGolden;
    std::uint64_t z = state_;
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
  }

  // [0, bound) by modulo reduction (rng.hpp:24); bound must be > 0.
  std::uint64_t next_below(std::uint64_t bound) { return next() % bound; }

  // [0, 1) from the top 53 bits (rng.hpp:27).
  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

  static constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;

 private:
  static constexpr std::uint64_t kMix1 = 0xbf58476d1ce4e5b9ull;
  static constexpr std::uint64_t kMix2 = 0x94d049bb133111ebull;
  std::uint64_t state_;
};

// Boost-style combine (rng.hpp:33-36).
inline std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {
  return a ^ (b + SplitMix64::kGolden + (a << 6) + (a >> 2));
}

// In-place Fisher-Yates, last slot first (rng.hpp:38-43).
template <typename T>
void deterministic_shuffle(std::vector<T>& v, SplitMix64& rng) {
  for (std::size_t n = v.size(); n > 1; --n) {
    const auto pick = static_cast<std::size_t>(rng.next_below(n));
    std::swap(v[n - 1], v[pick]);
  }
}

}  // namespace eps
