// Counter-based sampling stream and SplitMix64 engine, host side.
// Semantics follow the reference bit for bit:
//   mix / unit_uniform / derive_seed   proj/src/rng.cpp:7-24
//   SplitMix64 + below + shuffle       proj/include/parac/rng.hpp:35-61, src/rng.cpp:26-33
//   domain salts                       proj/include/parac/rng.hpp:24-29
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

namespace parac_gpu {

inline constexpr std::uint64_t kSaltSampling = 0x73616d706c696e67ULL;
inline constexpr std::uint64_t kSaltOrdering = 0x6f72646572696e67ULL;
inline constexpr std::uint64_t kSaltTieBreak = 0x7469656272656b00ULL;
inline constexpr std::uint64_t kSaltRhs = 0x7268735f76656320ULL;
inline constexpr std::uint64_t kSaltCells = 0x63656c6c636f6566ULL;
inline constexpr std::uint64_t kSaltRmat = 0x726d61745f67656eULL;  // this repo's R-MAT stream

inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline double unit_uniform(std::uint64_t seed, std::int64_t key, std::uint64_t counter) {
  std::uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (static_cast<std::uint64_t>(key) + 1);
  x = mix64(x);
  x = mix64(x ^ (0xd1b54a32d192ed03ULL * (counter + 1)));
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t salt) {
  return mix64(seed ^ mix64(salt));
}

struct SplitMix64 {
  std::uint64_t state = 0;
  explicit SplitMix64(std::uint64_t s = 0) : state(s) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t below(std::uint64_t n) {
    if (n <= 1) return 0;
    const std::uint64_t bound = n * (~0ULL / n);
    std::uint64_t r = next();
    while (r >= bound) r = next();
    return r % n;
  }
};

template <typename T>
void shuffle(std::vector<T>& values, SplitMix64& rng) {
  for (std::size_t i = values.size(); i > 1; --i) {
    std::size_t j = static_cast<std::size_t>(rng.below(i));
    std::swap(values[i - 1], values[j]);
  }
}

}  // namespace parac_gpu
