#pragma once
// Counter-based hashing / RNG primitives with the same outputs as the reference's
// proj/include/curator/hashing.hpp:13-63 (FNV-1a 64 and splitmix64 with their published
// constants). They key every synthetic tensor, initial weight and dropout mask of the
// runtime, so the CPU oracle and the GPU kernels derive bit-identical streams.
//
// All functions are constexpr-friendly and usable from host and device code.

#include <cstddef>
#include <cstdint>
#include <string_view>

#if defined(__CUDACC__)
#define CURATOR_HD __host__ __device__
#else
#define CURATOR_HD
#endif

namespace curator {

inline constexpr std::uint64_t kFnvOffsetBasis = 14695981039346656037ull;  // 0xcbf29ce484222325
inline constexpr std::uint64_t kFnvPrime = 1099511628211ull;               // 0x100000001b3

/// FNV-1a over raw bytes, chainable through `h`.
inline std::uint64_t fnv1a64(const void* data, std::size_t len, std::uint64_t h = kFnvOffsetBasis) {
  const unsigned char* bytes = static_cast<const unsigned char*>(data);
  for (const unsigned char* end = bytes + len; bytes != end; ++bytes) h = (h ^ *bytes) * kFnvPrime;
  return h;
}

inline std::uint64_t fnv1a64(std::string_view text, std::uint64_t h = kFnvOffsetBasis) {
  return fnv1a64(text.data(), text.size(), h);
}

/// Feeds the little-endian bytes of a 32-bit value.
inline std::uint64_t fnv1a64_u32(std::uint32_t v, std::uint64_t h) {
  for (int i = 0; i < 4; ++i) h = (h ^ ((v >> (8 * i)) & 0xffu)) * kFnvPrime;
  return h;
}

/// Feeds the little-endian bytes of a 64-bit value.
inline std::uint64_t fnv1a64_u64(std::uint64_t v, std::uint64_t h) {
  for (int i = 0; i < 8; ++i) h = (h ^ ((v >> (8 * i)) & 0xffu)) * kFnvPrime;
  return h;
}

/// splitmix64 finaliser of a Weyl step.
CURATOR_HD inline constexpr std::uint64_t splitmix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/// Two-input mixer: splitmix64(a ^ splitmix64(b)).
CURATOR_HD inline constexpr std::uint64_t mix64(std::uint64_t a, std::uint64_t b) {
  return splitmix64(a ^ splitmix64(b));
}

/// Top 53 bits mapped to the open interval (0, 1): (bits/2^11 + 1/2) / 2^53.
CURATOR_HD inline constexpr double uniform_unit(std::uint64_t bits) {
  return (static_cast<double>(bits >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

}  // namespace curator
