#pragma once
// Counter-based dropout masks and synthetic-tensor streams, shared bit-for-bit by the CUDA
// kernels and the CPU oracle (oracle/). Built on the reference's hashing primitives
// (proj/include/curator/hashing.hpp:45-63) and its seed-derivation pattern
// `mix64(seed, fnv1a64(name))` (proj/src/pipeline.cpp:708-711).
//
// Mask definition (one SplitMix64 output per group of 4 consecutive elements, 16 uniform bits each):
//   bits = splitmix64(site_seed + (idx >> 2) * 0x9e3779b97f4a7c15)   i.e. output (idx>>2)+1 of the
//          SplitMix64 generator seeded with site_seed (reference hashing.hpp:45-50)
//   u16  = (bits >> (16 * (idx & 3))) & 0xffff
//   keep = u16 >= dropout_threshold16(p)          kept values are scaled by 1 / (1 - p)
// site_seed itself is derived with the reference's mix64 pattern (see site_seed() below).

#include <cmath>
#include <cstdint>
#include <string_view>

#include "curator/hashing.hpp"

namespace curator {

/// 16-bit drop threshold for probability p (p <= 0 keeps all, p >= 1 drops all).
inline std::uint32_t dropout_threshold16(double p) {
  if (!(p > 0.0)) return 0;
  if (p >= 1.0) return 65536;
  return static_cast<std::uint32_t>(std::llround(p * 65536.0));
}

inline constexpr std::uint64_t kSplitMixGamma = 0x9e3779b97f4a7c15ull;

/// 64 random bits for the group of 4 elements containing idx.
CURATOR_HD inline constexpr std::uint64_t dropout_bits(std::uint64_t site_seed, std::uint64_t group) {
  return splitmix64(site_seed + group * kSplitMixGamma);
}

CURATOR_HD inline constexpr bool dropout_keep(std::uint64_t site_seed, std::uint64_t idx, std::uint32_t thresh16) {
  const std::uint64_t bits = dropout_bits(site_seed, idx >> 2);
  const std::uint32_t u16 = static_cast<std::uint32_t>((bits >> (16u * static_cast<unsigned>(idx & 3u))) & 0xffffu);
  return u16 >= thresh16;
}

/// Dropout seed of training iteration `step`: iteration 0 keeps the base seed (so single-iteration
/// parity fixtures do not depend on the step), later iterations mix the step in with the reference's
/// mix64 so the masks of a microbatch differ from one training step to the next.
CURATOR_HD inline constexpr std::uint64_t step_seed(std::uint64_t seed, std::uint64_t step) {
  return step == 0 ? seed : mix64(seed, step);
}

/// Per-site seed: mix64(seed, fnv1a64(site) ^ (layer << 32 | microbatch)).
inline std::uint64_t site_seed(std::uint64_t seed, std::string_view site, std::uint32_t layer, std::uint32_t microbatch) {
  return mix64(seed, fnv1a64(site) ^ ((static_cast<std::uint64_t>(layer) << 32) | microbatch));
}

/// Element i of the standard-normal stream `key` (Box-Muller over pairs of uniform_unit draws).
CURATOR_HD inline double normal_at(std::uint64_t key, std::uint64_t i) {
  const std::uint64_t pair = i >> 1;
  const double u1 = uniform_unit(mix64(key, 2 * pair));
  const double u2 = uniform_unit(mix64(key, 2 * pair + 1));
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586 * u2;
  return (i & 1) ? r * sin(a) : r * cos(a);
}

}  // namespace curator
