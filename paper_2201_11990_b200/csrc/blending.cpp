// Largest-remainder dataset blending (curator::next_batch_composition), restated from the
// reference's semantics (proj/src/blending.cpp:10-97, contract in blending.hpp:31-36): the fp64
// evaluation order of quota = credit + weight * batch and credit' = quota - count is kept so the
// count stream and the carried credit are bit-identical to the reference (tests/test_feed.py diffs
// them live against the reference compiled from its own source).
#include "curator/blending.hpp"

#include <cmath>
#include <stdexcept>

#include "curator/errors.hpp"

namespace curator {

void validate_weights(std::span<const DatasetSpec> specs) {
  if (specs.empty()) throw ConfigError("no datasets configured");
  double total = 0.0;
  for (const DatasetSpec& s : specs) {
    if (!(s.weight > 0.0) || s.weight > 1.0) throw ConfigError("dataset \"" + s.name + "\" weight must be in (0,1]");
    total += s.weight;
  }
  if (std::fabs(total - 1.0) > 1e-9)
    throw ConfigError("dataset weights sum to " + std::to_string(total) + ", expected 1");
}

void normalize_weights(std::vector<DatasetSpec>& specs) {
  double total = 0.0;
  for (const DatasetSpec& s : specs) total += s.weight;
  if (!(total > 0.0)) throw ConfigError("dataset weights must be positive");
  for (DatasetSpec& s : specs) s.weight /= total;
}

BlendState BlendState::create(std::size_t dataset_count) {
  BlendState st;
  st.drawn = std::vector<std::uint64_t>(dataset_count, 0);
  st.credit = std::vector<double>(dataset_count, 0.0);
  return st;
}

std::vector<std::uint64_t> next_batch_composition(BlendState& state, std::span<const DatasetSpec> specs,
                                                  std::uint64_t batch_size) {
  validate_weights(specs);
  if (batch_size == 0) throw std::invalid_argument("batch_size must be >= 1");
  const std::size_t n = specs.size();
  if (state.drawn.size() != n || state.credit.size() != n)
    throw std::invalid_argument("state size does not match specs");

  std::vector<double> quota(n), frac(n);
  std::vector<std::uint64_t> counts(n, 0);
  std::int64_t left = static_cast<std::int64_t>(batch_size);
  for (std::size_t i = 0; i < n; ++i) {
    quota[i] = state.credit[i] + specs[i].weight * static_cast<double>(batch_size);
    const double whole = std::floor(quota[i]);
    if (whole > 0.0) counts[i] = static_cast<std::uint64_t>(whole);
    left -= static_cast<std::int64_t>(counts[i]);
    frac[i] = quota[i] - static_cast<double>(counts[i]);
  }
  // Rank datasets by fractional remainder, largest first, earlier dataset first on ties
  // (insertion sort: n is the number of datasets, and it is stable by construction).
  std::vector<std::size_t> rank(n);
  for (std::size_t i = 0; i < n; ++i) {
    std::size_t j = i;
    while (j > 0 && frac[rank[j - 1]] < frac[i]) {
      rank[j] = rank[j - 1];
      --j;
    }
    rank[j] = i;
  }
  for (std::size_t k = 0; k < n && left > 0; ++k, --left) ++counts[rank[k]];
  // Negative carried credit can over-assign; give samples back from the smallest remainders.
  for (std::size_t k = n; k > 0 && left < 0; --k) {
    if (counts[rank[k - 1]] > 0) {
      --counts[rank[k - 1]];
      ++left;
    }
  }
  ++state.step;
  for (std::size_t i = 0; i < n; ++i) {
    state.drawn[i] += counts[i];
    state.credit[i] = quota[i] - static_cast<double>(counts[i]);
  }
  return counts;
}

}  // namespace curator
