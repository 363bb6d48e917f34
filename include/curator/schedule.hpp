#pragma once
// 1F1B pipeline schedule and tensor-parallel shard layout — the host-side partition/schedule
// logic the reference describes but does not implement (PAPER.md:152-192 for PipeDream-Flush
// 1F1B; PAPER.md:133-150 for Megatron tensor slicing; SPEC.md:557 lists 1F1B simulation as a
// non-goal of the reference). Written in the reference's API style (value types, free functions,
// std::invalid_argument on domain errors) and pinned by its formulas: the simulated bubble of
// one_f_one_b equals curator::pipeline_efficiency exactly.

#include <cstdint>
#include <vector>

namespace curator {

enum class PipeOpKind : int { Forward = 0, Backward = 1 };

struct PipeOp {
  PipeOpKind kind = PipeOpKind::Forward;
  int micro_batch = 0;
  bool operator==(const PipeOp& o) const { return kind == o.kind && micro_batch == o.micro_batch; }
};

/// Op order of `stage` in a `stages`-deep 1F1B pipeline over `micro_batches` microbatches:
/// min(stages - stage - 1, MB) warmup forwards, then MB - warmup (F, B) pairs, then the
/// remaining backwards. Length 2 * MB.
std::vector<PipeOp> one_f_one_b(int stage, int stages, int micro_batches);

/// Dependency-respecting simulation of all stages with integer op costs (F(mb) on stage s after
/// F(mb) on s-1; B(mb) on s after B(mb) on s+1 and F(mb) on s; each stage executes its list in
/// order). Returns the makespan.
std::int64_t simulate_one_f_one_b(int stages, int micro_batches, int t_forward, int t_backward);

/// Half-open index range.
struct Range {
  std::int64_t begin = 0;
  std::int64_t end = 0;
  std::int64_t size() const { return end - begin; }
  bool operator==(const Range& o) const { return begin == o.begin && end == o.end; }
};

/// Tensor-parallel shard of one transformer layer on `tp_rank` of `tp_size` (Megatron layout):
/// attention heads [heads.begin, heads.end); rows of the column-parallel QKV weight
/// (global rows ordered head, {q,k,v}, head_dim) and fc1 weight; columns of the row-parallel
/// attention-out and fc2 weights. LayerNorm parameters and the row-parallel biases are replicated.
struct LayerShard {
  Range heads;
  Range qkv_rows;       // of [3h, h]
  Range proj_cols;      // of [h, h]
  Range fc1_rows;       // of [ffn*h, h]
  Range fc2_cols;       // of [h, ffn*h]
};

LayerShard layer_shard(int hidden, int heads, int ffn_mult, int tp_size, int tp_rank);

/// Contiguous block of layers owned by pipeline stage `stage` (layers split evenly).
Range stage_layers(int layers, int stages, int stage);

}  // namespace curator
