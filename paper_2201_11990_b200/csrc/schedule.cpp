// 1F1B schedule, its simulation, and the tensor-parallel shard layout (see curator/schedule.hpp).
#include "curator/schedule.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace curator {

std::vector<PipeOp> one_f_one_b(int stage, int stages, int micro_batches) {
  if (stages < 1 || micro_batches < 1) throw std::invalid_argument("stages and micro_batches must be >= 1");
  if (stage < 0 || stage >= stages) throw std::invalid_argument("stage out of range");
  const int warmup = std::min(stages - stage - 1, micro_batches);
  std::vector<PipeOp> ops;
  ops.reserve(2 * static_cast<std::size_t>(micro_batches));
  int next_f = 0, next_b = 0;
  for (int i = 0; i < warmup; ++i) ops.push_back({PipeOpKind::Forward, next_f++});
  for (int i = 0; i < micro_batches - warmup; ++i) {
    ops.push_back({PipeOpKind::Forward, next_f++});
    ops.push_back({PipeOpKind::Backward, next_b++});
  }
  while (next_b < micro_batches) ops.push_back({PipeOpKind::Backward, next_b++});
  return ops;
}

std::int64_t simulate_one_f_one_b(int stages, int micro_batches, int t_forward, int t_backward) {
  if (t_forward < 0 || t_backward < 0) throw std::invalid_argument("op costs must be >= 0");
  std::vector<std::vector<PipeOp>> lists(stages);
  for (int s = 0; s < stages; ++s) lists[s] = one_f_one_b(s, stages, micro_batches);
  // finish[s][kind][mb]; -1 = not yet executed
  std::vector<std::vector<std::int64_t>> fin_f(stages, std::vector<std::int64_t>(micro_batches, -1));
  std::vector<std::vector<std::int64_t>> fin_b(stages, std::vector<std::int64_t>(micro_batches, -1));
  std::vector<std::size_t> pos(stages, 0);
  std::vector<std::int64_t> clock(stages, 0);
  std::size_t remaining = static_cast<std::size_t>(stages) * 2 * micro_batches;
  while (remaining > 0) {
    bool progressed = false;
    for (int s = 0; s < stages; ++s) {
      while (pos[s] < lists[s].size()) {
        const PipeOp op = lists[s][pos[s]];
        std::int64_t ready = clock[s];
        if (op.kind == PipeOpKind::Forward) {
          if (s > 0) {
            if (fin_f[s - 1][op.micro_batch] < 0) break;
            ready = std::max(ready, fin_f[s - 1][op.micro_batch]);
          }
          clock[s] = ready + t_forward;
          fin_f[s][op.micro_batch] = clock[s];
        } else {
          if (fin_f[s][op.micro_batch] < 0) break;
          ready = std::max(ready, fin_f[s][op.micro_batch]);
          if (s + 1 < stages) {
            if (fin_b[s + 1][op.micro_batch] < 0) break;
            ready = std::max(ready, fin_b[s + 1][op.micro_batch]);
          }
          clock[s] = ready + t_backward;
          fin_b[s][op.micro_batch] = clock[s];
        }
        ++pos[s];
        --remaining;
        progressed = true;
      }
    }
    if (!progressed) throw std::logic_error("1F1B schedule deadlocked");
  }
  return *std::max_element(clock.begin(), clock.end());
}

LayerShard layer_shard(int hidden, int heads, int ffn_mult, int tp_size, int tp_rank) {
  if (hidden <= 0 || heads <= 0 || ffn_mult <= 0 || tp_size <= 0)
    throw std::invalid_argument("layer dimensions and TP must be positive");
  if (tp_rank < 0 || tp_rank >= tp_size) throw std::invalid_argument("tp_rank out of range");
  if (hidden % heads != 0) throw std::invalid_argument("hidden not divisible by heads");
  if (heads % tp_size != 0)
    throw std::invalid_argument("heads (" + std::to_string(heads) + ") not divisible by TP (" + std::to_string(tp_size) +
                                ")");
  const std::int64_t h = hidden, head_dim = hidden / heads, local_heads = heads / tp_size;
  const std::int64_t ffn = std::int64_t{ffn_mult} * h, ffn_local = ffn / tp_size;
  if (ffn % tp_size != 0) throw std::invalid_argument("ffn width not divisible by TP");
  LayerShard s;
  s.heads = {tp_rank * local_heads, (tp_rank + 1) * local_heads};
  s.qkv_rows = {s.heads.begin * 3 * head_dim, s.heads.end * 3 * head_dim};
  s.proj_cols = {s.heads.begin * head_dim, s.heads.end * head_dim};
  s.fc1_rows = {tp_rank * ffn_local, (tp_rank + 1) * ffn_local};
  s.fc2_cols = s.fc1_rows;
  return s;
}

Range stage_layers(int layers, int stages, int stage) {
  if (layers < 1 || stages < 1 || stage < 0 || stage >= stages)
    throw std::invalid_argument("bad layers/stages/stage");
  if (layers % stages != 0)
    throw std::invalid_argument("layers (" + std::to_string(layers) + ") not divisible by PP (" +
                                std::to_string(stages) + ")");
  const std::int64_t per = layers / stages;
  return {stage * per, (stage + 1) * per};
}

}  // namespace curator
