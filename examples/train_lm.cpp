// Example C++ caller of the C ABI (the binding a reference maintainer adds): one
// process per GPU trains a language-model pipeline stage from a blend manifest. Compiled (syntax only)
// by tests/test_capi.py so the documented calls stay in sync with include/mtnlg.h.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "curator/blending.hpp"
#include "curator/errors.hpp"
#include "curator/planner.hpp"
#include "mtnlg.h"

static void check(int rc) {  // status -> the reference's exception taxonomy
  if (rc == MT_ERR_CONFIG) throw curator::ConfigError(mt_last_error());
  if (rc != MT_OK) throw curator::DataError(mt_last_error());
}

void train(int rank, int world, const unsigned char nccl_id[128], const char* manifest, int64_t steps, cudaStream_t s) {
  mt_ctx* ctx = nullptr;
  check(mt_ctx_create(rank, &ctx));
  mt_parallel_config par{/*tensor*/ 2, /*pipeline*/ 2, /*data*/ world / 4, /*batch*/ 16, /*micro_batches*/ 8};
  check(mt_ctx_init_comm(ctx, nccl_id, world, rank, &par));  // groups from curator::map_topology
  mt_rank_placement place{};
  check(mt_ctx_placement(ctx, &place));

  mt_stage_desc d{};
  d.layer = {12288, 96, 2048, 1, 0, 0, 4, 0.1f, 0.1f, 1e-5f, 20260808ull, 0};
  d.layers = 4;
  d.micro_batches = 8;
  mt_stage* st = nullptr;
  check(mt_stage_create(ctx, &d, &st));
  for (int i = 0; i < d.layers / par.pipeline; ++i) {
    mt_layer* l = nullptr;
    check(mt_stage_layer(st, i, &l));
    check(mt_layer_init_params(l, s));
  }
  mt_vocab_desc vd{50257, 12288, 2048, 1, par.tensor, place.tensor, 0.1f, 1e-5f, 1234};
  mt_vocab* voc = nullptr;
  check(mt_vocab_create(ctx, &vd, &voc));
  check(mt_stage_attach_vocab(st, voc));  // inputs / targets become int32 token ids

  mt_feed_desc fd{50257, 2048, /*micro_batch*/ 1, par.data, place.data, 1234};
  mt_feed* feed = nullptr;
  check(mt_feed_open(manifest, &fd, &feed));
  const int32_t max_mb = d.micro_batches;
  std::vector<int32_t> tokens(size_t(max_mb) * 2048), targets(tokens.size());
  double tokens_seen = 0;
  for (int64_t step = 0; step < steps; ++step) {
    int64_t global_batch = 0;
    int32_t mb = 0;
    check(mt_feed_step_info(feed, step, &global_batch, &mb));
    check(mt_feed_fill(feed, step, tokens.data(), targets.data(), max_mb));
    check(mt_stage_set_micro_batches(st, mb));
    float loss = 0.f, grad_norm = 0.f;
    check(mt_stage_train_step(st, tokens.data(), targets.data(), &loss, s));
    mt_adam_desc a{};
    check(mt_adam_defaults(&a));  // TrainingRecipe constants; lr < 0 -> curator::lr_at(tokens_seen)
    a.step = static_cast<int32_t>(step + 1);
    a.tokens_seen = tokens_seen;
    check(mt_stage_optimizer_step(st, &a, &grad_norm, s));
    tokens_seen += static_cast<double>(global_batch) * 2048;
  }
  check(mt_feed_destroy(feed));
  check(mt_stage_destroy(st));
  check(mt_vocab_destroy(voc));
  check(mt_ctx_destroy(ctx));
}
