/* mtnlg.h — C ABI of the B200-native MT-NLG training-step runtime (libmtnlg.so).
 *
 * Drop-in boundary for the hot path of arxiv/paper_2201_11990: the reference keeps only the
 * analytical planner (proj/include/curator/planner.hpp:7-128, C++, statically linked) and has no
 * runtime below it. This ABI exposes (1) the planner's partition and
 * schedule functions in plain C so any FFI can bind them, and (2) the GPU runtime that executes
 * the layout the planner decides: the tensor-sliced transformer layer forward/backward on sm_100a
 * kernels, its TP all-reduces, the 1F1B pipeline and the DP gradient all-reduce over NCCL.
 *
 * Conventions: plain pointers and sizes, no exceptions across the boundary.
 * Every function returns MT_OK (0), MT_ERR_CONFIG (1: bad argument / layout — the reference's
 * ConfigError / std::invalid_argument) or MT_ERR_DATA (2: CUDA / NCCL / data failure — the
 * reference's DataError); mt_last_error() holds the message (thread-local).
 * Streams are cudaStream_t passed as void*. The caller owns host buffers and device buffers it
 * passes in; the library owns what *_create allocates and frees it in *_destroy.
 */
#ifndef MTNLG_H
#define MTNLG_H

#include <stddef.h>
#include <stdint.h>

#include "mtnlg_gemm.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { MT_OK = 0, MT_ERR_CONFIG = 1, MT_ERR_DATA = 2 };

const char* mt_last_error(void);
const char* mt_version(void);

/* ------------------------------------------------------------------ planner (host, pure) */
/* Mirrors curator::ClusterTopology / ParallelConfig / RankPlacement (planner.hpp:18-36, 84-90). */
typedef struct mt_cluster_topology {
  int32_t nodes, gpus_per_node;
  double intra_node_bw, inter_node_bw, peak_flops_per_gpu;
} mt_cluster_topology;

typedef struct mt_parallel_config {
  int32_t tensor, pipeline, data, batch, micro_batches;
} mt_parallel_config;

typedef struct mt_rank_placement {
  int32_t data, pipeline, tensor, node, gpu;
} mt_rank_placement;

typedef struct mt_model_shape {
  double parameters;
  int32_t layers, hidden, heads, sequence, vocab;
} mt_model_shape;

/* curator::map_topology (reference proj/src/planner.cpp:84-128). Writes min(cap, n) placements,
 * *n = TP*PP*DP. Errors: MT_ERR_CONFIG with the reference's message. */
int mt_map_topology(const mt_cluster_topology* topo, const mt_parallel_config* par, mt_rank_placement* out,
                    int64_t cap, int64_t* n);
/* curator::pipeline_efficiency (planner.cpp:27-32) */
int mt_pipeline_efficiency(int32_t micro_batches, int32_t stages, double* out);
/* curator::estimated_tflops_per_gpu (planner.cpp:39-57) */
int mt_estimated_tflops_per_gpu(const mt_model_shape* shape, const mt_parallel_config* par,
                                const mt_cluster_topology* topo, double iteration_seconds, double* out);
/* curator::weight_init_std, activation_bytes, model_state_bytes, lr_at, batch_size_at */
int mt_weight_init_std(double hidden, double* out);
int mt_activation_bytes(double batch, double layers, double sequence, double hidden, double* out);
int mt_model_state_bytes(double parameters, double* out);
int mt_lr_at(double tokens_seen, double* out);
int mt_batch_size_at(double tokens_seen, int32_t* out);
/* curator::parse_planner_config + build_plan_report + render_plan_report: writes up to cap bytes
 * (NUL-terminated) of the rendered report; *len = full length. */
int mt_plan_report(const char* config_path, int32_t as_json, char* out, int64_t cap, int64_t* len);

/* 1F1B (PipeDream-Flush) op order of one stage: warmup = min(PP-stage-1, MB)
 * forwards, then MB-warmup (F, B) pairs, then warmup backwards. kind 0 = forward, 1 = backward. */
typedef struct mt_pipe_op {
  int32_t kind, micro_batch;
} mt_pipe_op;
int mt_pipeline_schedule(int32_t stage, int32_t stages, int32_t micro_batches, mt_pipe_op* out, int32_t cap,
                         int32_t* n);
/* Unit-cost simulation of the 1F1B schedule over all stages with integer op costs; *makespan in
 * cost units. Pins pipeline_efficiency: makespan == (MB + PP - 1) * (t_fwd + t_bwd). */
int mt_pipeline_simulate(int32_t stages, int32_t micro_batches, int32_t t_fwd, int32_t t_bwd, int64_t* makespan);

/* ------------------------------------------------------------------ layer parameters */
enum mt_param {
  MT_P_LN1_GAMMA = 0, MT_P_LN1_BETA, MT_P_QKV_W, MT_P_QKV_B, MT_P_PROJ_W, MT_P_PROJ_B,
  MT_P_LN2_GAMMA, MT_P_LN2_BETA, MT_P_FC1_W, MT_P_FC1_B, MT_P_FC2_W, MT_P_FC2_B, MT_P_COUNT
};

typedef struct mt_layer_desc {
  int32_t hidden, heads, seq, micro_batch; /* h, H, s, b */
  int32_t tp_size, tp_rank;
  int32_t ffn_mult;                         /* 4 */
  float dropout_hidden, dropout_attn, ln_eps;
  uint64_t seed;
  uint32_t layer_index;                     /* global layer id: keys weights and dropout sites */
} mt_layer_desc;

/* TP shard of parameter `param` (Megatron layout): global [rows, cols], this
 * rank's block starts at (row0, col0) with shape [shard_rows, shard_cols]. Pure. */
int mt_param_shard(const mt_layer_desc* d, int32_t param, int64_t global_shape[2], int64_t shard_origin[2],
                   int64_t shard_shape[2]);
/* Seed key of a parameter / synthetic stream: mix64(seed, fnv1a64(name) ^ (layer << 32 | micro_batch)). */
uint64_t mt_stream_key(uint64_t seed, const char* name, uint32_t layer, uint32_t micro_batch);
/* Dropout threshold used by the mask definition in include/curator/dropout.hpp. */
uint32_t mt_dropout_threshold16(double p);

/* ------------------------------------------------------------------ runtime */
typedef struct mt_ctx mt_ctx;
typedef struct mt_layer mt_layer;

int mt_ctx_create(int32_t device, mt_ctx** out);
int mt_ctx_destroy(mt_ctx* ctx);
/* NCCL bootstrap: rank 0 creates the id, the caller broadcasts the 128 bytes (e.g. over
 * torch.distributed's store), every rank calls mt_ctx_init_comm. The TP / PP / DP communicators
 * are split from the world communicator by curator::map_topology(nodes=1, gpus_per_node=world). */
int mt_nccl_unique_id(unsigned char out[128]);
int mt_ctx_init_comm(mt_ctx* ctx, const unsigned char id[128], int32_t world_size, int32_t rank,
                     const mt_parallel_config* par);
/* Bounded wait for the work queued on `stream` (use it instead of a plain stream sync after the
 * asynchronous mt_stage_train_step_dev when peers are involved). Every cross-rank wait of the runtime
 * is bounded by MT_COMM_TIMEOUT_S (default 300 s): device-side spins of the fused / NVLS all-reduce
 * kernels raise the context's error flag, and this wait (also used by mt_stage_train_step) aborts
 * the NCCL communicators on the deadline, a device timeout or an NCCL async error and returns 2. */
int mt_ctx_wait(mt_ctx* ctx, void* stream);
/* 0 = healthy, 1 = a device-side peer wait timed out, 2 = the host aborted the iteration,
 * 3 = communicators aborted (the context can no longer communicate: destroy it). */
int mt_ctx_error(const mt_ctx* ctx, int32_t* state);
int mt_ctx_placement(const mt_ctx* ctx, mt_rank_placement* out);
/* Single-process measurement of ONE tensor-parallel shard (layers created with tp_size > 1): the
 * layers run their shard's kernels and skip the TP all-reduces. Compute-only numbers; the
 * collectives are measured in real multi-GPU runs. Rejected when the context has a world > 1. */
int mt_ctx_shard_only(mt_ctx* ctx, int32_t enable);
/* Megatron sequence parallelism for TP > 1 (also MT_SEQ_PARALLEL=1 at mt_ctx_init_comm): layer
 * inputs / outputs (and stage inputs, targets, PP transfers) are this TP rank's token rows
 * [r * b*s/TP, (r+1) * b*s/TP); LayerNorm / bias-dropout-residual run on those rows only; the TP
 * all-reduces become reduce-scatter + all-gather. The TP-replicated parameters' gradients are partial
 * until mt_layer_finish_grads (the stage driver calls it). Set before creating layers. */
int mt_ctx_set_sequence_parallel(mt_ctx* ctx, int32_t enable);
/* Diagnostic (fused TP all-reduce contexts): time one NVLS all-reduce (multimem.ld_reduce + st) of
 * `elems` bf16 of the symmetric row-parallel buffer with `ctas` x 1024 threads, contiguous shares or
 * the GEMM's 128 x 256 unit pattern of a row-major [*, ld] matrix. Collective over the TP group. */
int mt_ctx_nvls_probe(mt_ctx* ctx, int64_t elems, int64_t ld, int32_t strided, int32_t ctas, int32_t iters,
                      double* us_per_iter);
/* Per-GEMM CUDA-event timing of every tcgen05 GEMM the context's layers launch (stream-ordered
 * events around each launch). _read synchronises, returns the summed kernel time, summed
 * algorithmic FLOPs and launch count since enabling / the last read, and resets. */
int mt_ctx_gemm_timing(mt_ctx* ctx, int32_t enable);
/* Per-op timing of the layers' forward/backward (stream-ordered event marks between ops; adds
 * ~40 event records per layer call). _read renders "op total_ms count" lines (NUL-terminated). */
int mt_ctx_op_timing(mt_ctx* ctx, int32_t enable);
int mt_ctx_op_timing_read(mt_ctx* ctx, char* out, int64_t cap, int64_t* len);
int mt_ctx_gemm_timing_read(mt_ctx* ctx, double* total_ms, double* total_flops, int64_t* launches);

int mt_layer_create(mt_ctx* ctx, const mt_layer_desc* d, mt_layer** out);
int mt_layer_destroy(mt_layer* l);
/* On-device seeded init of this rank's shard (weights ~ N(0, sqrt(1/(3h))), biases and LN beta
 * ~ N(0, 0.02), LN gamma ~ 1 + N(0, 0.02)); identical global tensors for every TP degree. */
int mt_layer_init_params(mt_layer* l, void* stream);
/* Copy this rank's shard out of a full (global, row-major, bf16) host tensor. */
int mt_layer_set_param(mt_layer* l, int32_t param, const void* host_global_bf16);
/* Read back this rank's bf16 parameter shard (shard_shape elements, raw bf16 bits). */
int mt_layer_get_param(mt_layer* l, int32_t param, void* host_shard_bf16);
/* Read back this rank's fp32 gradient shard (shard_shape elements). */
int mt_layer_get_grad(mt_layer* l, int32_t param, float* host_shard);
int mt_layer_zero_grads(mt_layer* l, void* stream);
/* Forward of one microbatch: x, y device bf16 [b*s, h]. x must stay valid until the matching
 * backward (it is the LayerNorm-1 input the backward re-reads). Activations are saved per
 * microbatch id. */
int mt_layer_forward(mt_layer* l, const void* x, void* y, uint32_t micro_batch, void* stream);
/* Backward of one microbatch (frees its saved activations): dy -> dx (device bf16 [b*s, h]);
 * parameter gradients accumulate in fp32. */
int mt_layer_backward(mt_layer* l, const void* dy, void* dx, uint32_t micro_batch, void* stream);
/* Activation recompute (full-layer checkpointing): the forward keeps only the layer
 * input; the backward re-runs the forward (identical dropout masks) before differentiating, so the
 * executed FLOPs follow the reference cost model's recompute-inclusive 96 coefficient
 * (proj/src/planner.cpp:52-54). Only while no microbatch is in flight. */
int mt_layer_set_recompute(mt_layer* l, int32_t enable);
/* Sequence parallel: TP all-reduce of the replicated parameters' gradient partials (collective over
 * the TP group; call once after the last backward of an iteration; no-op otherwise). */
int mt_layer_finish_grads(mt_layer* l, void* stream);
/* Training step whose dropout masks the next forwards draw: every dropout site seeds from
 * curator::step_seed(desc.seed, step) (= desc.seed at step 0), so masks differ across iterations; a
 * backward replays the masks of its own forward. The stage driver sets it each iteration. */
int mt_layer_set_step(mt_layer* l, uint64_t step);
/* Parity inspection: copy the dropout keep bits the forward of microbatch `mb` saved for its backward
 * (the microbatch must have activations in flight, i.e. forward done, backward not yet). which = 0:
 * attention dropout, uint32 words [b][heads/t][s][s/32], bit c % 32 of word c / 32 = score (row, c)
 * kept — written for the causal 128-column blocks only (fused attention); which = 1 / 2: the hidden
 * dropout after the attention-out / MLP-out projection, bytes [b*s][h/8], bit j of byte v = element
 * 8 v + j kept. *bytes_out = bytes copied; status 1 when that mask was not saved (no dropout, the
 * unfused attention path, activation recompute, or MT_HIDDEN_KEEP=0). Synchronises the device. */
int mt_layer_dropout_keep_bits(mt_layer* l, uint32_t mb, int32_t which, void* host_out, int64_t capacity,
                               int64_t* bytes_out);
/* Kernel launches one forward / backward issues (for the bench's gpu_launches claim). */
int mt_layer_launch_counts(const mt_layer* l, int32_t* fwd, int32_t* bwd);
/* Device pointer to the flat fp32 gradient buffer of the layer and its element count. */
int mt_layer_grad_buffer(mt_layer* l, float** ptr, int64_t* n);

/* loss += sum 0.5 (y - t)^2 / n and dy = (y - t) / n over n bf16 elements. */
int mt_mse_loss(const void* y, const void* t, void* dy, float* loss_dev, int64_t n, void* stream);
/* out[i] = bf16(mean + std * normal_at(key, i)), i < n. */
int mt_fill_normal(void* out, int64_t n, uint64_t key, float mean, float std, void* stream);

/* Collectives on the context's groups (device buffers, stream-ordered). */
int mt_tp_allreduce_bf16(mt_ctx* ctx, void* buf, int64_t n, void* stream);
int mt_dp_allreduce_f32(mt_ctx* ctx, float* buf, int64_t n, int32_t average, void* stream);
int mt_pp_send_bf16(mt_ctx* ctx, const void* buf, int64_t n, int32_t peer_stage, void* stream);
int mt_pp_recv_bf16(mt_ctx* ctx, void* buf, int64_t n, int32_t peer_stage, void* stream);

/* ------------------------------------------------------------------ optimizer */
/* AdamW + global gradient-norm clipping with the reference recipe (curator::TrainingRecipe,
 * planner.hpp:39-53) and learning rate curator::lr_at(tokens_seen) (planner.cpp:59-70) when lr < 0. */
typedef struct mt_adam_desc {
  float lr;              /* < 0: lr_at(tokens_seen) */
  double tokens_seen;
  float beta1, beta2, eps, weight_decay, grad_clip;  /* grad_clip <= 0 disables clipping */
  int64_t step;          /* 1-based step count (bias correction) */
} mt_adam_desc;
int mt_adam_defaults(mt_adam_desc* out);  /* recipe constants, lr = -1, step = 1 */
/* One layer on its own (no collectives): norm over this layer's gradients only. */
int mt_layer_adam_step(mt_layer* l, const mt_adam_desc* d, float* grad_norm_out, void* stream);
/* Read back the optimizer state of a parameter shard (fp32, shard_shape elements each; NULL skips). */
int mt_layer_get_optimizer_state(mt_layer* l, int32_t param, float* master, float* m, float* v);

/* ------------------------------------------------------------------ vocab */
/* Vocab-parallel word embedding (+ replicated learned position embedding, embedding dropout), final
 * LayerNorm and tied LM head with vocab-parallel cross-entropy (Megatron). The table is padded to a
 * multiple of 128 * TP rows; rank r owns rows [r * V_pad / TP, (r + 1) * V_pad / TP). */
typedef struct mt_vocab mt_vocab;
typedef struct mt_vocab_desc {
  int32_t vocab, hidden, seq, micro_batch, tp_size, tp_rank;
  float dropout, ln_eps;
  uint64_t seed;
} mt_vocab_desc;
int mt_vocab_create(mt_ctx* ctx, const mt_vocab_desc* d, mt_vocab** out);
int mt_vocab_destroy(mt_vocab* v);
int mt_vocab_padded(const mt_vocab* v, int64_t* vocab_padded, int64_t* slice_begin, int64_t* slice_rows);
/* param 0: word embedding [V_pad, h] (global bf16, this rank's rows are copied), 1: position [seq, h],
 * 2: final-LN gamma [h], 3: final-LN beta [h]. Gradients are fp32 of this rank's shard. */
int mt_vocab_set_param(mt_vocab* v, int32_t param, const void* host_global_bf16);
int mt_vocab_get_grad(mt_vocab* v, int32_t param, float* host);
/* This rank's shard of a parameter (bf16; word: [slice_rows, h]). */
int mt_vocab_get_param(mt_vocab* v, int32_t param, void* host_bf16);
int mt_vocab_zero_grads(mt_vocab* v, void* stream);
/* x (device bf16 [b*s, h]) = dropout(E[tokens] + P[pos]); tokens device int32 [b*s]. */
int mt_vocab_embed_forward(mt_vocab* v, const int32_t* tokens, void* x, uint32_t micro_batch, void* stream);
/* Training step keying the embedding-dropout masks (as mt_layer_set_step). */
int mt_vocab_set_step(mt_vocab* v, uint64_t step);
/* Multiplier of mt_vocab_head_loss's loss and gradient (default 1; the stage sets 1 / microbatches so
 * the iteration's loss is the batch mean). */
int mt_vocab_set_loss_scale(mt_vocab* v, float scale);
/* scatter-add of the embedding gradient (dx = gradient w.r.t. the embedding output). */
int mt_vocab_embed_backward(mt_vocab* v, const int32_t* tokens, const void* dx, uint32_t micro_batch, void* stream);
/* loss_dev += mean cross-entropy of LN_f(y) E^T against targets; dy = d loss / d y (forward+backward). */
int mt_vocab_head_loss(mt_vocab* v, const void* y, const int32_t* targets, void* dy, float* loss_dev, void* stream);

/* ------------------------------------------------------------------ pipeline stage (1F1B driver) */
typedef struct mt_stage mt_stage;
typedef struct mt_stage_desc {
  mt_layer_desc layer;          /* template: layer_index is filled per layer; tp fields from ctx */
  int32_t layers;               /* total transformer layers of the model (split evenly over PP) */
  int32_t micro_batches;        /* MB per iteration per DP replica */
} mt_stage_desc;

int mt_stage_create(mt_ctx* ctx, const mt_stage_desc* d, mt_stage** out);
int mt_stage_destroy(mt_stage* st);
int mt_stage_layer(mt_stage* st, int32_t i, mt_layer** out);
/* One training iteration of this rank: zero grads, 1F1B over MB microbatches (first stage reads
 * inputs_host[mb] — host bf16 [b*s*h] per microbatch, copied in-stream; last stage computes the
 * synthetic MSE loss against targets_host), PP send/recv, TP all-reduces inside the layers, then
 * the DP gradient all-reduce (mean). The loss is the batch mean — each microbatch's mean loss / MB
 * (Megatron's convention; gradients scale alike) — DP-averaged; *loss_out holds it on the last stage,
 * else 0. Host buffers should be pinned. If inputs_host is NULL the stage
 * generates inputs/targets on device from the seed (no host traffic). */
int mt_stage_train_step(mt_stage* st, const void* inputs_host, const void* targets_host, float* loss_out,
                        void* stream);
/* Same iteration with device-resident inputs: inputs_dev / targets_dev are device bf16
 * [MB][b*s*h] (first / last stage; may be NULL on other stages); no host copies, no host sync.
 * The summed loss stays on device in *loss_dev (may be NULL). */
int mt_stage_train_step_dev(mt_stage* st, const void* inputs_dev, const void* targets_dev, float* loss_dev,
                            void* stream);
int mt_stage_launch_count(const mt_stage* st, int64_t* launches_per_step);
int mt_stage_set_recompute(mt_stage* st, int32_t enable);
/* Optimizer step of this rank's layers after mt_stage_train_step: the squared gradient norm is
 * summed over the model-parallel group (TP and PP; TP-replicated parameters counted once; DP
 * replicas already hold the averaged gradient), clipped to grad_clip, then fused AdamW. */
int mt_stage_optimizer_step(mt_stage* st, const mt_adam_desc* d, float* grad_norm_out, void* stream);
/* Attach the vocab module (not owned; must outlive the stage) so the stage trains a language model:
 * the first stage embeds int32 token ids, the last stage runs the tied LM head + cross-entropy
 * against int32 target ids. Inputs/targets of mt_stage_train_step(_dev) then become int32
 * [MB][b*s] token arrays. With PP > 1 the word-embedding gradient is all-reduced between the first
 * and the last stage (tied weights, Megatron); DP averages all vocab gradients; the optimizer step
 * covers the vocab parameters (word embedding counted once in the gradient norm). */
int mt_stage_attach_vocab(mt_stage* st, mt_vocab* v);
/* Training step of the next iteration (starts at 0, +1 per mt_stage_train_step[_dev]): the stage
 * passes it to its layers and vocab (mt_layer_set_step) so dropout masks change every iteration;
 * set it to resume a run or to replay an iteration bit-exactly. */
int mt_stage_set_step(mt_stage* st, uint64_t step);
int mt_stage_get_step(const mt_stage* st, uint64_t* step);
/* Microbatches of the next iterations (1 .. the micro_batches the stage was created with): a batch
 * ramp (curator::batch_size_at) changes the global batch, hence the microbatch count, at fixed b. */
int mt_stage_set_micro_batches(mt_stage* st, int32_t micro_batches);
/* Host<->device bytes this rank moved in its last mt_stage_train_step (with TP > 1 each rank of a
 * TP group copies only its 1/TP slice of the inputs / targets; the slices are all-gathered over
 * NVLink). */
int mt_stage_host_traffic(const mt_stage* st, int64_t* h2d_bytes, int64_t* d2h_bytes);

/* ------------------------------------------------------------------ data feed */
/* Dataset blending: curator::next_batch_composition (include/curator/blending.hpp) over n datasets.
 * normalize != 0 scales the weights to sum 1 first (curator::normalize_weights). */
typedef struct mt_blend mt_blend;
int mt_blend_create(int32_t n, const char* const* names, const double* weights, const uint64_t* available,
                    int32_t normalize, mt_blend** out);
int mt_blend_destroy(mt_blend* b);
int mt_blend_weights(const mt_blend* b, double* weights);
/* counts[n] of the next batch; credit / drawn (may be NULL) = the state after it. */
int mt_blend_next(mt_blend* b, uint64_t batch_size, uint64_t* counts, double* credit, uint64_t* drawn);
/* The reference blend stage (proj/src/pipeline.cpp:551-647): dataset i has doc_counts[i] documents
 * doc_ids[i][...] in corpus order; weights are normalised; `steps` batches of batch_size samples
 * (or batch_per_step[step] when non-NULL) are drawn and written to `path` as blend_manifest.jsonl
 * lines {"step":t,"dataset":"name","doc_id":id}. shuffle != 0 draws each dataset in the seeded
 * order of stage_seed (= mix64(config seed, fnv1a64("blend")) in the reference pipeline). */
int mt_blend_manifest(int32_t n, const char* const* names, const double* weights, const uint64_t* const* doc_ids,
                      const uint64_t* doc_counts, uint64_t steps, uint64_t batch_size,
                      const uint64_t* batch_per_step, int32_t shuffle, uint64_t stage_seed, const char* path);

/* Token feed over a blend manifest: step t's lines are its global batch G_t (file order); DP rank r
 * takes samples [r G/DP, (r+1) G/DP), split into G/(micro_batch DP) microbatches. Tokens of a
 * sample are the synthetic stream of its (dataset, doc_id) (mt_feed_doc_tokens): inputs = tokens
 * [0, seq), targets = tokens [1, seq]. */
typedef struct mt_feed mt_feed;
typedef struct mt_feed_desc {
  int32_t vocab, seq, micro_batch, data_parallel, dp_rank;
  uint64_t seed;
} mt_feed_desc;
int mt_feed_open(const char* manifest_path, const mt_feed_desc* d, mt_feed** out);
int mt_feed_destroy(mt_feed* f);
int mt_feed_steps(const mt_feed* f, int64_t* steps);
int mt_feed_dataset_name(const mt_feed* f, int32_t index, const char** name);
/* Global batch of a step and this rank's microbatch count (status 1 unless G % (b DP) == 0). */
int mt_feed_step_info(const mt_feed* f, int64_t step, int64_t* global_batch, int32_t* micro_batches);
int mt_feed_sample(const mt_feed* f, int64_t step, int64_t index, int32_t* dataset, uint64_t* doc_id);
/* This rank's inputs / targets of a step: int32 [micro_batches][micro_batch * seq] (either may be NULL). */
int mt_feed_fill(const mt_feed* f, int64_t step, int32_t* tokens, int32_t* targets, int32_t max_micro_batches);
int mt_feed_doc_tokens(uint64_t seed, const char* dataset, uint64_t doc_id, int32_t vocab, int64_t n, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
