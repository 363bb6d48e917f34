// Internal C++ runtime objects behind the C ABI (mtnlg.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "curator/planner.hpp"
#include "curator/schedule.hpp"
#include "mtnlg.h"
#include "mtnlg_gemm.h"

struct mt_layer;
struct mt_ctx;

namespace mt {
struct FusedAllReduce;  // tp_fused.cu
FusedAllReduce* fused_ar_create(mt_ctx* c);
void fused_ar_destroy(mt_ctx* c, FusedAllReduce* f);
mt_gemm_allreduce* fused_ar_begin(mt_ctx* c);
void fused_ar_end(mt_ctx* c, cudaStream_t st, void* d, int64_t ldd);
void fused_ar_prepare(mt_ctx* c, cudaStream_t st);
int fused_ar_gemm_ctas(mt_ctx* c);
void nvls_allreduce(mt_ctx* c, int64_t elems, cudaStream_t st, int which = 0);
int nvls_bwd_ctas(mt_ctx* c);
void op_mark(mt_ctx* c, cudaStream_t st, const char* label);  // runtime.cpp (op timing)

// Failed CUDA / NCCL call -> DataError-class status 2.
struct RuntimeFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check_cuda(cudaError_t e, const char* what);
void check_nccl(ncclResult_t r, const char* what);
// Bounded host wait for the work queued on `s` (the iteration's sync point): polls the stream, the
// NCCL communicators' async errors and the device error flag; on a peer timeout / NCCL error / the
// context's deadline it releases the device spins, aborts the communicators and throws
// RuntimeFailure (status 2). Replaces cudaStreamSynchronize on paths that wait for peers.
void wait_stream(mt_ctx* c, cudaStream_t s, const char* what);
void abort_comms(mt_ctx* c);

// Host watchdog of a multi-rank context: a thread that aborts the context's NCCL communicators when
// an armed API call (one that may block in NCCL — e.g. a lazily connected collective waiting for a
// peer that never calls it — or wait for peers' kernels) runs past the context's bound. The blocked
// NCCL call then returns an error and the API call returns status 2. Arming nests (depth counter).
struct Watchdog {
  std::thread thread;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  std::atomic<int64_t> deadline_ns{0};  // steady_clock time since epoch; 0 = disarmed
  int depth = 0;                        // nesting of armed calls (the context's own thread only)
};
void watchdog_start(mt_ctx* c);
void watchdog_stop(mt_ctx* c);
struct WatchdogArm {  // RAII: arms the context's watchdog for the duration of an API call
  mt_ctx* c;
  explicit WatchdogArm(mt_ctx* ctx);
  ~WatchdogArm();
};

// Device buffer owned by the runtime.
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n);
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(o.ptr), bytes(o.bytes) {
    o.ptr = nullptr;
    o.bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
  void ensure(size_t n);  // grow (contents discarded)
};

void ensure_optimizer_state(mt_layer* l, cudaStream_t s);
void layer_grad_sq(mt_layer* l, float* sq, cudaStream_t s);
void layer_adamw(mt_layer* l, const mt_adam_desc& d, float lr, const float* clip_coef, cudaStream_t s);
void clip_coefficient(const float* sq, float max_norm, float* out, cudaStream_t s);
void grad_sq_segment(const float* g, int64_t n, float* out, cudaStream_t s);
void adamw_segment(const float* g, float* m, float* v, float* master, void* w_bf16, int64_t n, const mt_adam_desc& d,
                   float lr, int decay, const float* clip, cudaStream_t s);
void bf16_to_f32(const void* w, float* out, int64_t n, cudaStream_t s);
// vocab module hooks for the stage driver (vocab.cu)
int64_t vocab_tokens(const mt_vocab* v);  // b*s
int64_t vocab_hidden(const mt_vocab* v);
int vocab_tp(const mt_vocab* v);
void vocab_zero_grads(mt_vocab* v, cudaStream_t s);
// first: word embedding counted in the norm (once per model-parallel group); pos/LN_f always
// (they are zero where unused); sq[0] sharded, sq[1] TP-replicated
void vocab_grad_sq(mt_vocab* v, bool count_word, float* sq, cudaStream_t s);
void vocab_adamw(mt_vocab* v, const mt_adam_desc& d, float lr, const float* clip, cudaStream_t s);
void vocab_allreduce_grads(mt_vocab* v, ncclComm_t comm, bool word_only, bool average, cudaStream_t s);

}  // namespace mt

struct mt_ctx {
  int device = 0;
  int world_size = 1, rank = 0;
  curator::ParallelConfig par;
  curator::RankPlacement place;
  ncclComm_t world = nullptr, tp = nullptr, pp = nullptr, dp = nullptr;
  ncclComm_t tp_side = nullptr;  // same TP group, CTA-capped: collectives overlapped with GEMMs
  ncclComm_t emb = nullptr;
  // TP > 1: the two [M, h] buffers the layers all-reduce over TP (row-parallel outputs in the forward,
  // LN-input gradients in the backward) can live in NCCL symmetric memory (ncclMemAlloc + window
  // registered on tp and tp_side), so NCCL runs its symmetric (NVLS / load-store) all-reduce kernels
  // on them (MT_TP_SYMMETRIC=1). Allocation and registration are collective over the TP group.
  struct SymBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    ncclWindow_t win_tp = nullptr, win_side = nullptr;
  } sym_h[2];
  // DP > 1: the gradient all-reduce of each layer is issued on dp_stream over a CTA-capped DP
  // communicator (dp_side) as soon as the layer's last backward finished, overlapping the backward of
  // the layers below it (MT_DP_OVERLAP=0 disables); GEMMs issued meanwhile are capped at gemm_cap CTAs
  ncclComm_t dp_side = nullptr;
  cudaStream_t dp_stream = nullptr;
  cudaEvent_t ev_dp_ready = nullptr, ev_dp_done = nullptr;
  bool dp_overlap = true;
  int gemm_cap = 0;
  // Megatron sequence parallelism (MT_SEQ_PARALLEL=1 / mt_ctx_set_sequence_parallel): with TP > 1 the
  // layer input/output and the LayerNorm / bias-dropout-residual work are split over the TP ranks by
  // token rows (rank r owns rows [r M/t, (r+1) M/t)); the all-reduces become reduce-scatter +
  // all-gather of the same volume, and the replicated [M, h] element-wise work shrinks by t.
  bool seq_parallel = false;
  bool tp_symmetric = false;
  // forward row-parallel GEMM + TP all-reduce fused in one kernel over NVLink SHARP (MT_TP_FUSED=1;
  // implies symmetric buffers); state in tp_fused.cu
  bool tp_fused = false;
  bool tp_nvls = false;  // forward row-parallel all-reduce by nvls_allreduce instead of NCCL (MT_TP_NVLS=1)
  // backward LN-input-gradient all-reduces by nvls_allreduce on the side stream (MT_TP_NVLS_BWD)
  bool tp_nvls_bwd = false;
  mt::FusedAllReduce* fused_ar = nullptr;  // PP > 1: first + last stage of the same (dp, tp): tied word-embedding grads
  // compute-only measurement of one TP shard on a single GPU: the layer skips its TP collectives
  // (mt_ctx_shard_only); never set in a real multi-GPU run
  bool shard_only = false;
  // scratch shared by all layers of this context (sized to the largest layer)
  mt::DeviceBuffer scratch_h[4];   // [M, h] bf16 temporaries
  mt::DeviceBuffer scratch_ffn;    // [M, ffn/t] bf16
  mt::DeviceBuffer scratch_ctx;    // [M, h/t] bf16
  mt::DeviceBuffer scratch_qkv;    // [M, 3h/t] bf16
  mt::DeviceBuffer scratch_attn;   // [heads/t, s, s] bf16
  mt::DeviceBuffer scratch_stats;  // [heads/t, s, s / bn] float2: score-block softmax statistics
  mt::DeviceBuffer scratch_dq;     // fused attention backward: fp32 dQ accumulator [heads/t, s, hd]
  mt::DeviceBuffer scratch_ws;     // fp32 column-reduction workspace
  mt::DeviceBuffer gemm_ws;        // split-K tail workspace (zeroed counters + partial tiles)
  mt::DeviceBuffer opt_scratch;    // optimizer: squared norms + {norm, clip coefficient}
  // side stream for TP collectives overlapped with independent GEMMs (backward: the all-reduce of
  // an LN-input gradient runs while the matching wgrad GEMM executes on SMs left free for NCCL)
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  int comm_sms = 16;  // SMs kept free for the collective during an overlapped GEMM
  // Hang safety. Every device-side cross-rank spin (fused / NVLS all-reduce kernels) is bounded by
  // timeout_ns and raises *err_dev (a host-mapped word, also readable as *err_host) when a peer never
  // arrives; the host-side waits of an iteration poll the stream with the same bound and, on expiry,
  // raise the flag (which releases the device spins) and abort the NCCL communicators (which
  // releases NCCL's kernels), so a dead or diverged rank surfaces as status 2 instead of a wedged GPU.
  // MT_COMM_TIMEOUT_S (default 300) sets the bound.
  uint32_t* err_host = nullptr;
  uint32_t* err_dev = nullptr;
  uint64_t timeout_ns = 300ull * 1000000000ull;
  std::atomic<bool> aborted{false};  // NCCL communicators were aborted: the context can no longer communicate
  std::mutex abort_mu;
  std::unique_ptr<mt::Watchdog> watchdog;  // world > 1 only
  // optional per-op timing (MT_OP_TIMING=1): stream-ordered marks between consecutive layer ops
  bool op_timing = false;
  std::vector<std::pair<const char*, cudaEvent_t>> marks;
  size_t marks_used = 0;
  std::map<std::string, std::pair<double, int>> op_acc;
  // optional per-GEMM CUDA-event timing (bench.py's live roofline measurement)
  bool gemm_timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<double> ev_flops;
};

struct mt_layer {
  mt_ctx* ctx = nullptr;
  mt_layer_desc d{};
  int64_t M = 0, h = 0, hl = 0, ffl = 0, qkvl = 0, heads_local = 0, head_dim = 0;
  curator::LayerShard shard;
  int64_t param_off[MT_P_COUNT] = {};  // element offsets into params / grads
  int64_t param_rows[MT_P_COUNT] = {}, param_cols[MT_P_COUNT] = {};
  int64_t param_total = 0;
  mt::DeviceBuffer params;  // bf16
  mt::DeviceBuffer grads;   // fp32
  struct Saved {
    const void* x = nullptr;
    uint64_t step = 0;  // training step of the forward (keys the dropout masks the backward replays)
    mt::DeviceBuffer ln1, qkv, S, P, lse, ctx, x1, ln2, pre, act, stats;  // stats: mean1,rstd1,mean2,rstd2
    mt::DeviceBuffer mask;      // fused attention: the forward's dropout keep bits [b][heads/t][s][s/32]
    bool mask_valid = false;    // the forward wrote `mask` (the backward reads it instead of re-hashing)
    // hidden dropout keep bytes of the two bias-dropout-residual sites (attention-out, MLP-out), one
    // byte per 8 elements [2][rows][h / 8], written by the forward, read by the backward's dropout'
    mt::DeviceBuffer hmask;
  };
  std::map<uint32_t, std::unique_ptr<Saved>> saved;
  bool recompute = false;           // activation recompute (full-layer checkpointing)
  // training step whose dropout masks the next forwards draw (curator::step_seed; set by the stage
  // driver each iteration, mt_layer_set_step)
  uint64_t step = 0;
  std::unique_ptr<Saved> work;      // recompute: the one set of intermediate buffers
  std::vector<std::unique_ptr<Saved>> free_slots;
  int fwd_launches = 0, bwd_launches = 0;
  // fused flash attention (attention_sm100.cu) instead of score GEMM + softmax + PV GEMM; S / P are
  // then never materialised (opt-in with MT_ATTN_FUSED=1; parity-tested, not yet the faster path)
  bool fused_attn = false;
  // Logically zero gradients: the next backward writes (=) instead of accumulating (+=), which
  // saves both the memset and the read half of the fp32 read-modify-write in the wgrad epilogues.
  bool grads_fresh = false;
  bool sp_partial = false;  // sequence parallel: replicated-param grads await mt_layer_finish_grads
  // Optional row-chunk gate on the layer input (set by the stage for the first layer when its input
  // streams in from the host): forward runs LN1 + the QKV GEMM chunk by chunk, calling
  // input_gate(k, stream) before chunk k so the copy of chunk k+1 overlaps the compute of chunk k.
  int input_chunks = 1;
  std::function<void(int, cudaStream_t)> input_gate;
  // optimizer state (created on the first optimizer step): fp32 master weights, Adam moments
  mt::DeviceBuffer opt_master, opt_m, opt_v;
  void* param_ptr(int p) const { return static_cast<uint16_t*>(params.ptr) + param_off[p]; }
  float* grad_ptr(int p) const { return grads.as<float>() + param_off[p]; }
};
