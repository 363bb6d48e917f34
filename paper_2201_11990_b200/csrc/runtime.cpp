// Tensor-sliced transformer layer runtime: context, NCCL groups, parameter shards, layer forward
// and backward (PAPER.md:133-150 restated), and their C ABI.
//
// Per layer and microbatch (M = b*s tokens, t = TP, local widths h/t, 3h/t, 4h/t):
//   forward   LN1 -> QKV GEMM(+bias) -> [S = QK^T/sqrt(d) -> causal softmax+dropout -> P V] per head
//             -> attn-out GEMM -> TP all-reduce -> bias+dropout+residual -> LN2
//             -> fc1 GEMM(+bias, GeLU) -> fc2 GEMM -> TP all-reduce -> bias+dropout+residual
//   backward  the transposed chain with dgrad GEMMs (MN-major weight operand), wgrad GEMMs
//             (both operands MN-major, fp32 accumulation in the epilogue), the GeLU derivative fused
//             into the fc2-dgrad epilogue, softmax backward, LayerNorm backward, bias-grad column
//             sums, and the TP all-reduce of the LN inputs' gradients ("f" operator).
#include "runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>

#include "curator/dropout.hpp"
#include "curator/errors.hpp"
#include "curator/hashing.hpp"
#include "kernels.cuh"

namespace mt {

namespace {
thread_local std::string g_last_error;
thread_local mt_ctx* tl_ctx = nullptr;  // context of the layer call in progress (GEMM timing)
}

void set_error(const std::string& e) { g_last_error = e; }
const char* last_error() { return g_last_error.c_str(); }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw RuntimeFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw RuntimeFailure(std::string(what) + ": " + ncclGetErrorString(r));
}

void abort_comms(mt_ctx* c) {
  std::lock_guard<std::mutex> lk(c->abort_mu);
  if (c->aborted) return;
  if (c->err_host) __atomic_store_n(c->err_host, 2u, __ATOMIC_SEQ_CST);  // 2 = host abort: device spins return
  c->aborted = true;
  for (ncclComm_t* cm : {&c->dp_side, &c->emb, &c->tp_side, &c->tp, &c->pp, &c->dp, &c->world})
    if (*cm) {
      ncclComm_t h = *cm;
      *cm = nullptr;
      ncclCommAbort(h);  // releases NCCL calls blocked on the host and NCCL kernels on the device
    }
}

void watchdog_start(mt_ctx* c) {
  if (c->watchdog) return;
  c->watchdog = std::make_unique<Watchdog>();
  Watchdog* w = c->watchdog.get();
  w->thread = std::thread([c, w] {
    std::unique_lock<std::mutex> lk(w->mu);
    while (!w->stop) {
      w->cv.wait_for(lk, std::chrono::milliseconds(50));
      const int64_t d = w->deadline_ns.load();
      if (d != 0 && std::chrono::steady_clock::now().time_since_epoch().count() > d) {
        w->deadline_ns = 0;
        lk.unlock();
        fprintf(stderr, "[mtnlg] rank %d: an API call exceeded the %.0f s communication bound; aborting the "
                        "context's NCCL communicators\n", c->rank, c->timeout_ns * 1e-9);
        abort_comms(c);
        lk.lock();
      }
    }
  });
}

void watchdog_stop(mt_ctx* c) {
  if (!c->watchdog) return;
  {
    std::lock_guard<std::mutex> lk(c->watchdog->mu);
    c->watchdog->stop = true;
  }
  c->watchdog->cv.notify_all();
  c->watchdog->thread.join();
  c->watchdog.reset();
}

WatchdogArm::WatchdogArm(mt_ctx* ctx) : c(ctx) {
  if (!c || !c->watchdog) return;
  if (c->watchdog->depth++ == 0)
    c->watchdog->deadline_ns = (std::chrono::steady_clock::now() + std::chrono::nanoseconds(c->timeout_ns) +
                                std::chrono::seconds(5))
                                   .time_since_epoch()
                                   .count();
}
WatchdogArm::~WatchdogArm() {
  if (!c || !c->watchdog) return;
  if (--c->watchdog->depth == 0) c->watchdog->deadline_ns = 0;
}

void wait_stream(mt_ctx* c, cudaStream_t s, const char* what) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  const auto deadline = t0 + std::chrono::nanoseconds(c->timeout_ns) + std::chrono::seconds(5);
  auto fail = [&](const std::string& why) {
    abort_comms(c);
    // the aborted NCCL kernels and the released device spins let the queued work drain
    const auto drain = clock::now() + std::chrono::seconds(60);
    while (cudaStreamQuery(s) == cudaErrorNotReady && clock::now() < drain)
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    throw RuntimeFailure(std::string(what) + ": " + why +
                         " (a peer rank is dead or diverged; the context's communicators were aborted)");
  };
  for (int polls = 0;; ++polls) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) check_cuda(e, what);
    if ((polls & 63) == 0) {
      if (c->err_host && __atomic_load_n(c->err_host, __ATOMIC_SEQ_CST) != 0)
        fail("device-side wait for a peer timed out");
      for (ncclComm_t cm : {c->world, c->tp, c->tp_side, c->pp, c->dp, c->dp_side, c->emb}) {
        ncclResult_t r = ncclSuccess;
        if (cm && ncclCommGetAsyncError(cm, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress)
          fail(std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
      }
      if (clock::now() > deadline) fail("timed out waiting for the iteration");
    }
    // spin-yield for the first second (an iteration is 2-300 ms: a sleeping poll would add its
    // wake-up latency to every step's end-to-end time), then sleep between polls
    if (clock::now() - t0 < std::chrono::seconds(1))
      std::this_thread::yield();
    else
      std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  if (c->err_host && __atomic_load_n(c->err_host, __ATOMIC_SEQ_CST) != 0)
    fail("device-side wait for a peer timed out");
}

DeviceBuffer::DeviceBuffer(size_t n) { ensure(n); }
DeviceBuffer::~DeviceBuffer() {
  if (ptr) cudaFree(ptr);
}
void DeviceBuffer::ensure(size_t n) {
  if (n <= bytes) return;
  if (ptr) check_cuda(cudaFree(ptr), "cudaFree");
  ptr = nullptr;
  bytes = 0;
  check_cuda(cudaMalloc(&ptr, n), "cudaMalloc");
  bytes = n;
}

// Runs `f`, mapping exceptions to the ABI's status codes.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return MT_OK;
  } catch (const curator::ConfigError& e) {
    set_error(e.what());
    return MT_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return MT_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_error(e.what());
    return MT_ERR_DATA;
  }
}

namespace {

// --------------------------------------------------------------------------- GEMM helper
struct Gemm {
  mt_gemm_args a{};
  Gemm(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn, void* D, int64_t ldd, int64_t m,
       int64_t n, int64_t k) {
    a.a = A;
    a.lda = lda;
    a.a_mn_major = a_mn;
    a.b = B;
    a.ldb = ldb;
    a.b_mn_major = b_mn;
    a.d = D;
    a.ldd = ldd;
    a.m = m;
    a.n = n;
    a.k = k;
    a.batch = 1;
    a.alpha = 1.f;
    a.epilogue = MT_EPI_STORE_BF16;
  }
  Gemm& epi(int e) {
    a.epilogue = e;
    return *this;
  }
  Gemm& bias(const void* b) {
    a.bias = b;
    return *this;
  }
  Gemm& aux(void* p, int64_t ld) {
    a.aux = p;
    a.ld_aux = ld;
    return *this;
  }
  Gemm& alpha(float v) {
    a.alpha = v;
    return *this;
  }
  Gemm& batched(int64_t b, int64_t abs, int64_t bbs, int64_t dbs) {
    a.batch = b;
    a.a_batch_stride = abs;
    a.b_batch_stride = bbs;
    a.d_batch_stride = dbs;
    return *this;
  }
  Gemm& causal(int c) {
    a.causal = c;
    return *this;
  }
  Gemm& max_ctas(int n) {
    a.max_ctas = n;
    return *this;
  }
  Gemm& allreduce(mt_gemm_allreduce* ar) {
    a.allreduce = ar;
    return *this;
  }
  // Algorithmic FLOPs of this call (causal contractions count the lower triangle only).
  double flops() const {
    double f = 2.0 * double(a.m) * double(a.n) * double(a.k) * double(a.batch);
    if (a.causal != MT_CAUSAL_NONE) f *= (double(a.m) + 1.0) / (2.0 * double(a.m));
    return f;
  }
  void run(cudaStream_t s, int& launches) {
    mt_ctx* c = tl_ctx;
    const bool timed = c && c->gemm_timing;
    if (timed) {
      while (c->ev_pool.size() < c->ev_used + 2) {
        cudaEvent_t e;
        check_cuda(cudaEventCreate(&e), "cudaEventCreate");
        c->ev_pool.push_back(e);
      }
      check_cuda(cudaEventRecord(c->ev_pool[c->ev_used], s), "cudaEventRecord");
    }
    if (c && c->gemm_cap > 0) a.max_ctas = a.max_ctas > 0 ? std::min(a.max_ctas, c->gemm_cap) : c->gemm_cap;
    if (c && c->gemm_ws.ptr) {
      a.workspace = c->gemm_ws.ptr;
      a.workspace_bytes = static_cast<int64_t>(c->gemm_ws.bytes);
    }
    const int rc = mt_gemm(&a, s);
    if (rc == 1) throw std::invalid_argument("mt_gemm: invalid arguments");
    if (rc != 0) throw RuntimeFailure(std::string("mt_gemm: ") + cudaGetErrorString(cudaGetLastError()));
    if (timed) {
      check_cuda(cudaEventRecord(c->ev_pool[c->ev_used + 1], s), "cudaEventRecord");
      c->ev_used += 2;
      c->ev_flops.push_back(flops());
    }
    ++launches;
  }
};

uint64_t key_of(uint64_t seed, const char* name, uint32_t layer, uint32_t mb) {
  return curator::site_seed(seed, name, layer, mb);
}

const char* kParamNames[MT_P_COUNT] = {"ln1.gamma", "ln1.beta", "qkv.weight", "qkv.bias", "proj.weight", "proj.bias",
                                       "ln2.gamma", "ln2.beta", "fc1.weight", "fc1.bias", "fc2.weight", "fc2.bias"};

struct ShardInfo {
  int64_t grows, gcols, r0, c0, rows, cols;
};

ShardInfo shard_info(const mt_layer_desc& d, int p) {
  const auto sh = curator::layer_shard(d.hidden, d.heads, d.ffn_mult, d.tp_size, d.tp_rank);
  const int64_t h = d.hidden, ff = int64_t{d.ffn_mult} * d.hidden;
  switch (p) {
    case MT_P_LN1_GAMMA:
    case MT_P_LN1_BETA:
    case MT_P_LN2_GAMMA:
    case MT_P_LN2_BETA:
    case MT_P_PROJ_B:
    case MT_P_FC2_B:
      return {1, h, 0, 0, 1, h};
    case MT_P_QKV_W:
      return {3 * h, h, sh.qkv_rows.begin, 0, sh.qkv_rows.size(), h};
    case MT_P_QKV_B:
      return {1, 3 * h, 0, sh.qkv_rows.begin, 1, sh.qkv_rows.size()};
    case MT_P_PROJ_W:
      return {h, h, 0, sh.proj_cols.begin, h, sh.proj_cols.size()};
    case MT_P_FC1_W:
      return {ff, h, sh.fc1_rows.begin, 0, sh.fc1_rows.size(), h};
    case MT_P_FC1_B:
      return {1, ff, 0, sh.fc1_rows.begin, 1, sh.fc1_rows.size()};
    case MT_P_FC2_W:
      return {h, ff, 0, sh.fc2_cols.begin, h, sh.fc2_cols.size()};
    default:
      throw std::invalid_argument("unknown parameter id");
  }
}

void validate_desc(const mt_layer_desc& d) {
  if (d.hidden <= 0 || d.heads <= 0 || d.seq <= 0 || d.micro_batch <= 0 || d.ffn_mult <= 0)
    throw std::invalid_argument("layer dimensions must be positive");
  if (d.hidden % 64 != 0) throw std::invalid_argument("hidden must be a multiple of 64");
  if (d.seq % 64 != 0) throw std::invalid_argument("sequence must be a multiple of 64");
  if ((d.hidden / d.heads) % 16 != 0) throw std::invalid_argument("head dim must be a multiple of 16");
  if (d.dropout_hidden < 0 || d.dropout_hidden >= 1 || d.dropout_attn < 0 || d.dropout_attn >= 1)
    throw std::invalid_argument("dropout must be in [0, 1)");
  (void)curator::layer_shard(d.hidden, d.heads, d.ffn_mult, d.tp_size, d.tp_rank);
  if ((int64_t{d.hidden} / d.tp_size) % 8 != 0) throw std::invalid_argument("h / TP must be a multiple of 8");
}

// Collective over the TP group (every rank reaches the same ensure calls in the same order).
void release_symmetric(mt_ctx* c, mt_ctx::SymBuffer& sb) {
  if (!sb.ptr) return;
  if (sb.win_side && c->tp_side) ncclCommWindowDeregister(c->tp_side, sb.win_side);
  if (sb.win_tp && c->tp) ncclCommWindowDeregister(c->tp, sb.win_tp);
  ncclMemFree(sb.ptr);
  sb = mt_ctx::SymBuffer{};
}
void ensure_symmetric(mt_ctx* c, mt_ctx::SymBuffer& sb, size_t bytes) {
  bytes = (bytes + 4095) / 4096 * 4096;
  if (bytes <= sb.bytes) return;
  check_cuda(cudaDeviceSynchronize(), "sync");
  release_symmetric(c, sb);
  check_nccl(ncclMemAlloc(&sb.ptr, bytes), "ncclMemAlloc");
  sb.bytes = bytes;
  check_nccl(ncclCommWindowRegister(c->tp, sb.ptr, bytes, &sb.win_tp, NCCL_WIN_COLL_SYMMETRIC),
             "ncclCommWindowRegister(tp)");
  check_nccl(ncclCommWindowRegister(c->tp_side, sb.ptr, bytes, &sb.win_side, NCCL_WIN_COLL_SYMMETRIC),
             "ncclCommWindowRegister(tp_side)");
}
// The [M, h] buffer i (0: row-parallel output / its gradient, 1: LN-input gradient) that the layers
// all-reduce over TP: symmetric memory when enabled and allocated, else the plain scratch.
void* tp_buffer(mt_ctx* c, int i) { return c->sym_h[i].ptr ? c->sym_h[i].ptr : c->scratch_h[i].ptr; }

}  // namespace
}  // namespace mt

using namespace mt;

// Materialise logically-zero gradients before anyone reads the buffer.
static void settle_fresh_grads(mt_layer* l, cudaStream_t s) {
  if (!l->grads_fresh) return;
  check_cuda(cudaMemsetAsync(l->grads.ptr, 0, l->param_total * 4, s), "cudaMemsetAsync");
  l->grads_fresh = false;
}


// =========================================================================== context & comm
extern "C" const char* mt_last_error(void) { return mt::last_error(); }
extern "C" const char* mt_version(void) { return "mtnlg-b200 0.1 (sm_100a)"; }

extern "C" int mt_ctx_create(int32_t device, mt_ctx** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null out");
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new mt_ctx();
    c->device = device;
    if (const char* e = getenv("MT_COMM_TIMEOUT_S")) {
      const double sec = atof(e);
      if (sec > 0) c->timeout_ns = static_cast<uint64_t>(sec * 1e9);
    }
    check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(uint32_t), cudaHostAllocMapped),
               "cudaHostAlloc(error flag)");
    *c->err_host = 0;
    check_cuda(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0),
               "cudaHostGetDevicePointer(error flag)");
    c->gemm_ws.ensure(MT_GEMM_WORKSPACE_BYTES);
    check_cuda(cudaMemset(c->gemm_ws.ptr, 0, MT_GEMM_WORKSPACE_BYTES), "cudaMemset(gemm workspace)");
    *out = c;
  });
}

extern "C" int mt_ctx_destroy(mt_ctx* c) {
  return guarded([&] {
    if (!c) return;
    watchdog_stop(c);
    if (c->fused_ar) fused_ar_destroy(c, c->fused_ar);
    c->fused_ar = nullptr;
    for (auto& sb : c->sym_h) release_symmetric(c, sb);
    if (c->dp_stream) cudaStreamDestroy(c->dp_stream);
    if (c->ev_dp_ready) cudaEventDestroy(c->ev_dp_ready);
    if (c->ev_dp_done) cudaEventDestroy(c->ev_dp_done);
    for (ncclComm_t* cm : {&c->dp_side, &c->emb, &c->tp_side, &c->tp, &c->pp, &c->dp, &c->world})
      if (*cm) ncclCommDestroy(*cm);  // aborted communicators were already released (nullptr)
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (auto& m : c->marks) cudaEventDestroy(m.second);
    if (c->comm) cudaStreamDestroy(c->comm);
    if (c->ev_ready) cudaEventDestroy(c->ev_ready);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    if (c->err_host) cudaFreeHost(c->err_host);
    delete c;
  });
}

extern "C" int mt_nccl_unique_id(unsigned char out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    check_nccl(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
  });
}

extern "C" int mt_ctx_init_comm(mt_ctx* c, const unsigned char id_bytes[128], int32_t world_size, int32_t rank,
                                const mt_parallel_config* par) {
  return guarded([&] {
    if (!c || !par) throw std::invalid_argument("null argument");
    curator::ClusterTopology topo;
    topo.nodes = 1;
    topo.gpus_per_node = world_size;
    curator::ParallelConfig p;
    p.tensor = par->tensor;
    p.pipeline = par->pipeline;
    p.data = par->data;
    p.batch = par->batch;
    p.micro_batches = par->micro_batches;
    const auto ranks = curator::map_topology(topo, p);  // throws invalid_argument on bad layouts
    if (rank < 0 || rank >= world_size) throw std::invalid_argument("rank out of range");
    c->world_size = world_size;
    c->rank = rank;
    c->par = p;
    c->place = ranks[rank];
    check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
    if (world_size == 1) return;
    watchdog_start(c);
    WatchdogArm arm(c);  // communicator creation also waits for every peer
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, 128);
    check_nccl(ncclCommInitRank(&c->world, world_size, id, rank), "ncclCommInitRank");
    const auto& me = c->place;
    // TP group: same (dp, pp); PP group: same (dp, tp); DP group: same (pp, tp).
    const int tp_color = me.pipeline * p.data + me.data;
    const int pp_color = me.data * p.tensor + me.tensor;
    const int dp_color = me.pipeline * p.tensor + me.tensor;
    // Two communicators over the TP group: `tp` (all channels) for the critical-path forward
    // all-reduces, `tp_side` capped at comm_sms CTAs for the backward all-reduces that run beside a
    // wgrad GEMM launched on the remaining SMs.
    check_nccl(ncclCommSplit(c->world, tp_color, me.tensor, &c->tp, nullptr), "ncclCommSplit(tp)");
    if (const char* e = getenv("MT_COMM_SMS")) c->comm_sms = atoi(e);
    ncclConfig_t side_cfg = NCCL_CONFIG_INITIALIZER;
    side_cfg.maxCTAs = std::max(1, c->comm_sms);
    side_cfg.minCTAs = std::min(side_cfg.maxCTAs, 4);
    check_nccl(ncclCommSplit(c->world, tp_color, me.tensor, &c->tp_side, &side_cfg), "ncclCommSplit(tp_side)");
    check_nccl(ncclCommSplit(c->world, pp_color, me.pipeline, &c->pp, nullptr), "ncclCommSplit(pp)");
    check_nccl(ncclCommSplit(c->world, dp_color, me.data, &c->dp, nullptr), "ncclCommSplit(dp)");
    if (p.data > 1) {
      if (const char* e = getenv("MT_DP_OVERLAP")) c->dp_overlap = e[0] != '0';
      ncclConfig_t dcfg = NCCL_CONFIG_INITIALIZER;
      dcfg.maxCTAs = std::max(1, c->comm_sms);
      dcfg.minCTAs = std::min(dcfg.maxCTAs, 4);
      check_nccl(ncclCommSplit(c->world, dp_color, me.data, &c->dp_side, &dcfg), "ncclCommSplit(dp_side)");
      int lo = 0, hi = 0;
      check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
      check_cuda(cudaStreamCreateWithPriority(&c->dp_stream, cudaStreamNonBlocking, hi), "dp stream");
      check_cuda(cudaEventCreateWithFlags(&c->ev_dp_ready, cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreateWithFlags(&c->ev_dp_done, cudaEventDisableTiming), "event");
    }
    if (p.pipeline > 1) {  // tied word embeddings live on the first and the last stage
      const bool ends = me.pipeline == 0 || me.pipeline == p.pipeline - 1;
      check_nccl(ncclCommSplit(c->world, ends ? pp_color : NCCL_SPLIT_NOCOLOR, me.pipeline, &c->emb, nullptr),
                 "ncclCommSplit(emb)");
    }
    if (p.tensor > 1) {
      int lo = 0, hi = 0;
      check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
      check_cuda(cudaStreamCreateWithPriority(&c->comm, cudaStreamNonBlocking, hi), "comm stream");
      check_cuda(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming), "event");
      if (const char* e = getenv("MT_TP_SYMMETRIC")) c->tp_symmetric = e[0] == '1';
      if (const char* e = getenv("MT_SEQ_PARALLEL")) c->seq_parallel = e[0] == '1';
      // forward row-parallel GEMM + all-reduce fused (column-group NVLS reducer beside the GEMM): on by
      // default (GPT-3 layer: TP=2 9.25 vs 9.35 ms, TP=4 5.20 vs 5.31 ms against the standalone NVLS
      // kernel); MT_TP_FUSED=0/1 overrides
      c->tp_fused = p.tensor >= 2;
      if (const char* e = getenv("MT_TP_FUSED")) c->tp_fused = e[0] == '1';
      // NVLink SHARP all-reduce kernel for the forward row-parallel outputs: on by default from TP = 4
      // (GPT-3 layer at TP=4: 5.33 vs 5.38 ms/step; neutral at TP=2); MT_TP_NVLS=0/1 overrides
      c->tp_nvls = p.tensor >= 4;
      if (const char* e = getenv("MT_TP_NVLS")) c->tp_nvls = e[0] == '1';
      // backward all-reduces over the NVLS kernel: measured no faster than NCCL's (which already runs
      // its NVLS algorithm on the symmetric windows) beside the wgrad GEMM — TP=4 GPT-3 5.18 / 5.06
      // (8 CTAs) vs 5.06 ms, profiles/r02_nvls_bwd_ab.log — so opt-in (MT_TP_NVLS_BWD=1)
      c->tp_nvls_bwd = false;
      if (const char* e = getenv("MT_TP_NVLS_BWD")) c->tp_nvls_bwd = e[0] == '1';
      if (c->tp_fused || c->tp_nvls || c->tp_nvls_bwd) c->tp_symmetric = true;
    }
  });
}

extern "C" int mt_ctx_wait(mt_ctx* c, void* stream) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null ctx");
    WatchdogArm arm(c);
    wait_stream(c, (cudaStream_t)stream, "mt_ctx_wait");
  });
}

extern "C" int mt_ctx_error(const mt_ctx* c, int32_t* state) {
  return guarded([&] {
    if (!c || !state) throw std::invalid_argument("null argument");
    *state = c->aborted ? 3 : static_cast<int32_t>(__atomic_load_n(c->err_host, __ATOMIC_SEQ_CST));
  });
}

extern "C" int mt_ctx_gemm_timing(mt_ctx* c, int32_t enable) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null ctx");
    c->gemm_timing = enable != 0;
    c->ev_used = 0;
    c->ev_flops.clear();
  });
}

extern "C" int mt_ctx_gemm_timing_read(mt_ctx* c, double* total_ms, double* total_flops, int64_t* launches) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null ctx");
    check_cuda(cudaDeviceSynchronize(), "sync");
    double ms = 0, fl = 0;
    for (size_t i = 0; i + 1 < c->ev_used; i += 2) {
      float t = 0;
      check_cuda(cudaEventElapsedTime(&t, c->ev_pool[i], c->ev_pool[i + 1]), "cudaEventElapsedTime");
      ms += t;
    }
    for (double f : c->ev_flops) fl += f;
    if (total_ms) *total_ms = ms;
    if (total_flops) *total_flops = fl;
    if (launches) *launches = static_cast<int64_t>(c->ev_flops.size());
    c->ev_used = 0;
    c->ev_flops.clear();
  });
}

extern "C" int mt_ctx_op_timing(mt_ctx* c, int32_t enable) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null ctx");
    c->op_timing = enable != 0;
    c->marks_used = 0;
    c->op_acc.clear();
  });
}

// Accumulates the marks recorded so far into per-op totals, then renders "label total_ms count" lines.
extern "C" int mt_ctx_op_timing_read(mt_ctx* c, char* out, int64_t cap, int64_t* len) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null ctx");
    check_cuda(cudaDeviceSynchronize(), "sync");
    for (size_t i = 1; i < c->marks_used; ++i) {
      if (std::string(c->marks[i].first) == "begin") continue;
      float t = 0;
      check_cuda(cudaEventElapsedTime(&t, c->marks[i - 1].second, c->marks[i].second), "elapsed");
      auto& a = c->op_acc[c->marks[i].first];
      a.first += t;
      a.second += 1;
    }
    c->marks_used = 0;
    std::string text;
    for (const auto& [k, v] : c->op_acc)
      text += k + " " + std::to_string(v.first) + " " + std::to_string(v.second) + "\n";
    *len = static_cast<int64_t>(text.size());
    if (out && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, *len);
      std::memcpy(out, text.data(), static_cast<size_t>(k));
      out[k] = '\0';
    }
  });
}

extern "C" int mt_ctx_shard_only(mt_ctx* c, int32_t enable) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null ctx");
    if (enable && c->world_size > 1) throw std::invalid_argument("shard-only mode is for single-process runs");
    c->shard_only = enable != 0;
  });
}

extern "C" int mt_ctx_placement(const mt_ctx* c, mt_rank_placement* out) {
  return guarded([&] {
    if (!c || !out) throw std::invalid_argument("null argument");
    out->data = c->place.data;
    out->pipeline = c->place.pipeline;
    out->tensor = c->place.tensor;
    out->node = c->place.node;
    out->gpu = c->place.gpu;
  });
}

extern "C" int mt_tp_allreduce_bf16(mt_ctx* c, void* buf, int64_t n, void* stream) {
  return guarded([&] {
    if (c->par.tensor <= 1) return;
    check_nccl(ncclAllReduce(buf, buf, n, ncclBfloat16, ncclSum, c->tp, (cudaStream_t)stream), "ncclAllReduce(tp)");
  });
}

extern "C" int mt_dp_allreduce_f32(mt_ctx* c, float* buf, int64_t n, int32_t average, void* stream) {
  return guarded([&] {
    if (c->par.data <= 1) return;
    check_nccl(ncclAllReduce(buf, buf, n, ncclFloat32, average ? ncclAvg : ncclSum, c->dp, (cudaStream_t)stream),
               "ncclAllReduce(dp)");
  });
}

extern "C" int mt_pp_send_bf16(mt_ctx* c, const void* buf, int64_t n, int32_t peer, void* stream) {
  return guarded([&] {
    check_nccl(ncclSend(buf, n, ncclBfloat16, peer, c->pp, (cudaStream_t)stream), "ncclSend(pp)");
  });
}

extern "C" int mt_pp_recv_bf16(mt_ctx* c, void* buf, int64_t n, int32_t peer, void* stream) {
  return guarded([&] {
    check_nccl(ncclRecv(buf, n, ncclBfloat16, peer, c->pp, (cudaStream_t)stream), "ncclRecv(pp)");
  });
}

// =========================================================================== parameters
extern "C" int mt_param_shard(const mt_layer_desc* d, int32_t p, int64_t g[2], int64_t o[2], int64_t s[2]) {
  return guarded([&] {
    if (!d) throw std::invalid_argument("null desc");
    const ShardInfo si = shard_info(*d, p);
    g[0] = si.grows;
    g[1] = si.gcols;
    o[0] = si.r0;
    o[1] = si.c0;
    s[0] = si.rows;
    s[1] = si.cols;
  });
}

extern "C" uint64_t mt_stream_key(uint64_t seed, const char* name, uint32_t layer, uint32_t mb) {
  return key_of(seed, name, layer, mb);
}

extern "C" uint32_t mt_dropout_threshold16(double p) { return curator::dropout_threshold16(p); }

extern "C" int mt_layer_create(mt_ctx* c, const mt_layer_desc* d, mt_layer** out) {
  return guarded([&] {
    if (!c || !d || !out) throw std::invalid_argument("null argument");
    validate_desc(*d);
    check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
    auto l = std::make_unique<mt_layer>();
    l->ctx = c;
    l->d = *d;
    l->M = int64_t{d->micro_batch} * d->seq;
    l->h = d->hidden;
    l->hl = d->hidden / d->tp_size;
    l->ffl = int64_t{d->ffn_mult} * d->hidden / d->tp_size;
    l->qkvl = 3 * l->hl;
    l->heads_local = d->heads / d->tp_size;
    l->head_dim = d->hidden / d->heads;
    l->shard = curator::layer_shard(d->hidden, d->heads, d->ffn_mult, d->tp_size, d->tp_rank);
    {
      // Default: fused flash attention. head_dim <= 128: two-query-tile forward + one-kernel backward,
      // faster than score GEMM + causal softmax + PV GEMM (GPT-3 layer 18.0-18.3 vs 18.9 ms,
      // profiles/r02_attn_default_ab.log); head_dim 160 (MT-NLG): single-tile forward + dK/dV, dQ pair,
      // a tie in time with the unfused path (0.37 ms per TP=8 shard, profiles/r02_attn_hd160_ab.log)
      // without the [s x s] score / probability buffers. MT_ATTN_FUSED=0/1 forces.
      const char* e = getenv("MT_ATTN_FUSED");
      const int hd = static_cast<int>(l->head_dim);
      const bool want = e && e[0] ? e[0] == '1' : true;
      l->fused_attn = want && d->seq % 128 == 0 && (hd == 64 || hd == 128 || hd == 160);
    }
    int64_t off = 0;
    for (int p = 0; p < MT_P_COUNT; ++p) {
      const ShardInfo si = shard_info(*d, p);
      l->param_off[p] = off;
      l->param_rows[p] = si.rows;
      l->param_cols[p] = si.cols;
      off += (si.rows * si.cols + 63) / 64 * 64;  // 128-byte aligned bf16 slices
    }
    l->param_total = off;
    l->params.ensure(off * 2);
    l->grads.ensure(off * 4);
    check_cuda(cudaMemset(l->grads.ptr, 0, off * 4), "cudaMemset");
    // shared scratch
    const int64_t M = l->M;
    for (auto& b : c->scratch_h) b.ensure(M * l->h * 2);
    if (c->tp_symmetric && d->tp_size > 1 && c->tp && !c->shard_only) {
      for (auto& sb : c->sym_h) ensure_symmetric(c, sb, static_cast<size_t>(M * l->h * 2));
      if ((c->tp_fused || c->tp_nvls || c->tp_nvls_bwd) && !c->fused_ar) {
        // all TP ranks must agree on the all-reduce path: fall back to NCCL everywhere if any rank
        // cannot set up the multicast state
        int ok = 1;
        try {
          c->fused_ar = fused_ar_create(c);
        } catch (const std::exception& e) {
          ok = 0;
          fprintf(stderr, "[mtnlg] NVLS all-reduce unavailable (%s): using NCCL\n", e.what());
        }
        DeviceBuffer flag(sizeof(int));
        check_cuda(cudaMemcpy(flag.ptr, &ok, sizeof(int), cudaMemcpyHostToDevice), "H2D");
        check_nccl(ncclAllReduce(flag.ptr, flag.ptr, 1, ncclInt32, ncclMin, c->tp, nullptr), "ncclAllReduce(nvls ok)");
        check_cuda(cudaMemcpy(&ok, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
        if (!ok) {
          if (c->fused_ar) fused_ar_destroy(c, c->fused_ar);
          c->fused_ar = nullptr;
          c->tp_fused = c->tp_nvls = c->tp_nvls_bwd = false;
        }
      }
    }
    c->scratch_ffn.ensure(M * l->ffl * 2);
    c->scratch_ctx.ensure(M * l->hl * 2);
    c->scratch_qkv.ensure(M * l->qkvl * 2);
    c->scratch_attn.ensure(l->fused_attn ? l->heads_local * int64_t{d->seq} * 4
                                         : l->heads_local * int64_t{d->seq} * d->seq * 2);
    if (l->fused_attn) c->scratch_dq.ensure(l->heads_local * int64_t{d->seq} * l->head_dim * 4);  // fp32 dQ acc
    c->scratch_stats.ensure(l->heads_local * int64_t{d->seq} * ((d->seq + 127) / 128) * 8);
    size_t ws = 0;
    for (int64_t n : {l->h, l->ffl, l->qkvl}) ws = std::max(ws, mt::colsum_workspace_floats((int)M, (int)n));
    c->scratch_ws.ensure(ws * 4);
    *out = l.release();
  });
}

extern "C" int mt_layer_destroy(mt_layer* l) {
  return guarded([&] { delete l; });
}

extern "C" int mt_layer_init_params(mt_layer* l, void* stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    const double wstd = curator::weight_init_std(l->d.hidden);
    for (int p = 0; p < MT_P_COUNT; ++p) {
      const ShardInfo si = shard_info(l->d, p);
      const uint64_t key = key_of(l->d.seed, kParamNames[p], l->d.layer_index, 0);
      float mean = 0.f, std = 0.02f;
      if (p == MT_P_QKV_W || p == MT_P_PROJ_W || p == MT_P_FC1_W || p == MT_P_FC2_W) std = (float)wstd;
      if (p == MT_P_LN1_GAMMA || p == MT_P_LN2_GAMMA) mean = 1.f;
      mt::fill_normal(l->param_ptr(p), si.rows, si.cols, si.gcols, si.r0, si.c0, key, mean, std, s);
    }
    check_cuda(cudaGetLastError(), "fill_normal");
  });
}

extern "C" int mt_layer_set_param(mt_layer* l, int32_t p, const void* host_global) {
  return guarded([&] {
    const ShardInfo si = shard_info(l->d, p);
    const uint16_t* src = static_cast<const uint16_t*>(host_global) + si.r0 * si.gcols + si.c0;
    check_cuda(cudaMemcpy2D(l->param_ptr(p), si.cols * 2, src, si.gcols * 2, si.cols * 2, si.rows,
                            cudaMemcpyHostToDevice),
               "cudaMemcpy2D(param)");
  });
}

extern "C" int mt_layer_get_param(mt_layer* l, int32_t p, void* host) {
  return guarded([&] {
    if (p < 0 || p >= MT_P_COUNT) throw std::invalid_argument("unknown parameter id");
    check_cuda(cudaDeviceSynchronize(), "sync");
    check_cuda(cudaMemcpy(host, l->param_ptr(p), l->param_rows[p] * l->param_cols[p] * 2, cudaMemcpyDeviceToHost),
               "cudaMemcpy(param)");
  });
}

extern "C" int mt_layer_get_grad(mt_layer* l, int32_t p, float* host) {
  return guarded([&] {
    if (p < 0 || p >= MT_P_COUNT) throw std::invalid_argument("unknown parameter id");
    settle_fresh_grads(l, nullptr);
    check_cuda(cudaDeviceSynchronize(), "sync");
    check_cuda(cudaMemcpy(host, l->grad_ptr(p), l->param_rows[p] * l->param_cols[p] * 4, cudaMemcpyDeviceToHost),
               "cudaMemcpy(grad)");
  });
}

extern "C" int mt_layer_zero_grads(mt_layer* l, void* stream) {
  return guarded([&] {
    if (!l) throw std::invalid_argument("null layer");
    (void)stream;
    l->grads_fresh = true;  // the next backward stores instead of accumulating
  });
}

extern "C" int mt_layer_grad_buffer(mt_layer* l, float** ptr, int64_t* n) {
  return guarded([&] {
    settle_fresh_grads(l, nullptr);
    *ptr = l->grads.as<float>();
    *n = l->param_total;
  });
}

extern "C" int mt_layer_set_recompute(mt_layer* l, int32_t enable) {
  return guarded([&] {
    if (!l) throw std::invalid_argument("null layer");
    if (!l->saved.empty()) throw std::invalid_argument("cannot switch recompute with activations in flight");
    l->recompute = enable != 0;
    for (auto& f : l->free_slots) f.reset(new mt_layer::Saved());  // drop full-size slots
  });
}

extern "C" int mt_layer_set_step(mt_layer* l, uint64_t step) {
  return guarded([&] {
    if (!l) throw std::invalid_argument("null layer");
    l->step = step;
  });
}

namespace {
uint8_t* hidden_keep(mt_layer* l, mt_layer::Saved& sv, int i);  // defined with the forward below
}  // namespace

extern "C" int mt_layer_dropout_keep_bits(mt_layer* l, uint32_t mb, int32_t which, void* host_out, int64_t capacity,
                                          int64_t* bytes_out) {
  return guarded([&] {
    if (!l || !host_out || !bytes_out || which < 0 || which > 2) throw std::invalid_argument("bad argument");
    *bytes_out = 0;
    auto it = l->saved.find(mb);
    if (it == l->saved.end() || l->recompute) throw std::invalid_argument("no saved activations for this microbatch");
    mt_layer::Saved& sv = *it->second;
    const void* src = nullptr;
    int64_t n = 0;
    if (which == 0) {
      if (!l->fused_attn || !sv.mask_valid) throw std::invalid_argument("attention keep bits not saved");
      src = sv.mask.ptr;
      n = int64_t{l->d.micro_batch} * l->heads_local * l->d.seq * (l->d.seq / 32) * 4;
    } else {
      src = hidden_keep(l, sv, which - 1);
      if (!src) throw std::invalid_argument("hidden-dropout keep bytes not saved");
      n = l->M * (l->h / 8);
    }
    if (capacity < n) throw std::invalid_argument("host buffer too small");
    check_cuda(cudaSetDevice(l->ctx->device), "cudaSetDevice");
    check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    check_cuda(cudaMemcpy(host_out, src, static_cast<size_t>(n), cudaMemcpyDeviceToHost), "D2H keep bits");
    *bytes_out = n;
  });
}

extern "C" int mt_layer_launch_counts(const mt_layer* l, int32_t* f, int32_t* b) {
  return guarded([&] {
    *f = l->fwd_launches;
    *b = l->bwd_launches;
  });
}

// =========================================================================== forward
namespace {

// TP all-reduce of `buf` on the context's comm stream, ordered after the work already queued on
// `st`; returns the CTA cap for GEMMs that overlap it (0 when there is nothing to overlap).
int tp_allreduce_async(mt_ctx* c, void* buf, int64_t n, cudaStream_t st, const char* what) {
  check_cuda(cudaEventRecord(c->ev_ready, st), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(c->comm, c->ev_ready, 0), "cudaStreamWaitEvent");
  int sms = 0;
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device), "attr");
  if (c->fused_ar && c->tp_nvls_bwd && buf == c->sym_h[1].ptr) {
    // NVLink SHARP all-reduce kernel on the side stream (multimem.ld_reduce + multimem.st, bounded
    // cross-rank waits) instead of NCCL's ring/NVLS kernels
    nvls_allreduce(c, n, c->comm, 1);
    check_cuda(cudaEventRecord(c->ev_done, c->comm), "cudaEventRecord");
    return std::max(2, sms - nvls_bwd_ctas(c));
  }
  check_nccl(ncclAllReduce(buf, buf, n, ncclBfloat16, ncclSum, c->tp_side, c->comm), what);
  check_cuda(cudaEventRecord(c->ev_done, c->comm), "cudaEventRecord");
  return std::max(2, sms - c->comm_sms);
}
void tp_allreduce_join(mt_ctx* c, cudaStream_t st) {
  check_cuda(cudaStreamWaitEvent(st, c->ev_done, 0), "cudaStreamWaitEvent");
}

// Sequence parallelism: rows [rank * ms, (rank + 1) * ms) of a [M, h] buffer are this rank's.
template <class T>
T* rows_of(T* p, int64_t r0, int64_t h) {
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) + static_cast<uintptr_t>(r0 * h * 2));
}
void sp_allgather(mt_ctx* c, void* buf, int64_t slice_elems, cudaStream_t st) {
  check_nccl(ncclAllGather(static_cast<uint16_t*>(buf) + c->place.tensor * slice_elems, buf, slice_elems, ncclBfloat16,
                           c->tp, st),
             "ncclAllGather(sequence-parallel rows)");
}
void sp_reduce_scatter(mt_ctx* c, ncclComm_t comm, void* buf, int64_t slice_elems, cudaStream_t st) {
  check_nccl(ncclReduceScatter(buf, static_cast<uint16_t*>(buf) + c->place.tensor * slice_elems, slice_elems,
                               ncclBfloat16, ncclSum, comm, st),
             "ncclReduceScatter(sequence-parallel rows)");
}
// reduce-scatter on the side stream (overlapping an independent GEMM); returns that GEMM's CTA cap
int sp_reduce_scatter_async(mt_ctx* c, void* buf, int64_t slice_elems, cudaStream_t st) {
  check_cuda(cudaEventRecord(c->ev_ready, st), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(c->comm, c->ev_ready, 0), "cudaStreamWaitEvent");
  sp_reduce_scatter(c, c->tp_side, buf, slice_elems, c->comm);
  check_cuda(cudaEventRecord(c->ev_done, c->comm), "cudaEventRecord");
  int sms = 0;
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device), "attr");
  return std::max(2, sms - c->comm_sms);
}

// Stream-ordered mark for per-op timing; the time between consecutive marks is attributed to the
// op named by the later mark. No-op unless the context has op timing enabled.
void mark(mt_ctx* c, cudaStream_t st, const char* label) {
  if (!c->op_timing) return;
  if (c->marks_used == c->marks.size()) {
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    c->marks.push_back({label, e});
  }
  c->marks[c->marks_used].first = label;
  check_cuda(cudaEventRecord(c->marks[c->marks_used].second, st), "cudaEventRecord");
  ++c->marks_used;
}

}  // namespace
namespace mt {
void op_mark(mt_ctx* c, cudaStream_t st, const char* label) { mark(c, st, label); }
}  // namespace mt
namespace {

// Whether the layer performs its TP collectives (TP > 1 with a communicator); TP > 1 without one
// is only legal in shard-only (compute-only measurement) mode.
bool tp_collectives(const mt_ctx* c, const mt_layer_desc& d) {
  if (d.tp_size <= 1) return false;
  if (c->aborted) throw RuntimeFailure("the context's communicators were aborted after a peer failure");
  if (c->tp) return true;
  if (c->shard_only) return false;
  throw std::invalid_argument("TP > 1 needs mt_ctx_init_comm (or mt_ctx_shard_only for a compute-only shard run)");
}

// Row-parallel output block of the forward: z = in W^T (partial sums), TP all-reduce ("g"), then
// out = resid + dropout(z + bias) and optionally LayerNorm(out). With TP > 1 the all-reduce is fused
// into the GEMM (NVLink SHARP reducer beside it) when K is long enough to hide it, else an NVLS or
// NCCL all-reduce follows the GEMM.
struct LnOut {
  const void* gamma;
  const void* beta;
  void* y;
  float* mean;
  float* rstd;
  float eps;
};

struct SeqPar {
  bool on = false;
  int64_t ms = 0, r0 = 0;  // this rank's token rows [r0, r0 + ms)
};

template <class GemmFor>
void row_parallel_block(mt_ctx* c, bool tpc, const SeqPar& sp, int64_t M, int64_t h, int64_t k_dim, GemmFor gemm_rows,
                        void* z, const void* bias, const void* resid, void* out, uint64_t site, uint32_t th,
                        float scale, const LnOut* ln, cudaStream_t st, int& n, const char* gemm_label,
                        uint8_t* keep) {
  if (sp.on) {
    // sequence parallel: reduce-scatter the partial sums to this rank's rows, then the element-wise
    // epilogue on those rows only, and all-gather the LayerNorm output the next GEMM needs in full
    gemm_rows(0, M, 0, nullptr);
    mark(c, st, gemm_label);
    sp_reduce_scatter(c, c->tp, z, sp.ms * h, st);
    ++n;
    mark(c, st, "fwd.tp_reduce_scatter");
    n += bias_dropout_residual_ln(rows_of(z, sp.r0, h), bias, resid, out, ln ? ln->gamma : nullptr,
                                  ln ? ln->beta : nullptr, ln ? rows_of(ln->y, sp.r0, h) : nullptr,
                                  ln ? ln->mean : nullptr, ln ? ln->rstd : nullptr, (int)sp.ms, (int)h,
                                  ln ? ln->eps : 0.f, site, th, scale, static_cast<uint64_t>(sp.r0 * h), st, keep);
    mark(c, st, "fwd.bias_dropout_residual_ln");
    if (ln) {
      sp_allgather(c, ln->y, sp.ms * h, st);
      ++n;
      mark(c, st, "fwd.tp_allgather");
    }
    return;
  }
  auto row_ptr = [&](const void* p, int64_t r) {
    return static_cast<void*>(const_cast<uint16_t*>(static_cast<const uint16_t*>(p)) + r * h);
  };
  auto epilogue = [&](int64_t r0, int64_t nr) {
    n += bias_dropout_residual_ln(row_ptr(z, r0), bias, row_ptr(resid, r0), row_ptr(out, r0), ln ? ln->gamma : nullptr,
                             ln ? ln->beta : nullptr, ln ? row_ptr(ln->y, r0) : nullptr, ln ? ln->mean + r0 : nullptr,
                             ln ? ln->rstd + r0 : nullptr, (int)nr, (int)h, ln ? ln->eps : 0.f, site, th, scale,
                             static_cast<uint64_t>(r0 * h), st, keep ? keep + r0 * (h / 8) : nullptr);
  };
  if (!tpc) {
    gemm_rows(0, M, 0, nullptr);
    mark(c, st, gemm_label);
    epilogue(0, M);
    mark(c, st, "fwd.bias_dropout_residual_ln");
    return;
  }
  // fused GEMM + all-reduce when the GEMM is long enough to hide the reduction (K >= 4096); a short-K
  // GEMM (e.g. the attention-out projection at TP >= 4) is followed by the standalone NVLS kernel
  // instead (TP=4: proj 0.27 vs 0.32 ms fused)
  if (c->fused_ar && c->tp_fused && z == c->sym_h[0].ptr && M % c->par.tensor == 0 && k_dim >= 4096) {
    // one kernel: GEMM tiles + their all-reduce over NVLink SHARP from the epilogue warps
    mt_gemm_allreduce* ar = fused_ar_begin(c);
    fused_ar_prepare(c, st);
    check_cuda(cudaEventRecord(c->ev_ready, st), "cudaEventRecord");  // the reducer starts after this
    gemm_rows(0, M, fused_ar_gemm_ctas(c), ar);
    fused_ar_end(c, st, z, h);
    ++n;
    mark(c, st, gemm_label);
    epilogue(0, M);
    mark(c, st, "fwd.bias_dropout_residual_ln");
    return;
  }
  gemm_rows(0, M, 0, nullptr);
  mark(c, st, gemm_label);
  if (c->fused_ar && (c->tp_nvls || c->tp_fused) && z == c->sym_h[0].ptr) {
    nvls_allreduce(c, M * h, st);  // NVLink SHARP all-reduce kernel + counter wait
    n += 2;
  } else {
    check_nccl(ncclAllReduce(z, z, M * h, ncclBfloat16, ncclSum, c->tp, st), "ncclAllReduce(row-parallel out)");
    ++n;
  }
  mark(c, st, "fwd.tp_allreduce");
  epilogue(0, M);
  mark(c, st, "fwd.bias_dropout_residual_ln");
}

// The forward's hidden-dropout keep bytes feed the backward's dropout' (MT_HIDDEN_KEEP=0: the backward
// re-hashes the counter-based mask instead; same bits either way).
bool hidden_keep_enabled() {  // read per call so tests can switch it
  const char* e = getenv("MT_HIDDEN_KEEP");
  return !(e && e[0] == '0');
}

// Keep bytes of hidden-dropout site i (0: attention-out, 1: MLP-out) in the slot (nullptr: no dropout
// or no buffer; writer and reader then both fall back to the counter-based hash).
uint8_t* hidden_keep(mt_layer* l, mt_layer::Saved& sv, int i) {
  if (!(l->d.dropout_hidden > 0.f) || !sv.hmask.ptr || !hidden_keep_enabled()) return nullptr;
  return sv.hmask.as<uint8_t>() + i * l->M * (l->h / 8);
}

void ensure_slot_buffers(mt_layer* l, mt_layer::Saved& sv) {
  const int64_t M = l->M, b = l->d.micro_batch, s = l->d.seq, Hl = l->heads_local;
  sv.ln1.ensure(M * l->h * 2);
  sv.qkv.ensure(M * l->qkvl * 2);
  if (!l->fused_attn) {
    sv.S.ensure(b * Hl * s * s * 2);
    sv.P.ensure(b * Hl * s * s * 2);
  } else if (l->d.dropout_attn > 0.f) {
    sv.mask.ensure(b * Hl * s * (s / 32) * 4);
  }
  sv.lse.ensure(b * Hl * s * 4);
  sv.ctx.ensure(M * l->hl * 2);
  sv.x1.ensure(M * l->h * 2);
  sv.ln2.ensure(M * l->h * 2);
  sv.pre.ensure(M * l->ffl * 2);
  sv.act.ensure(M * l->ffl * 2);
  sv.stats.ensure(4 * M * 4);
  if (l->d.dropout_hidden > 0.f) sv.hmask.ensure(2 * M * (l->h / 8));
}

// Per-microbatch slot. With activation recompute the slot keeps only the layer
// input; the intermediate tensors live in one per-layer work slot that the backward refills by
// re-running the forward (same microbatch id -> identical dropout masks).
mt_layer::Saved& acquire_slot(mt_layer* l, uint32_t mb) {
  if (l->saved.count(mb)) throw std::invalid_argument("microbatch already has saved activations");
  std::unique_ptr<mt_layer::Saved> sv;
  if (!l->free_slots.empty()) {
    sv = std::move(l->free_slots.back());
    l->free_slots.pop_back();
  } else {
    sv = std::make_unique<mt_layer::Saved>();
  }
  if (!l->recompute) ensure_slot_buffers(l, *sv);
  auto& ref = *sv;
  l->saved[mb] = std::move(sv);
  return ref;
}

mt_layer::Saved& work_slot(mt_layer* l) {
  if (!l->work) l->work = std::make_unique<mt_layer::Saved>();
  ensure_slot_buffers(l, *l->work);
  return *l->work;
}

// `mseed` = curator::step_seed(desc seed, training step): the seed the dropout sites derive from.
void forward_into(mt_layer* l, const void* x, void* y, uint32_t mb, uint64_t mseed, cudaStream_t st,
                  mt_layer::Saved& sv);

void layer_forward(mt_layer* l, const void* x, void* y, uint32_t mb, cudaStream_t st) {
  auto& slot = acquire_slot(l, mb);
  slot.x = x;
  slot.step = l->step;
  forward_into(l, x, y, mb, curator::step_seed(l->d.seed, slot.step), st, l->recompute ? work_slot(l) : slot);
}

void forward_into(mt_layer* l, const void* x, void* y, uint32_t mb, uint64_t mseed, cudaStream_t st,
                  mt_layer::Saved& sv) {
  mt_ctx* c = l->ctx;
  tl_ctx = c;
  const mt_layer_desc& d = l->d;
  const int64_t M = l->M, h = l->h, hl = l->hl, ffl = l->ffl, ld3 = l->qkvl, s = d.seq, Hl = l->heads_local,
                hd = l->head_dim;
  const bool tpc = tp_collectives(c, d);
  SeqPar sp;
  sp.on = tpc && c->seq_parallel;
  sp.ms = sp.on ? M / d.tp_size : M;
  sp.r0 = sp.on ? int64_t{d.tp_rank} * sp.ms : 0;
  sv.x = x;
  float* mean1 = sv.stats.as<float>();
  float* rstd1 = mean1 + M;
  float* mean2 = rstd1 + M;
  float* rstd2 = mean2 + M;
  int n = 0;
  const float scale_h = 1.f / (1.f - d.dropout_hidden), scale_a = 1.f / (1.f - d.dropout_attn);
  const uint32_t th_h = curator::dropout_threshold16(d.dropout_hidden);
  const uint32_t th_a = curator::dropout_threshold16(d.dropout_attn);
  const uint64_t site_attn = key_of(mseed, "attn.probs", d.layer_index, mb);
  const uint64_t site_out1 = key_of(mseed, "attn.out", d.layer_index, mb);
  const uint64_t site_out2 = key_of(mseed, "mlp.out", d.layer_index, mb);
  void* z = tp_buffer(c, 0);
  mark(c, st, "begin");

  if (sp.on) {  // x holds this rank's rows: LN1 on them, then all-gather the LN1 output
    ln_fwd(x, l->param_ptr(MT_P_LN1_GAMMA), l->param_ptr(MT_P_LN1_BETA), rows_of(sv.ln1.ptr, sp.r0, h), mean1, rstd1,
           (int)sp.ms, (int)h, d.ln_eps, st);
    ++n;
    sp_allgather(c, sv.ln1.ptr, sp.ms * h, st);
    ++n;
    mark(c, st, "fwd.ln1");
  }
  // LN1 + QKV GEMM, by row chunks when the input arrives in chunks (input_gate)
  const int in_chunks = (!sp.on && l->input_gate && l->input_chunks > 1 && M % (int64_t{l->input_chunks} * 128) == 0)
                            ? l->input_chunks
                            : 1;
  const int64_t in_rows = M / in_chunks;
  for (int k = 0; k < in_chunks; ++k) {
    const int64_t r0 = k * in_rows;
    if (l->input_gate && !sp.on) l->input_gate(k, st);
    if (!sp.on) {
      ln_fwd(static_cast<const uint16_t*>(x) + r0 * h, l->param_ptr(MT_P_LN1_GAMMA), l->param_ptr(MT_P_LN1_BETA),
             sv.ln1.as<uint16_t>() + r0 * h, mean1 + r0, rstd1 + r0, (int)in_rows, (int)h, d.ln_eps, st);
      ++n;
      mark(c, st, "fwd.ln1");
    }
    Gemm(sv.ln1.as<uint16_t>() + r0 * h, h, false, l->param_ptr(MT_P_QKV_W), h, false,
         sv.qkv.as<uint16_t>() + r0 * ld3, ld3, in_rows, ld3, h)
        .bias(l->param_ptr(MT_P_QKV_B))
        .run(st, n);
    mark(c, st, "fwd.qkv_gemm");
  }
  const float alpha = 1.f / std::sqrt((float)hd);
  for (int64_t bb = 0; bb < d.micro_batch; ++bb) {
    const uint16_t* q = sv.qkv.as<uint16_t>() + bb * s * ld3;
    float* lse = sv.lse.as<float>() + bb * Hl * s;
    const long long head_base = bb * d.heads + int64_t{d.tp_rank} * Hl;
    if (l->fused_attn) {
      int written = 0;
      uint32_t* mask = sv.mask.ptr ? sv.mask.as<uint32_t>() + bb * Hl * s * (s / 32) : nullptr;
      const int rc = attention_fwd(q, ld3, (int)Hl, (int)s, (int)hd, head_base, alpha, site_attn, th_a, scale_a,
                                   sv.ctx.as<uint16_t>() + bb * s * hl, hl, lse, mask, &written, st);
      sv.mask_valid = written != 0;
      if (rc != 0) throw RuntimeFailure("attention_fwd failed");
      ++n;
      mark(c, st, "fwd.flash_attention");
      continue;
    }
    uint16_t* S = sv.S.as<uint16_t>() + bb * Hl * s * s;
    uint16_t* P = sv.P.as<uint16_t>() + bb * Hl * s * s;
    Gemm(q, ld3, false, q + hd, ld3, false, S, s, s, s, hd)
        .batched(Hl, 3 * hd, 3 * hd, s * s)
        .alpha(alpha)
        .causal(MT_CAUSAL_SKIP_UPPER_TILES)
        .run(st, n);
    mark(c, st, "fwd.attn_s_gemm");
    softmax_fwd(S, P, lse, (int)Hl, (int)s, head_base, site_attn, th_a, scale_a, st);
    ++n;
    mark(c, st, "fwd.softmax");
    Gemm(P, s, false, q + 2 * hd, ld3, true, sv.ctx.as<uint16_t>() + bb * s * hl, hl, s, hd, s)
        .batched(Hl, s * s, 3 * hd, hd)
        .causal(MT_CAUSAL_K_LE_M)
        .run(st, n);
    mark(c, st, "fwd.attn_pv_gemm");
  }
  {
    const LnOut ln2{l->param_ptr(MT_P_LN2_GAMMA), l->param_ptr(MT_P_LN2_BETA), sv.ln2.ptr, mean2, rstd2, d.ln_eps};
    row_parallel_block(
        c, tpc, sp, M, h, hl,
        [&](int64_t r0, int64_t nr, int cap, mt_gemm_allreduce* ar) {
          Gemm(sv.ctx.as<uint16_t>() + r0 * hl, hl, false, l->param_ptr(MT_P_PROJ_W), hl, false,
               static_cast<uint16_t*>(z) + r0 * h, h, nr, h, hl)
              .max_ctas(cap)
              .allreduce(ar)
              .run(st, n);
        },
        z, l->param_ptr(MT_P_PROJ_B), x, sv.x1.ptr, site_out1, th_h, scale_h, &ln2, st, n, "fwd.proj_gemm",
        hidden_keep(l, sv, 0));
  }
  Gemm(sv.ln2.ptr, h, false, l->param_ptr(MT_P_FC1_W), h, false, sv.act.ptr, ffl, M, ffl, h)
      .epi(MT_EPI_BIAS_GELU)
      .bias(l->param_ptr(MT_P_FC1_B))
      .aux(sv.pre.ptr, ffl)
      .run(st, n);
  mark(c, st, "fwd.fc1_gemm");
  row_parallel_block(
      c, tpc, sp, M, h, ffl,
      [&](int64_t r0, int64_t nr, int cap, mt_gemm_allreduce* ar) {
        Gemm(sv.act.as<uint16_t>() + r0 * ffl, ffl, false, l->param_ptr(MT_P_FC2_W), ffl, false,
             static_cast<uint16_t*>(z) + r0 * h, h, nr, h, ffl)
            .max_ctas(cap)
            .allreduce(ar)
            .run(st, n);
      },
      z, l->param_ptr(MT_P_FC2_B), sv.x1.ptr, y, site_out2, th_h, scale_h, nullptr, st, n, "fwd.fc2_gemm",
      hidden_keep(l, sv, 1));
  check_cuda(cudaGetLastError(), "layer forward launch");
  l->fwd_launches = n;
}

void backward_from(mt_layer* l, const void* dy, void* dx, uint32_t mb, uint64_t mseed, cudaStream_t st,
                   mt_layer::Saved& sv);

void layer_backward(mt_layer* l, const void* dy, void* dx, uint32_t mb, cudaStream_t st) {
  auto it = l->saved.find(mb);
  if (it == l->saved.end()) throw std::invalid_argument("backward without a saved forward for this microbatch");
  const uint64_t mseed = curator::step_seed(l->d.seed, it->second->step);  // the forward's masks
  if (l->recompute) {
    mt_layer::Saved& w = work_slot(l);
    const int fwd_n = l->fwd_launches;
    forward_into(l, it->second->x, l->ctx->scratch_h[3].ptr, mb, mseed, st, w);  // regenerate the activations
    const int refwd = l->fwd_launches;
    l->fwd_launches = fwd_n;
    backward_from(l, dy, dx, mb, mseed, st, w);
    l->bwd_launches += refwd;
  } else {
    backward_from(l, dy, dx, mb, mseed, st, *it->second);
  }
  l->free_slots.push_back(std::move(it->second));
  l->saved.erase(it);
}

void backward_from(mt_layer* l, const void* dy, void* dx, uint32_t mb, uint64_t mseed, cudaStream_t st,
                   mt_layer::Saved& sv) {
  mt_ctx* c = l->ctx;
  tl_ctx = c;
  const mt_layer_desc& d = l->d;
  const bool tpc = tp_collectives(c, d);
  const int64_t M = l->M, h = l->h, hl = l->hl, ffl = l->ffl, ld3 = l->qkvl, s = d.seq, Hl = l->heads_local,
                hd = l->head_dim;
  float* mean1 = sv.stats.as<float>();
  float* rstd1 = mean1 + M;
  float* mean2 = rstd1 + M;
  float* rstd2 = mean2 + M;
  float* ws = c->scratch_ws.as<float>();
  int n = 0;
  const float scale_h = 1.f / (1.f - d.dropout_hidden), scale_a = 1.f / (1.f - d.dropout_attn);
  const uint32_t th_h = curator::dropout_threshold16(d.dropout_hidden);
  const uint32_t th_a = curator::dropout_threshold16(d.dropout_attn);
  const uint64_t site_attn = key_of(mseed, "attn.probs", d.layer_index, mb);
  const uint64_t site_out1 = key_of(mseed, "attn.out", d.layer_index, mb);
  const uint64_t site_out2 = key_of(mseed, "mlp.out", d.layer_index, mb);
  void* dm = tp_buffer(c, 0);   // mlp-out grad, later attn-out grad (dz)
  void* dln = tp_buffer(c, 1);  // grad wrt LN2 / LN1 output
  void* dx1 = c->scratch_h[2].ptr;  // grad wrt residual stream x1
  void* dpre = c->scratch_ffn.ptr;
  void* dctx = c->scratch_ctx.ptr;
  void* dqkv = c->scratch_qkv.ptr;
  uint16_t* dP = c->scratch_attn.as<uint16_t>();
  const bool acc = !l->grads_fresh;  // accumulate into the fp32 grads, or overwrite them
  l->grads_fresh = false;
  const int wg_epi = acc ? MT_EPI_ACCUM_F32 : MT_EPI_STORE_F32;
  // sequence parallel: dy / dx / x / x1 hold this rank's token rows; the replicated parameters'
  // gradients are partial sums over those rows until mt_layer_finish_grads
  SeqPar sp;
  sp.on = tpc && c->seq_parallel;
  sp.ms = sp.on ? M / d.tp_size : M;
  sp.r0 = sp.on ? int64_t{d.tp_rank} * sp.ms : 0;
  const uint64_t eoff = static_cast<uint64_t>(sp.r0 * h);
  if (sp.on) l->sp_partial = true;

  mark(c, st, "begin");
  // ---- MLP block
  dropout_bwd_bias_grad(dy, rows_of(dm, sp.r0, h), l->grad_ptr(MT_P_FC2_B), (int)sp.ms, (int)h, site_out2, th_h,
                        scale_h, ws, acc, st, eoff, hidden_keep(l, sv, 1));
  n += 2;
  if (sp.on) {
    sp_allgather(c, dm, sp.ms * h, st);
    ++n;
  }
  mark(c, st, "bwd.dropout_bias_grad");
  Gemm(dm, h, false, l->param_ptr(MT_P_FC2_W), ffl, true, dpre, ffl, M, ffl, h)
      .epi(MT_EPI_GELU_BWD)
      .aux(sv.pre.ptr, ffl)
      .run(st, n);
  mark(c, st, "bwd.fc2_dgrad_gelu");
  Gemm(dm, h, true, sv.act.ptr, ffl, true, l->grad_ptr(MT_P_FC2_W), ffl, h, ffl, M).epi(wg_epi).run(st, n);
  mark(c, st, "bwd.fc2_wgrad");
  // dgrad first so its TP all-reduce ("f") overlaps the independent wgrad and bias-grad work
  Gemm(dpre, ffl, false, l->param_ptr(MT_P_FC1_W), h, true, dln, h, M, h, ffl).run(st, n);
  mark(c, st, "bwd.fc1_dgrad");
  int cap = 0;
  if (tpc) {
    cap = sp.on ? sp_reduce_scatter_async(c, dln, sp.ms * h, st)
                : tp_allreduce_async(c, dln, M * h, st, "ncclAllReduce(ln2.grad)");
    ++n;
  }
  bias_grad(dpre, l->grad_ptr(MT_P_FC1_B), (int)M, (int)ffl, ffl, ws, acc, st);
  n += 2;
  mark(c, st, "bwd.bias_grad");
  Gemm(dpre, ffl, true, sv.ln2.ptr, h, true, l->grad_ptr(MT_P_FC1_W), h, ffl, h, M).epi(wg_epi).max_ctas(cap).run(st, n);
  mark(c, st, "bwd.fc1_wgrad");
  if (tpc) tp_allreduce_join(c, st);
  mark(c, st, "bwd.tp_allreduce_wait");
  n += ln_bwd(rows_of(dln, sp.r0, h), sv.x1.ptr, l->param_ptr(MT_P_LN2_GAMMA), mean2, rstd2, dy, dx1,
              l->grad_ptr(MT_P_LN2_GAMMA), l->grad_ptr(MT_P_LN2_BETA), (int)sp.ms, (int)h, ws, acc, st);
  mark(c, st, "bwd.ln_bwd");
  // ---- attention block
  void* dz = dm;
  dropout_bwd_bias_grad(dx1, rows_of(dz, sp.r0, h), l->grad_ptr(MT_P_PROJ_B), (int)sp.ms, (int)h, site_out1, th_h,
                        scale_h, ws, acc, st, eoff, hidden_keep(l, sv, 0));
  n += 2;
  if (sp.on) {
    sp_allgather(c, dz, sp.ms * h, st);
    ++n;
  }
  mark(c, st, "bwd.dropout_bias_grad");
  Gemm(dz, h, false, l->param_ptr(MT_P_PROJ_W), hl, true, dctx, hl, M, hl, h).run(st, n);
  mark(c, st, "bwd.proj_dgrad");
  Gemm(dz, h, true, sv.ctx.ptr, hl, true, l->grad_ptr(MT_P_PROJ_W), hl, h, hl, M).epi(wg_epi).run(st, n);
  mark(c, st, "bwd.proj_wgrad");
  const float alpha = 1.f / std::sqrt((float)hd);
  for (int64_t bb = 0; bb < d.micro_batch; ++bb) {
    const uint16_t* q = sv.qkv.as<uint16_t>() + bb * s * ld3;
    uint16_t* dq = static_cast<uint16_t*>(dqkv) + bb * s * ld3;
    const uint16_t* dc = static_cast<const uint16_t*>(dctx) + bb * s * hl;
    if (l->fused_attn) {
      const long long head_base = bb * d.heads + int64_t{d.tp_rank} * Hl;
      const int rc = attention_bwd(q, ld3, sv.ctx.as<uint16_t>() + bb * s * hl, dc, hl, (int)Hl, (int)s, (int)hd,
                                   head_base, alpha, site_attn, th_a, scale_a, sv.lse.as<float>() + bb * Hl * s,
                                   c->scratch_attn.as<float>(), dq,
                                   sv.mask_valid ? sv.mask.as<uint32_t>() + bb * Hl * s * (s / 32) : nullptr,
                                   c->scratch_dq.as<float>(), st);
      if (rc != 0) throw RuntimeFailure("attention_bwd failed");
      n += 3;
      mark(c, st, "bwd.flash_attention");
      continue;
    }
    const uint16_t* S = sv.S.as<uint16_t>() + bb * Hl * s * s;
    const uint16_t* P = sv.P.as<uint16_t>() + bb * Hl * s * s;
    const float* lse = sv.lse.as<float>() + bb * Hl * s;
    // dP_dropped = dctx_h V_h^T
    Gemm(dc, hl, false, q + 2 * hd, ld3, false, dP, s, s, s, hd)
        .batched(Hl, hd, 3 * hd, s * s)
        .causal(MT_CAUSAL_SKIP_UPPER_TILES)
        .run(st, n);
    mark(c, st, "bwd.attn_dp_gemm");
    // dV_h = P_h^T dctx_h
    Gemm(P, s, true, dc, hl, true, dq + 2 * hd, ld3, s, hd, s)
        .batched(Hl, s * s, hd, 3 * hd)
        .causal(MT_CAUSAL_K_GE_M)
        .run(st, n);
    mark(c, st, "bwd.attn_dv_gemm");
    const long long head_base = bb * d.heads + int64_t{d.tp_rank} * Hl;
    // row term D_i = dctx_i . ctx_i per head (= sum_j P_ij dP_ij) from a tiny kernel, so the softmax
    // backward is one pass over S and dP
    float* Dbuf = c->scratch_stats.as<float>();
    attn_rowdot(dc, sv.ctx.as<uint16_t>() + bb * s * hl, hl, (int)hd, (int)Hl, (int)s, Dbuf, st);
    softmax_bwd_rowdot(S, lse, Dbuf, dP, (int)Hl, (int)s, head_base, site_attn, th_a, scale_a, alpha, st);
    n += 2;
    mark(c, st, "bwd.softmax");
    // dQ_h = dS_h K_h ; dK_h = dS_h^T Q_h   (dS already carries the 1/sqrt(d) factor)
    Gemm(dP, s, false, q + hd, ld3, true, dq, ld3, s, hd, s)
        .batched(Hl, s * s, 3 * hd, 3 * hd)
        .causal(MT_CAUSAL_K_LE_M)
        .run(st, n);
    Gemm(dP, s, true, q, ld3, true, dq + hd, ld3, s, hd, s)
        .batched(Hl, s * s, 3 * hd, 3 * hd)
        .causal(MT_CAUSAL_K_GE_M)
        .run(st, n);
    mark(c, st, "bwd.attn_dq_dk_gemm");
  }
  Gemm(dqkv, ld3, false, l->param_ptr(MT_P_QKV_W), h, true, dln, h, M, h, ld3).run(st, n);
  mark(c, st, "bwd.qkv_dgrad");
  cap = 0;
  if (tpc) {
    cap = sp.on ? sp_reduce_scatter_async(c, dln, sp.ms * h, st)
                : tp_allreduce_async(c, dln, M * h, st, "ncclAllReduce(ln1.grad)");
    ++n;
  }
  bias_grad(dqkv, l->grad_ptr(MT_P_QKV_B), (int)M, (int)ld3, ld3, ws, acc, st);
  n += 2;
  mark(c, st, "bwd.bias_grad");
  Gemm(dqkv, ld3, true, sv.ln1.ptr, h, true, l->grad_ptr(MT_P_QKV_W), h, ld3, h, M).epi(wg_epi).max_ctas(cap).run(st, n);
  mark(c, st, "bwd.qkv_wgrad");
  if (tpc) tp_allreduce_join(c, st);
  mark(c, st, "bwd.tp_allreduce_wait");
  n += ln_bwd(rows_of(dln, sp.r0, h), sv.x, l->param_ptr(MT_P_LN1_GAMMA), mean1, rstd1, dx1, dx,
              l->grad_ptr(MT_P_LN1_GAMMA), l->grad_ptr(MT_P_LN1_BETA), (int)sp.ms, (int)h, ws, acc, st);
  mark(c, st, "bwd.ln_bwd");
  check_cuda(cudaGetLastError(), "layer backward launch");
  l->bwd_launches = n;
}

// Sequence parallelism leaves the TP-replicated parameters' gradients (LayerNorms, row-parallel
// biases) as per-rank partial sums over token rows; one grouped TP all-reduce completes them.
void finish_layer_grads(mt_layer* l, cudaStream_t st) {
  if (!l->sp_partial) return;
  l->sp_partial = false;
  if (l->grads_fresh) return;  // logically zero on every rank
  mt_ctx* c = l->ctx;
  check_nccl(ncclGroupStart(), "group");
  for (int p : {MT_P_LN1_GAMMA, MT_P_LN1_BETA, MT_P_PROJ_B, MT_P_LN2_GAMMA, MT_P_LN2_BETA, MT_P_FC2_B})
    check_nccl(ncclAllReduce(l->grad_ptr(p), l->grad_ptr(p), l->param_rows[p] * l->param_cols[p], ncclFloat32, ncclSum,
                             c->tp, st),
               "ncclAllReduce(replicated grads)");
  check_nccl(ncclGroupEnd(), "group");
}

}  // namespace

extern "C" int mt_layer_finish_grads(mt_layer* l, void* stream) {
  return guarded([&] {
    if (!l) throw std::invalid_argument("null layer");
    finish_layer_grads(l, (cudaStream_t)stream);
  });
}

extern "C" int mt_ctx_set_sequence_parallel(mt_ctx* c, int32_t enable) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null context");
    c->seq_parallel = enable != 0;
  });
}

extern "C" int mt_layer_forward(mt_layer* l, const void* x, void* y, uint32_t mb, void* stream) {
  return guarded([&] {
    if (!l || !x || !y) throw std::invalid_argument("null argument");
    WatchdogArm arm(l->ctx);
    layer_forward(l, x, y, mb, (cudaStream_t)stream);
  });
}

extern "C" int mt_layer_backward(mt_layer* l, const void* dy, void* dx, uint32_t mb, void* stream) {
  return guarded([&] {
    if (!l || !dy || !dx) throw std::invalid_argument("null argument");
    WatchdogArm arm(l->ctx);
    layer_backward(l, dy, dx, mb, (cudaStream_t)stream);
  });
}

extern "C" int mt_mse_loss(const void* y, const void* t, void* dy, float* loss, int64_t n, void* stream) {
  return guarded([&] {
    if (n % 8) throw std::invalid_argument("n must be a multiple of 8");
    mt::mse_loss(y, t, dy, loss, n, (cudaStream_t)stream);
    check_cuda(cudaGetLastError(), "mse_loss");
  });
}

extern "C" int mt_fill_normal(void* out, int64_t n, uint64_t key, float mean, float std, void* stream) {
  return guarded([&] {
    mt::fill_normal(out, 1, n, n, 0, 0, key, mean, std, (cudaStream_t)stream);
    check_cuda(cudaGetLastError(), "fill_normal");
  });
}

// =========================================================================== optimizer (N1)
extern "C" int mt_adam_defaults(mt_adam_desc* o) {
  return guarded([&] {
    if (!o) throw std::invalid_argument("null out");
    const curator::TrainingRecipe r;
    o->lr = -1.f;
    o->tokens_seen = 0.0;
    o->beta1 = static_cast<float>(r.adam_beta1);
    o->beta2 = static_cast<float>(r.adam_beta2);
    o->eps = static_cast<float>(r.adam_eps);
    o->weight_decay = static_cast<float>(r.weight_decay);
    o->grad_clip = static_cast<float>(r.grad_clip);
    o->step = 1;
  });
}

float resolve_lr(const mt_adam_desc& d) {
  return d.lr >= 0.f ? d.lr : static_cast<float>(curator::lr_at(d.tokens_seen));
}

extern "C" int mt_layer_adam_step(mt_layer* l, const mt_adam_desc* d, float* grad_norm_out, void* stream) {
  return guarded([&] {
    if (!l || !d) throw std::invalid_argument("null argument");
    if (d->step < 1) throw std::invalid_argument("step must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    settle_fresh_grads(l, s);
    mt::DeviceBuffer& buf = l->ctx->opt_scratch;
    buf.ensure(4 * sizeof(float));
    float* sq = buf.as<float>();
    check_cuda(cudaMemsetAsync(sq, 0, 2 * sizeof(float), s), "memset");
    mt::layer_grad_sq(l, sq, s);
    mt::clip_coefficient(sq, d->grad_clip, sq + 2, s);
    mt::layer_adamw(l, *d, resolve_lr(*d), sq + 3, s);
    if (grad_norm_out) {
      check_cuda(cudaMemcpyAsync(grad_norm_out, sq + 2, sizeof(float), cudaMemcpyDeviceToHost, s), "D2H norm");
      check_cuda(cudaStreamSynchronize(s), "sync");
    }
  });
}

extern "C" int mt_layer_get_optimizer_state(mt_layer* l, int32_t p, float* master, float* m, float* v) {
  return guarded([&] {
    if (p < 0 || p >= MT_P_COUNT) throw std::invalid_argument("unknown parameter id");
    if (!l->opt_master.ptr) throw std::invalid_argument("no optimizer step has run");
    check_cuda(cudaDeviceSynchronize(), "sync");
    const size_t n = static_cast<size_t>(l->param_rows[p] * l->param_cols[p]) * 4;
    const size_t off = static_cast<size_t>(l->param_off[p]) * 4;
    if (master) check_cuda(cudaMemcpy(master, l->opt_master.as<char>() + off, n, cudaMemcpyDeviceToHost), "D2H");
    if (m) check_cuda(cudaMemcpy(m, l->opt_m.as<char>() + off, n, cudaMemcpyDeviceToHost), "D2H");
    if (v) check_cuda(cudaMemcpy(v, l->opt_v.as<char>() + off, n, cudaMemcpyDeviceToHost), "D2H");
  });
}
