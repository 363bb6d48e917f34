// Host side of the fused row-parallel GEMM + TP all-reduce (the forward "g" of PAPER.md:146-148).
//
// The [M, h] row-parallel output buffer lives in NCCL symmetric memory (ncclMemAlloc + a window
// registered on the TP communicator, runtime.cpp ensure_symmetric); this file adds a second small
// symmetric window for the completion counter and the per-column-group unit counters, and resolves
// through the NCCL device API (ncclDevCommCreate with lsaMultimem) the NVLink-SHARP multicast
// addresses of both windows. The GEMM kernel (gemm_sm100.cu) counts each finished output unit on its
// column group; a reducer kernel on the SMs the GEMM leaves free (allreduce_group_kernel) reduces
// each group over NVLink SHARP as soon as every rank finished it, while the GEMM still runs later
// groups, and the consumer waits on the completion counter instead of an NCCL all-reduce. Every
// cross-rank wait is bounded (mt_ctx timeout): a dead peer raises the context's error flag.
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "runtime.hpp"
#include "sm100_ptx.cuh"

namespace mt {

struct FusedAllReduce {
  ncclDevComm dev{};
  bool dev_created = false;
  void* flags = nullptr;  // [0]: completion counter (own 256-byte line); [kGroupBase..+64): group counters
  size_t flags_bytes = 0;
  ncclWindow_t flags_win = nullptr;
  void* z = nullptr;  // the symmetric output buffer the multicast address below belongs to
  void* z1 = nullptr;   // the second symmetric buffer (LN-input gradients, backward) and its multicast address
  void* mc1 = nullptr;
  mt_gemm_allreduce desc{};
  uint32_t target = 0;  // cumulative arrivals of all launches: the counter value that means "all done"
  int reducer_ctas = 16;  // reducer CTAs running beside the GEMM (MT_AR_CTAS)
  int nvls_ctas = 0;      // CTAs of the standalone NVLS all-reduce kernel (MT_NVLS_CTAS; 0: reducer_ctas)
  int groups = 6;         // column groups per fused launch (the reduction of group g overlaps groups > g)
  int bwd_ctas = 16;      // CTAs of the backward NVLS all-reduce beside the wgrad GEMM (MT_NVLS_BWD_CTAS)
};

namespace {

constexpr int64_t kGroupBase = 64;

__global__ void resolve_kernel(ncclWindow_t zwin, ncclWindow_t fwin, ncclWindow_t z1win, ncclDevComm dc, void** out) {
  out[0] = ncclGetLsaMultimemPointer(zwin, 0, dc);
  out[1] = ncclGetLsaMultimemPointer(fwin, 0, dc);
  out[2] = reinterpret_cast<void*>(static_cast<uintptr_t>(dc.lsaSize));
  out[3] = reinterpret_cast<void*>(static_cast<uintptr_t>(dc.lsaRank));
  out[4] = z1win ? ncclGetLsaMultimemPointer(z1win, 0, dc) : nullptr;
}

// Multicast addresses of the current symmetric buffers (collective: every TP rank resolves at the
// same point because buffer allocation is collective).
void resolve(mt_ctx* c, FusedAllReduce* f) {
  void** d_out = nullptr;
  check_cuda(cudaMalloc(&d_out, 5 * sizeof(void*)), "cudaMalloc");
  resolve_kernel<<<1, 1>>>(c->sym_h[0].win_tp, f->flags_win, c->sym_h[1].win_tp, f->dev, d_out);
  void* h[5] = {};
  check_cuda(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost), "resolve multicast addresses");
  cudaFree(d_out);
  const int lsa_size = static_cast<int>(reinterpret_cast<uintptr_t>(h[2]));
  const int lsa_rank = static_cast<int>(reinterpret_cast<uintptr_t>(h[3]));
  if (lsa_size != c->par.tensor || lsa_rank != c->place.tensor || !h[0] || !h[1])
    throw RuntimeFailure("fused TP all-reduce: the TP group is not one load/store-accessible multicast team");
  f->z = c->sym_h[0].ptr;
  f->z1 = c->sym_h[1].ptr;
  f->mc1 = h[4];
  mt_gemm_allreduce& d = f->desc;
  d = mt_gemm_allreduce{};
  d.d_multicast = h[0];
  d.counter_multicast = static_cast<uint32_t*>(h[1]);
  d.group_counters = static_cast<uint32_t*>(f->flags) + kGroupBase;
  d.rank = c->place.tensor;
  d.ranks = c->par.tensor;
  d.groups = f->groups;
  d.error_flag = c->err_dev;
  d.timeout_ns = c->timeout_ns;
}

}  // namespace

FusedAllReduce* fused_ar_create(mt_ctx* c) {
  auto f = new FusedAllReduce();
  if (const char* e = getenv("MT_AR_CTAS")) f->reducer_ctas = std::max(1, atoi(e));
  if (const char* e = getenv("MT_NVLS_CTAS")) f->nvls_ctas = std::max(0, atoi(e));
  if (const char* e = getenv("MT_NVLS_BWD_CTAS")) f->bwd_ctas = std::max(1, atoi(e));
  try {
    ncclDevCommRequirements req{};
    req.lsaMultimem = true;
    check_nccl(ncclDevCommCreate(c->tp, &req, &f->dev), "ncclDevCommCreate(tp, multimem)");
    f->dev_created = true;
    f->flags_bytes = 4096;
    check_nccl(ncclMemAlloc(&f->flags, f->flags_bytes), "ncclMemAlloc(flags)");
    check_nccl(ncclCommWindowRegister(c->tp, f->flags, f->flags_bytes, &f->flags_win, NCCL_WIN_COLL_SYMMETRIC),
               "ncclCommWindowRegister(flags)");
    check_cuda(cudaMemset(f->flags, 0, f->flags_bytes), "cudaMemset(flags)");
    check_cuda(cudaDeviceSynchronize(), "sync");
    // every rank's counter is zero before any rank can arrive on it
    check_nccl(ncclAllReduce(f->flags, f->flags, 1, ncclUint32, ncclSum, c->tp, nullptr), "ncclAllReduce(sync)");
    check_cuda(cudaDeviceSynchronize(), "sync");
    resolve(c, f);
  } catch (...) {
    fused_ar_destroy(c, f);
    throw;
  }
  return f;
}

void fused_ar_destroy(mt_ctx* c, FusedAllReduce* f) {
  if (!f) return;
  cudaDeviceSynchronize();
  if (c->tp) {  // an aborted communicator (peer timeout) owns nothing we may deregister
    if (f->flags_win) ncclCommWindowDeregister(c->tp, f->flags_win);
    if (f->flags) ncclMemFree(f->flags);
    if (f->dev_created) ncclDevCommDestroy(c->tp, &f->dev);
  }
  delete f;
}

// Descriptor for the next fused launch on buffer sym_h[0] (re-resolved if it was reallocated).
mt_gemm_allreduce* fused_ar_begin(mt_ctx* c) {
  FusedAllReduce* f = c->fused_ar;
  if (f->z != c->sym_h[0].ptr) resolve(c, f);
  f->desc.units = 0;
  f->desc.group_cols = 0;
  return &f->desc;
}

// The group counters must read zero when the GEMM starts.
void fused_ar_prepare(mt_ctx* c, cudaStream_t st) {
  FusedAllReduce* f = c->fused_ar;
  check_cuda(cudaMemsetAsync(f->desc.group_counters, 0, sizeof(uint32_t) * 64, st), "memset group counters");
}

// SMs the fused GEMM may use (the reducer kernel takes the rest).
int fused_ar_gemm_ctas(mt_ctx* c) {
  const FusedAllReduce* f = c->fused_ar;
  int sms = 0;
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device), "attr");
  return std::max(2, (sms - f->reducer_ctas) / 2 * 2);
}

// After the GEMM was enqueued on `st` (following ev_ready recorded just before it): the reducer runs
// on the side stream concurrently with the GEMM (it starts only after the work that preceded the
// GEMM on `st`, so it never holds SMs a preceding kernel still needs); `st` is then ordered after
// every rank's reducer by the completion counter.
void fused_ar_end(mt_ctx* c, cudaStream_t st, void* d, int64_t ldd) {
  (void)d;
  FusedAllReduce* f = c->fused_ar;
  const uint32_t* counter = static_cast<const uint32_t*>(f->flags);
  if (f->desc.group_cols <= 0) throw RuntimeFailure("fused GEMM + all-reduce: column-group geometry missing");
  const int groups = static_cast<int>((f->desc.geom[5] + f->desc.group_cols - 1) / f->desc.group_cols);
  const uint32_t base = f->target;
  f->target = base + static_cast<uint32_t>(c->par.tensor * (groups + f->reducer_ctas));
  check_cuda(cudaStreamWaitEvent(c->comm, c->ev_ready, 0), "cudaStreamWaitEvent");
  if (mt_gemm_allreduce_reduce_groups(&f->desc, ldd, f->desc.group_counters, counter, base, f->reducer_ctas, c->comm) !=
      0)
    throw RuntimeFailure("mt_gemm_allreduce_reduce_groups failed");
  check_cuda(cudaEventRecord(c->ev_done, c->comm), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(st, c->ev_done, 0), "cudaStreamWaitEvent");
  if (mt_gemm_allreduce_wait(&f->desc, counter, f->target, st) != 0) throw RuntimeFailure("mt_gemm_allreduce_wait failed");
}

// ---- diagnostic: raw NVLS all-reduce throughput over the symmetric buffer (mt_ctx_nvls_probe)
namespace {
__global__ void __launch_bounds__(1024) nvls_probe_kernel(__nv_bfloat16* mc, long long elems, int rank, int ranks,
                                                          int strided, long long ld) {
  // this rank's 1/ranks share in 16-byte chunks; contiguous (strided = 0) or as 128 x 256 tiles of
  // a row-major [*, ld] matrix (strided = 1, the GEMM unit pattern)
  const long long chunks = elems / 8, per = chunks / ranks, c0 = per * rank;
  constexpr int U = 4;
  for (long long base = c0 + blockIdx.x * (long long)blockDim.x * U + threadIdx.x; base < c0 + per;
       base += (long long)gridDim.x * blockDim.x * U) {
    uint32_t v[U][4];
    long long off[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      long long q = base + (long long)k * blockDim.x;
      if (strided) {  // chunk q -> tile t, row r, col chunk c (32 chunks per 256-wide tile row)
        const long long t = q / 4096, within = q % 4096, r = within / 32, c = within % 32;
        const long long tiles_per_row = ld / 256;
        const long long tr = t / tiles_per_row, tc = t % tiles_per_row;
        off[k] = (tr * 128 + r) * ld + tc * 256 + c * 8;
      } else {
        off[k] = q * 8;
      }
      if (q < c0 + per) multimem_ld_reduce_bf16x8(mc + off[k], v[k]);
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (base + (long long)k * blockDim.x < c0 + per) multimem_st_bf16x8(mc + off[k], v[k]);
  }
}
}  // namespace

extern "C" int mt_ctx_nvls_probe(mt_ctx* c, int64_t elems, int64_t ld, int32_t strided, int32_t ctas, int32_t iters,
                                 double* us_per_iter) {
  try {
    if (!c || !c->fused_ar || !c->sym_h[0].ptr) throw std::invalid_argument("no fused all-reduce state");
    if (elems * 2 > (int64_t)c->sym_h[0].bytes) throw std::invalid_argument("probe larger than the buffer");
    FusedAllReduce* f = c->fused_ar;
    if (f->z != c->sym_h[0].ptr) resolve(c, f);
    auto* mc = static_cast<__nv_bfloat16*>(f->desc.d_multicast);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    check_nccl(ncclAllReduce(f->flags, f->flags, 1, ncclUint32, ncclSum, c->tp, nullptr), "sync");
    nvls_probe_kernel<<<ctas, 1024>>>(mc, elems, c->place.tensor, c->par.tensor, strided, ld);
    check_cuda(cudaDeviceSynchronize(), "probe warmup");
    check_nccl(ncclAllReduce(f->flags, f->flags, 1, ncclUint32, ncclSum, c->tp, nullptr), "sync");
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i)
      nvls_probe_kernel<<<ctas, 1024>>>(mc, elems, c->place.tensor, c->par.tensor, strided, ld);
    cudaEventRecord(e1);
    check_cuda(cudaEventSynchronize(e1), "probe");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *us_per_iter = 1e3 * ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return MT_OK;
  } catch (const std::exception& e) {
    return MT_ERR_DATA;
  }
}

// ---- standalone NVLS all-reduce of the symmetric row-parallel buffer (MT_TP_NVLS=1): one kernel,
// entry barrier (every rank's GEMM output complete) -> this rank's 1/R share summed with
// multimem.ld_reduce and broadcast with multimem.st -> exit count on every rank's counter; the
// consumer waits on the counter (mt_gemm_allreduce_wait). Same counter as the fused path.
namespace {
__global__ void __launch_bounds__(1024) nvls_allreduce_kernel(__nv_bfloat16* mc, uint32_t* counter_mc,
                                                              const uint32_t* counter_local, uint32_t entry_target,
                                                              long long elems, int rank, int ranks, uint32_t* err,
                                                              unsigned long long timeout_ns) {
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      fence_acq_rel_sys();
      multimem_red_release_add_u32(counter_mc, 1u);
    }
    bounded_wait_geq<true>(counter_local, entry_target, err, timeout_ns);
  }
  __syncthreads();
  const long long chunks = elems / 8, per = (chunks + ranks - 1) / ranks, c0 = per * rank;
  const long long c1 = c0 + per < chunks ? c0 + per : chunks;
  constexpr int U = 4;
  for (long long base = c0 + (long long)blockIdx.x * blockDim.x * U + threadIdx.x; base < c1;
       base += (long long)gridDim.x * blockDim.x * U) {
    uint32_t v[U][4];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long q = base + (long long)k * blockDim.x;
      if (q < c1) multimem_ld_reduce_bf16x8(mc + q * 8, v[k]);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long q = base + (long long)k * blockDim.x;
      if (q < c1) multimem_st_bf16x8(mc + q * 8, v[k]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    multimem_red_release_add_u32(counter_mc, 1u);
  }
}
}  // namespace

// All-reduce (sum) of `elems` bf16 at offset 0 of the symmetric buffer sym_h[which] over the TP group
// (0: forward row-parallel outputs, on the compute stream; 1: backward LN-input gradients, on the side
// stream beside the weight-gradient GEMM). `st` is ordered after every rank's reduction.
void nvls_allreduce(mt_ctx* c, int64_t elems, cudaStream_t st, int which) {
  FusedAllReduce* f = c->fused_ar;
  if (f->z != c->sym_h[0].ptr || f->z1 != c->sym_h[1].ptr) resolve(c, f);
  void* mc = which == 0 ? f->desc.d_multicast : f->mc1;
  if (!mc) throw RuntimeFailure("NVLS all-reduce: no multicast address for the buffer");
  const int ctas = which == 1 ? f->bwd_ctas : (f->nvls_ctas > 0 ? f->nvls_ctas : f->reducer_ctas);
  const uint32_t entry = f->target + static_cast<uint32_t>(c->par.tensor);
  f->target = entry + static_cast<uint32_t>(c->par.tensor * ctas);
  nvls_allreduce_kernel<<<ctas, 1024, 0, st>>>(static_cast<__nv_bfloat16*>(mc), f->desc.counter_multicast,
                                               static_cast<const uint32_t*>(f->flags), entry, elems,
                                               c->place.tensor, c->par.tensor, c->err_dev, c->timeout_ns);
  check_cuda(cudaGetLastError(), "nvls_allreduce");
  if (mt_gemm_allreduce_wait(&f->desc, static_cast<const uint32_t*>(f->flags), f->target, st) != 0)
    throw RuntimeFailure("mt_gemm_allreduce_wait failed");
}

int nvls_bwd_ctas(mt_ctx* c) { return c->fused_ar ? c->fused_ar->bwd_ctas : 0; }

}  // namespace mt
