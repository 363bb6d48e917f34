// Host side of the fused row-parallel GEMM + TP all-reduce (the forward "g" of PAPER.md:146-148).
//
// The [M, h] row-parallel output buffer lives in NCCL symmetric memory (ncclMemAlloc + a window
// registered on the TP communicator, runtime.cpp ensure_symmetric); this file adds a second small
// symmetric window for the per-unit ready flags and the completion counter, and resolves through the
// NCCL device API (ncclDevCommCreate with lsaMultimem) the NVLink-SHARP multicast addresses of both
// windows and every peer's flag array. The GEMM kernel (gemm_sm100.cu, allreduce_unit) then does the
// reduction from its epilogue warps while its tensor cores work on later tiles, and the consumer
// waits on the counter (mt_gemm_allreduce_wait) instead of an NCCL all-reduce.
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>

#include "runtime.hpp"

namespace mt {

struct FusedAllReduce {
  ncclDevComm dev{};
  bool dev_created = false;
  void* flags = nullptr;  // [0]: completion counter; [kFlagBase..): per-unit flags
  size_t flags_bytes = 0;
  ncclWindow_t flags_win = nullptr;
  void* z = nullptr;  // the symmetric output buffer the multicast address below belongs to
  mt_gemm_allreduce desc{};
  uint32_t target = 0;  // cumulative units of all launches: the counter value that means "all done"
};

namespace {

constexpr int64_t kFlagBase = 64;  // counter on its own 256-byte line
constexpr int64_t kCapacity = 1 << 16;

__global__ void resolve_kernel(ncclWindow_t zwin, ncclWindow_t fwin, ncclDevComm dc, void** out) {
  out[0] = ncclGetLsaMultimemPointer(zwin, 0, dc);
  out[1] = ncclGetLsaMultimemPointer(fwin, 0, dc);
  for (int r = 0; r < dc.lsaSize && r < 8; ++r) out[2 + r] = ncclGetLsaPointer(fwin, 0, r);
  out[10] = reinterpret_cast<void*>(static_cast<uintptr_t>(dc.lsaSize));
  out[11] = reinterpret_cast<void*>(static_cast<uintptr_t>(dc.lsaRank));
}

// Multicast / peer addresses of the current symmetric buffers (collective: every TP rank resolves
// at the same point because buffer allocation is collective).
void resolve(mt_ctx* c, FusedAllReduce* f) {
  void** d_out = nullptr;
  check_cuda(cudaMalloc(&d_out, 12 * sizeof(void*)), "cudaMalloc");
  resolve_kernel<<<1, 1>>>(c->sym_h[0].win_tp, f->flags_win, f->dev, d_out);
  void* h[12] = {};
  check_cuda(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost), "resolve multicast addresses");
  cudaFree(d_out);
  const int lsa_size = static_cast<int>(reinterpret_cast<uintptr_t>(h[10]));
  const int lsa_rank = static_cast<int>(reinterpret_cast<uintptr_t>(h[11]));
  if (lsa_size != c->par.tensor || lsa_rank != c->place.tensor || !h[0] || !h[1])
    throw RuntimeFailure("fused TP all-reduce: the TP group is not one load/store-accessible multicast team");
  f->z = c->sym_h[0].ptr;
  mt_gemm_allreduce& d = f->desc;
  d = mt_gemm_allreduce{};
  d.d_multicast = h[0];
  d.counter_multicast = static_cast<uint32_t*>(h[1]);
  d.flags_local = static_cast<uint32_t*>(f->flags) + kFlagBase;
  for (int r = 0; r < c->par.tensor; ++r) d.flags_peer[r] = static_cast<const uint32_t*>(h[2 + r]) + kFlagBase;
  d.flag_capacity = kCapacity;
  d.rank = c->place.tensor;
  d.ranks = c->par.tensor;
}

}  // namespace

FusedAllReduce* fused_ar_create(mt_ctx* c) {
  auto f = new FusedAllReduce();
  try {
    ncclDevCommRequirements req{};
    req.lsaMultimem = true;
    check_nccl(ncclDevCommCreate(c->tp, &req, &f->dev), "ncclDevCommCreate(tp, multimem)");
    f->dev_created = true;
    f->flags_bytes = static_cast<size_t>((kFlagBase + kCapacity) * 4 + 4095) / 4096 * 4096;
    check_nccl(ncclMemAlloc(&f->flags, f->flags_bytes), "ncclMemAlloc(flags)");
    check_nccl(ncclCommWindowRegister(c->tp, f->flags, f->flags_bytes, &f->flags_win, NCCL_WIN_COLL_SYMMETRIC),
               "ncclCommWindowRegister(flags)");
    check_cuda(cudaMemset(f->flags, 0, f->flags_bytes), "cudaMemset(flags)");
    check_cuda(cudaDeviceSynchronize(), "sync");
    // every rank's flags are zero before any rank can publish into them
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
  if (f->flags_win) ncclCommWindowDeregister(c->tp, f->flags_win);
  if (f->flags) ncclMemFree(f->flags);
  if (f->dev_created) ncclDevCommDestroy(c->tp, &f->dev);
  delete f;
}

// Descriptor for the next fused launch on buffer sym_h[0] (re-resolved if it was reallocated).
mt_gemm_allreduce* fused_ar_begin(mt_ctx* c) {
  FusedAllReduce* f = c->fused_ar;
  if (f->z != c->sym_h[0].ptr) resolve(c, f);
  f->desc.epoch += 1;
  f->desc.units = 0;
  return &f->desc;
}

// Orders `st` after every unit of every rank of the launch described by `d`.
void fused_ar_end(mt_ctx* c, cudaStream_t st) {
  FusedAllReduce* f = c->fused_ar;
  f->target += static_cast<uint32_t>(f->desc.units);
  const int rc = mt_gemm_allreduce_wait(static_cast<const uint32_t*>(f->flags), f->target, st);
  if (rc != 0) throw RuntimeFailure("mt_gemm_allreduce_wait failed");
}

}  // namespace mt
