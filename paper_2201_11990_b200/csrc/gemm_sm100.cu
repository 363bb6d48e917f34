// Persistent, warp-specialised tcgen05 GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM).
//
// Roles (256 threads, one CTA per SM):
//   warp 0 lane 0 : TMA producer   — global -> smem ring of kStages {A,B} tiles (128B swizzle)
//   warp 1 lane 0 : MMA issuer     — tcgen05.mma.cta_group::1 M=128, N=BN, K=16, accumulator in TMEM
//   warp 2        : TMEM allocator — 2 accumulator buffers (double-buffered so the epilogue of
//                                    tile i overlaps the main loop of tile i+1)
//   warps 4..7    : epilogue       — tcgen05.ld TMEM -> registers, fused bias / GeLU / GeLU' /
//                                    fp32 accumulate, vectorised global stores
// Both operands may be K-major or MN-major (the UMMA descriptor major bits), which covers the
// forward (TN), dgrad (NN) and wgrad (TT) products of the layer and the attention contractions
// without any transpose kernels. The layer math these serve is restated from PAPER.md:133-150.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../../include/mtnlg_gemm.h"
#include "sm100_ptx.cuh"

namespace mt {
namespace {

#ifndef MT_GEMM_EPI_BUFS
#define MT_GEMM_EPI_BUFS 2
#endif
constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 256;
constexpr int kSmemBudget = 232448;  // 227 KB opt-in maximum per CTA

struct GemmParams {
  int m, n, k, batch;
  int mblocks, nblocks, kblocks, total_tiles;
  float alpha;
  int epilogue, causal;
  int hints;      // L2 eviction hints on the operand loads (MT_GEMM_HINTS=1 enables; A/B only)
  int n_fastest;  // tile raster: 0 = m-blocks vary fastest (B tile shared by concurrent CTAs), 1 = n-blocks
  __nv_bfloat16* d_bf16;
  float* d_f32;
  long long ldd, d_batch_stride;
  const __nv_bfloat16* bias;
  __nv_bfloat16* aux;
  long long ld_aux;
  // split-K tail: work items [0, full_tiles) are whole tiles; the remaining total_tiles - full_tiles
  // tiles (fewer than one wave) are each split over `splits` k-ranges run by otherwise idle CTAs.
  int full_tiles, splits, work_items;
  float* split_ws;  // fp32 partial tiles [tail][split][rank][128 x BN]
  int* split_cnt;   // arrival counters [tail][rank], self-resetting
  // fused TP all-reduce of D (mt_gemm_allreduce): every finished output unit is counted on its
  // column group's local counter (ar_group_cols column blocks per group); 0 disables
  uint32_t* ar_group_cnt;
  int ar_group_cols;
  uint64_t store_policy;  // L2 hint on fp32 output stores (0 = none)
  // dynamic tile scheduler: ticket counter (nullptr = static round-robin) and the number of tickets
  // one launch draws (the one drawing the last resets the counter for the next launch)
  int* tile_ctr;
  int sched_fetches;
};

// kPair: 2-CTA (cta_group::2) tiles of 256 x BN — each CTA of the pair holds 128 rows of A and
// BN/2 rows of B in its smem and 128 x BN of the accumulator in its TMEM.
template <int BN, bool kPair = false>
struct Cfg {
  static constexpr int kTileM = kPair ? 256 : 128;   // rows of the (pair) tile
  static constexpr int kBRows = kPair ? BN / 2 : BN;  // B rows (n) held by one CTA
  static constexpr int kBNAlloc = (kBRows + 63) / 64 * 64;
  static constexpr int kABytes = 128 * kBK * 2;  // one CTA always holds 128 rows of A
  static constexpr int kBBytes = kBNAlloc * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiBufs = MT_GEMM_EPI_BUFS;  // staging buffers per epilogue warp (TMA stores in flight)
  static constexpr int kEpiBytes = 4 * kEpiBufs * 4096;  // 4 epilogue warps x buffers x (32 rows x 128 B)
  static constexpr int kStagesRaw = (kSmemBudget - 2048 - kEpiBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kEpiBytes + 512;
  static constexpr uint32_t kTmemCols = (2 * BN <= 128) ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr uint32_t kAccStride = kTmemCols / 2;  // column offset of accumulator buffer 1
};

__device__ __forceinline__ void tile_coords(const GemmParams& p, int t, int& b, int& mb, int& nb) {
  const int per_batch = p.mblocks * p.nblocks;
  b = t / per_batch;
  const int rem = t - b * per_batch;
  if (p.n_fastest) {
    mb = rem / p.nblocks;
    nb = rem - mb * p.nblocks;
  } else {
    nb = rem / p.mblocks;
    mb = rem - nb * p.mblocks;
  }
}

template <int BN, int BMT>
__device__ __forceinline__ bool tile_valid(const GemmParams& p, int mb, int nb) {
  if (p.causal == MT_CAUSAL_SKIP_UPPER_TILES) return nb * BN <= mb * BMT + BMT - 1;
  return true;
}

template <int BMT>
__device__ __forceinline__ void k_range(const GemmParams& p, int mb, int& kb0, int& kb1) {
  kb0 = 0;
  kb1 = p.kblocks;
  if (p.causal == MT_CAUSAL_K_LE_M) {
    const int kend = min(p.k, (mb + 1) * BMT);
    kb1 = (kend + kBK - 1) / kBK;
  } else if (p.causal == MT_CAUSAL_K_GE_M) {
    kb0 = (mb * BMT) / kBK;
  }
}

struct Work {
  int b, mb, nb, kb0, kb1;
  int split;  // -1: whole tile; else the split index of a tail tile
  int tail;   // tail tile index (split items)
};

// Decodes work item w (identically in every role) into tile coordinates and its k-block range.
template <int BN, int BMT>
__device__ __forceinline__ bool get_work(const GemmParams& p, int w, Work& o) {
  int t = w;
  o.split = -1;
  o.tail = 0;
  if (w >= p.full_tiles) {
    const int j = w - p.full_tiles;
    o.tail = j / p.splits;
    o.split = j - o.tail * p.splits;
    t = p.full_tiles + o.tail;
  }
  tile_coords(p, t, o.b, o.mb, o.nb);
  if (!tile_valid<BN, BMT>(p, o.mb, o.nb)) return false;
  k_range<BMT>(p, o.mb, o.kb0, o.kb1);
  if (o.split >= 0) {
    const int a = o.kb0, len = o.kb1 - o.kb0;
    o.kb0 = a + (len * o.split) / p.splits;
    o.kb1 = a + (len * (o.split + 1)) / p.splits;
  }
  return true;
}

// The epilogue's hand-back of an accumulator buffer to the pair leader's MMA issuer (TMEM reads
// completed by tcgen05.wait::ld; no memory is published). MT_GEMM_RELEASE_ARRIVE=1 (compile-time)
// restores the release-semantics arrive for A/B measurements.
__device__ __forceinline__ void tmem_release_arrive(uint32_t bar) {
#if defined(MT_GEMM_RELEASE_ARRIVE) && MT_GEMM_RELEASE_ARRIVE
  mbar_arrive_cluster(bar, 0);
#else
  mbar_arrive_cluster_relaxed(bar, 0);
#endif
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Epilogue of one 32-row x 32-column piece held by one warp (thread t = row t, r[j] = column j):
// apply the fused epilogue, write the piece into a swizzled staging buffer and hand it to the TMA
// engine (store, or reduce-add into fp32 gradients). Rows/columns outside D are clipped by TMA.
struct EpiMaps {
  const CUtensorMap* d;
  const CUtensorMap* aux;
};

// bf16 piece: 32 rows x 64 B, SWIZZLE_64B (16-byte chunk j of row t lands at chunk j ^ ((t >> 1) & 3)).
__device__ __forceinline__ void stage_bf16(uint32_t buf, uint32_t lane, const float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t pos = j ^ ((lane >> 1) & 3);
    st_shared_v4(buf + lane * 64 + pos * 16, pack_bf16x2(x[8 * j], x[8 * j + 1]), pack_bf16x2(x[8 * j + 2], x[8 * j + 3]),
                 pack_bf16x2(x[8 * j + 4], x[8 * j + 5]), pack_bf16x2(x[8 * j + 6], x[8 * j + 7]));
  }
}
// wide bf16 piece: 32 rows x 64 columns = 128 B per row, SWIZZLE_128B (like the fp32 piece).
__device__ __forceinline__ void stage_bf16_wide(uint32_t buf, uint32_t lane, const float (&x)[64]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t pos = j ^ (lane & 7);
    st_shared_v4(buf + lane * 128 + pos * 16, pack_bf16x2(x[8 * j], x[8 * j + 1]), pack_bf16x2(x[8 * j + 2], x[8 * j + 3]),
                 pack_bf16x2(x[8 * j + 4], x[8 * j + 5]), pack_bf16x2(x[8 * j + 6], x[8 * j + 7]));
  }
}
// fp32 piece: 32 rows x 128 B, SWIZZLE_128B (chunk j of row t lands at chunk j ^ (t & 7)).
__device__ __forceinline__ void stage_f32(uint32_t buf, uint32_t lane, const float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t pos = j ^ (lane & 7);
    st_shared_v4(buf + lane * 128 + pos * 16, __float_as_uint(x[4 * j]), __float_as_uint(x[4 * j + 1]),
                 __float_as_uint(x[4 * j + 2]), __float_as_uint(x[4 * j + 3]));
  }
}

// Issue the TMA op for the staged piece from lane 0 once all lanes' smem writes are visible.
// policy != 0: L2 eviction hint for the store (MT_GEMM_STORE_HINT: fp32 outputs evict_first).
__device__ __forceinline__ void flush_piece(const CUtensorMap* map, uint32_t buf, uint32_t lane, int col, int row, int b,
                                            bool reduce, uint64_t policy = 0) {
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (policy != 0) {
      if (reduce)
        tma_reduce_add_3d_hint(map, buf, col, row, b, policy);
      else
        tma_store_3d_hint(map, buf, col, row, b, policy);
    } else if (reduce) {
      tma_reduce_add_3d(map, buf, col, row, b);
    } else {
      tma_store_3d(map, buf, col, row, b);
    }
    bulk_commit();
  }
}
// Before overwriting a staging buffer: at most one older bulk group may still be reading smem.
template <int NB>
__device__ __forceinline__ void reuse_wait(uint32_t lane) {
  if (lane == 0) bulk_wait_read<NB - 1>();
  __syncwarp();
}

// Fused TP all-reduce of the output (column-group mode): once all TMA stores of output unit w (this
// CTA's 128 rows x BN of a tile) are complete, the unit is counted on its column group's local
// counter with a gpu-scope release. Column blocks finish in raster order (m-blocks fastest), so the
// reducer kernel (allreduce_group_kernel, on the SMs the GEMM leaves free) can start the cross-rank
// NVLink-SHARP reduction of group g while the tensor cores still work on later groups. kPending =
// bulk groups of the tile issued after w that may still be in flight (never waited on here).
template <int kPending>
__device__ __forceinline__ void ar_publish(const GemmParams& p, int w, uint32_t lane) {
  if (lane == 0) bulk_wait<kPending>();
  __syncwarp();
  epi_bar();
  if (threadIdx.x == 128) {
    fence_proxy_async_global();
    int b, mb, nb;
    tile_coords(p, w, b, mb, nb);
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.ar_group_cnt + nb / p.ar_group_cols) : "memory");
  }
}

constexpr int kReduceThreads = 1024;

// Reducer of the column-group mode: groups of column blocks complete in order in the GEMM; for each
// group, wait until this rank's GEMM published all its units (local counter), then a cross-rank
// barrier on the multicast counter (one arrival per rank and group), then this rank's rows share of
// the group's columns is summed with multimem.ld_reduce and broadcast with multimem.st by all CTAs.
struct ArGroupParams {
  __nv_bfloat16* mc;
  const uint32_t* group_cnt;  // local per-group unit counters (zeroed before the GEMM)
  uint32_t* counter_mc;
  const uint32_t* counter_local;
  uint32_t base;              // counter value before this launch
  int rank, ranks, groups, group_cols, bn, m, n, mblocks, units_per_block;
  long long ldd;
  uint32_t* err;              // peer-timeout flag (bounded_wait_geq)
  unsigned long long timeout_ns;
};

__global__ void __launch_bounds__(kReduceThreads, 1) allreduce_group_kernel(const ArGroupParams p) {
  const int rows = p.m / p.ranks, r0 = p.rank * rows;  // this rank's share of every group
  for (int g = 0; g < p.groups; ++g) {
    const int cb0 = g * p.group_cols, cb1 = min((g + 1) * p.group_cols, (p.n + p.bn - 1) / p.bn);
    if (cb0 >= cb1) break;
    if (threadIdx.x == 0) {
      const uint32_t expect = (uint32_t)((cb1 - cb0) * p.mblocks * p.units_per_block);
      bounded_wait_geq<false>(p.group_cnt + g, expect, p.err, p.timeout_ns);  // this rank's GEMM (same GPU)
      if (blockIdx.x == 0) {
        fence_acq_rel_sys();
        multimem_red_release_add_u32(p.counter_mc, 1u);
      }
      bounded_wait_geq<true>(p.counter_local, p.base + (uint32_t)(p.ranks * (g + 1)), p.err, p.timeout_ns);
    }
    __syncthreads();
    const int c0 = cb0 * p.bn, c1 = min(cb1 * p.bn, p.n);
    const int cpr = (c1 - c0) / 8;
    const long long total = (long long)rows * cpr;
    constexpr int U = 4;
    for (long long base = (long long)blockIdx.x * kReduceThreads * U + threadIdx.x; base < total;
         base += (long long)gridDim.x * kReduceThreads * U) {
      uint32_t v[U][4];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long i = base + (long long)k * kReduceThreads;
        if (i < total) {
          const long long r = i / cpr, c = i - r * cpr;
          multimem_ld_reduce_bf16x8(p.mc + (r0 + r) * p.ldd + c0 + c * 8, v[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long i = base + (long long)k * kReduceThreads;
        if (i < total) {
          const long long r = i / cpr, c = i - r * cpr;
          multimem_st_bf16x8(p.mc + (r0 + r) * p.ldd + c0 + c * 8, v[k]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    multimem_red_release_add_u32(p.counter_mc, 1u);
  }
}

__global__ void allreduce_wait_kernel(const uint32_t* counter, uint32_t target, uint32_t* err,
                                      unsigned long long timeout_ns) {
  bounded_wait_geq<true>(counter, target, err, timeout_ns);
}

// Dynamic tile scheduler. The pair leader's producer draws work items from a global ticket counter
// (each pair's first item is its static one) and publishes each into a kSchedDepth-deep ring in both
// CTAs of the pair: st.async into each CTA's slot completing on that CTA's `full` mbarrier (one
// arrival = that CTA's producer's expect_tx). Consumers — the MMA issuer, the epilogue warps and the
// peer's producer — read the slot and hand it back on the leader's `empty` mbarrier. Items are handed
// out in raster order as units free up, so the CTAs that share an operand tile start it together and
// read it from L2 once (static round-robin let pairs drift apart over the waves: the fc1 forward read
// 3.2x its operands from DRAM).
constexpr int kSchedDepth = 4;
struct Sched {
  uint64_t* full;
  uint64_t* empty;
  int* slot;
};

__device__ __forceinline__ uint32_t mapa_cta(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void st_async_s32(uint32_t addr, int v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.s32 [%0], %1, [%2];" ::"r"(addr), "r"(v),
               "r"(bar)
               : "memory");
}

template <bool kPair>
__device__ __forceinline__ void sched_publish(const Sched& sc, int i, int w) {
  const int s = i & (kSchedDepth - 1);
  mbar_wait(smem_u32(&sc.empty[s]), ((i / kSchedDepth) & 1) ^ 1);
  const uint32_t full = smem_u32(&sc.full[s]), slot = smem_u32(&sc.slot[s]);
  if (kPair) {
    mbar_arrive_expect_tx(full, 4);
    st_async_s32(mapa_cta(slot, 0), w, mapa_cta(full, 0));
    st_async_s32(mapa_cta(slot, 1), w, mapa_cta(full, 1));
  } else {
    *reinterpret_cast<volatile int*>(&sc.slot[s]) = w;
    mbar_arrive(full);  // release.cta: the slot store is visible to the waiters
  }
}

// expect: the peer CTA's producer (the one arrival on its own `full` barrier).
template <bool kPair>
__device__ __forceinline__ int sched_take(const Sched& sc, int i, bool expect, uint32_t rank) {
  const int s = i & (kSchedDepth - 1);
  const uint32_t full = smem_u32(&sc.full[s]);
  if (expect) mbar_arrive_expect_tx(full, 4);
  mbar_wait(full, (i / kSchedDepth) & 1);
  const int w = *reinterpret_cast<volatile int*>(&sc.slot[s]);
  if (w != INT_MIN) {  // predicated on the loaded value: the hand-back cannot overtake the read
    const uint32_t e = smem_u32(&sc.empty[s]);
    if (!kPair || rank == 0)
      mbar_arrive(e);
    else
      mbar_arrive_cluster_relaxed(e, 0);
  }
  return w;
}

template <int BN, bool kAMN, bool kBMN, bool kPair, bool kAR>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                      const __grid_constant__ CUtensorMap tmap_d, const __grid_constant__ CUtensorMap tmap_aux,
                      const GemmParams p) {
  using C = Cfg<BN, kPair>;
  constexpr int BMT = C::kTileM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint8_t* epi_base = smem + C::kStages * C::kStageBytes;  // 1024-aligned (stage bytes are 1 KB multiples)
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_base + C::kEpiBytes);
  // bars[0..S) full, bars[S..2S) empty, bars[2S..2S+2) tmem_full, bars[2S+2..2S+4) tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4);
  volatile int* split_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
  Sched sc;
  sc.full = bars + 2 * C::kStages + 6;  // after tmem_slot / split_flag (8 bytes)
  sc.empty = sc.full + kSchedDepth;
  sc.slot = reinterpret_cast<int*>(sc.empty + kSchedDepth);
  const bool dyn = p.tile_ctr != nullptr;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = kPair ? cluster_ctarank() : 0;  // position in the CTA pair
  const bool leader = rank == 0;
  const int t_first = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int t_stride = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    tma_prefetch_desc(&tmap_d);
    if (p.epilogue == MT_EPI_BIAS_GELU) tma_prefetch_desc(&tmap_aux);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);
      mbar_init(smem_u32(&bars[C::kStages + s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&bars[2 * C::kStages + a]), 1);
      mbar_init(smem_u32(&bars[2 * C::kStages + 2 + a]), kPair ? 8 : 4);  // epilogue warps (of both CTAs)
    }
    for (int s = 0; s < kSchedDepth; ++s) {
      mbar_init(smem_u32(&sc.full[s]), 1);
      // MMA issuer + 4 epilogue warps (+ the peer's producer and 4 epilogue warps)
      mbar_init(smem_u32(&sc.empty[s]), kPair ? 10 : 5);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (kPair)
      tmem_alloc_pair<C::kTmemCols>(smem_u32(tmem_slot));
    else
      tmem_alloc<C::kTmemCols>(smem_u32(tmem_slot));
  }
  tc_fence_before();
  if (kPair)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      // bytes landing per stage on the (leader's) full barrier: both CTAs' halves in pair mode
      constexpr uint32_t kTx = (C::kABytes + (kBMN ? C::kBBytes : C::kBRows * kBK * 2)) * (kPair ? 2 : 1);
      // The operand re-read across the raster sweep is kept in L2 (evict_last); the one whose tile is
      // shared by the concurrently resident CTAs streams through once (evict_first).
      // hints == 2: only the re-read operand is marked evict_last (the streamed one stays normal, so
      // concurrently resident CTAs sharing its tiles still hit L2)
      const uint64_t pol_a = !p.hints ? kEvictNormal
                                      : (p.n_fastest ? (p.hints == 2 ? kEvictNormal : kEvictFirst) : kEvictLast);
      const uint64_t pol_b = !p.hints ? kEvictNormal
                                      : (p.n_fastest ? kEvictLast : (p.hints == 2 ? kEvictNormal : kEvictFirst));
      uint32_t stage = 0, phase = 0;
      int ticket = 0;  // the next dynamic ticket, drawn one item ahead
      for (int i = 0;; ++i) {
        int w;
        if (!dyn) {
          w = t_first + i * t_stride;
        } else if (leader) {
          if (i == 0) {
            w = t_first;
          } else {
            w = t_stride + ticket;
            if (ticket == p.sched_fetches - 1) *reinterpret_cast<volatile int*>(p.tile_ctr) = 0;  // last ticket
          }
          sched_publish<kPair>(sc, i, w);
          if (w < p.work_items) ticket = atomicAdd(p.tile_ctr, 1);
        } else {
          w = sched_take<kPair>(sc, i, true, rank);
        }
        if (w >= p.work_items) break;
        Work wk;
        if (!get_work<BN, BMT>(p, w, wk)) continue;
        const int b = wk.b, mb = wk.mb, nb = wk.nb;
        for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
          mbar_wait(smem_u32(&bars[C::kStages + stage]), phase ^ 1);
          const uint32_t full = smem_u32(&bars[stage]);
          if (leader) mbar_arrive_expect_tx(full, kTx);
          const uint32_t sa = smem_u32(stage_base + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
          const int m_off = mb * BMT + (int)rank * kBM;        // this CTA's 128 rows of A
          const int n_off = nb * BN + (int)rank * C::kBRows;   // this CTA's rows of B
          auto load = [&](uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t pol) {
            if (kPair)
              tma_load_3d_pair(dst, map, full, c0, c1, b, pol);
            else
              tma_load_3d(dst, map, full, c0, c1, b, pol);
          };
          if (kAMN) {
            load(sa, &tmap_a, m_off, kb * kBK, pol_a);
            load(sa + 8192, &tmap_a, m_off + 64, kb * kBK, pol_a);
          } else {
            load(sa, &tmap_a, kb * kBK, m_off, pol_a);
          }
          if (kBMN) {
#pragma unroll
            for (int c = 0; c < C::kBNAlloc / 64; ++c) load(sb + c * 8192, &tmap_b, n_off + c * 64, kb * kBK, pol_b);
          } else {
            load(sb, &tmap_b, kb * kBK, n_off, pol_b);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------------ MMA issuer (pair leader only)
      constexpr uint32_t idesc = umma_idesc_bf16(BMT, BN, kAMN ? 1 : 0, kBMN ? 1 : 0);
      uint32_t stage = 0, phase = 0, it = 0;
      for (int i = 0;; ++i) {
        const int w = dyn ? sched_take<kPair>(sc, i, false, 0) : t_first + i * t_stride;
        if (w >= p.work_items) break;
        Work wk;
        if (!get_work<BN, BMT>(p, w, wk)) continue;
        const int kb0 = wk.kb0, kb1 = wk.kb1;
        const uint32_t acc = it & 1, acc_phase = (it >> 1) & 1;
        mbar_wait(smem_u32(&bars[2 * C::kStages + 2 + acc]), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::kAccStride;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&bars[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(stage_base + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = kAMN ? umma_desc_sw128(sa + kk * 2048, 8192, 1024) : umma_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bd = kBMN ? umma_desc_sw128(sb + kk * 2048, 8192, 1024) : umma_desc_sw128(sb + kk * 32, 16, 1024);
            if (kPair)
              umma_bf16_pair(d_tmem, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            else
              umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          if (kPair)
            tc_commit_pair_mc(smem_u32(&bars[C::kStages + stage]), 0x3);  // frees the stage in both CTAs
          else
            tc_commit(smem_u32(&bars[C::kStages + stage]));
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (kPair)
          tc_commit_pair_mc(smem_u32(&bars[2 * C::kStages + acc]), 0x3);
        else
          tc_commit(smem_u32(&bars[2 * C::kStages + acc]));
        ++it;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const uint32_t quad = warp - 4;
    const uint32_t stg = smem_u32(epi_base) + quad * (C::kEpiBufs * 4096);  // kEpiBufs 4 KB staging buffers
    uint32_t bi = 0;
    const int ep = p.epilogue;
    const bool f32 = ep == MT_EPI_STORE_F32 || ep == MT_EPI_ACCUM_F32;
    const float alpha = p.alpha;
    uint32_t it = 0;
    // fused all-reduce: the previous tile, published once this tile's stores were issued
    int unpublished = -1;
    for (int i = 0;; ++i) {
      int w = t_first + i * t_stride;
      if (dyn) {
        int v = 0;
        if (lane == 0) v = sched_take<kPair>(sc, i, false, rank);
        w = __shfl_sync(0xffffffffu, v, 0);
      }
      if (w >= p.work_items) break;
      Work wk;
      if (!get_work<BN, BMT>(p, w, wk)) continue;
      const int b = wk.b, mb = wk.mb, nb = wk.nb;
      const uint32_t acc = it & 1, acc_phase = (it >> 1) & 1;
      mbar_wait(smem_u32(&bars[2 * C::kStages + acc]), acc_phase);
      tc_fence_after();
      const int row0 = mb * BMT + (int)rank * kBM + quad * 32;
      const int row = row0 + lane;
      const uint32_t tmem_row = tmem_base + ((quad * 32) << 16) + acc * C::kAccStride;
      const float* parts = nullptr;  // split-K: this CTA's partial tiles of the tail tile
      if (wk.split >= 0) {
        // Publish this split's raw partial (rows of this thread), then count arrivals; the last
        // arriving split reduces the others' partials into its accumulator and runs the epilogue.
        float* base = p.split_ws + (size_t)(wk.tail * p.splits) * 2 * (128 * BN);
        float* mine = base + ((size_t)wk.split * 2 + rank) * (128 * BN) + (size_t)(quad * 32 + lane) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_row + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(reinterpret_cast<float4*>(mine + c * 32 + 4 * j),
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                               __uint_as_float(r[4 * j + 3])));
        }
        __threadfence();
        epi_bar();
        if (threadIdx.x == 128) {
          const int old = atomicAdd(&p.split_cnt[wk.tail * 2 + rank], 1);
          *split_flag = (old == p.splits - 1) ? 1 : 0;
          if (old == p.splits - 1) p.split_cnt[wk.tail * 2 + rank] = 0;  // reset for the next launch
        }
        epi_bar();
        const bool last = *split_flag != 0;
        if (!last) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (kPair)
              tmem_release_arrive(smem_u32(&bars[2 * C::kStages + 2 + acc]));
            else
              mbar_arrive(smem_u32(&bars[2 * C::kStages + 2 + acc]));
          }
          ++it;
          continue;
        }
        __threadfence();
        parts = base + (size_t)rank * (128 * BN) + (size_t)(quad * 32 + lane) * BN;
      }
      // bf16 outputs with BN % 64 == 0: 64-column pieces (32 rows x 128 B, half the TMA stores,
      // fences and warp syncs of 32-column pieces); fp32 outputs and BN = 160 use 32-column pieces
      constexpr bool kWide = (BN % 64) == 0;
      const int c_begin = (kWide && !f32) ? BN / 32 : 0;
      // Accumulator reads are software-pipelined: the next piece's tcgen05.ld is in flight while this
      // piece is scaled, packed, staged and stored (the epilogue is one warp per SMSP, latency-bound).
      #if defined(MT_GEMM_NO_LDPIPE) && MT_GEMM_NO_LDPIPE
      constexpr bool kLdPipe = false;
#else
      constexpr bool kLdPipe = true;
#endif
      if (kWide && !f32) {
        uint32_t ra[32], rb[32];
        if (parts == nullptr) {
          tmem_ld_32x32b_x32(tmem_row, ra);
          tmem_ld_32x32b_x32(tmem_row + 32, rb);
        }
#pragma unroll 1
        for (int c2 = 0; c2 < BN / 64; ++c2) {
          const int col0 = nb * BN + c2 * 64;
          if (col0 >= p.n) break;
          float x[64];
          if (parts == nullptr) {
            if (!kLdPipe && c2 > 0) {
              tmem_ld_32x32b_x32(tmem_row + c2 * 64, ra);
              tmem_ld_32x32b_x32(tmem_row + c2 * 64 + 32, rb);
            }
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              x[j] = __uint_as_float(ra[j]);
              x[32 + j] = __uint_as_float(rb[j]);
            }
            if (kLdPipe && c2 + 1 < BN / 64 && col0 + 64 < p.n) {
              tmem_ld_32x32b_x32(tmem_row + (c2 + 1) * 64, ra);
              tmem_ld_32x32b_x32(tmem_row + (c2 + 1) * 64 + 32, rb);
            }
          } else {
            // split-K tail: the fixed-order sum of every split's published partial (this split's own
            // included), so the result does not depend on which split arrived last
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = 0.f;
            for (int sp = 0; sp < p.splits; ++sp) {
              const float* q = parts + (size_t)sp * 2 * (128 * BN) + c2 * 64;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(q + 4 * j));
                x[4 * j] += v.x;
                x[4 * j + 1] += v.y;
                x[4 * j + 2] += v.z;
                x[4 * j + 3] += v.w;
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] *= alpha;
          if (ep == MT_EPI_STORE_BF16 || ep == MT_EPI_BIAS_GELU) {
            if (p.bias != nullptr) {
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                if (col0 + 8 * v < p.n) {
                  const uint4 bv = __ldg(reinterpret_cast<const uint4*>(p.bias + col0 + 8 * v));
                  const uint32_t bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const float2 f = unpack_bf16x2(bw[q]);
                    x[8 * v + 2 * q] += f.x;
                    x[8 * v + 2 * q + 1] += f.y;
                  }
                }
              }
            }
            if (ep == MT_EPI_BIAS_GELU) {
              reuse_wait<C::kEpiBufs>(lane);
              stage_bf16_wide(stg + bi * 4096, lane, x);
              flush_piece(&tmap_aux, stg + bi * 4096, lane, col0, row0, 0, false);
              bi = (bi + 1) % C::kEpiBufs;
#pragma unroll
              for (int j = 0; j < 64; j += 2) {
                const float2 pr = unpack_bf16x2(pack_bf16x2(x[j], x[j + 1]));
                x[j] = gelu_tanh(pr.x);
                x[j + 1] = gelu_tanh(pr.y);
              }
            }
          } else {  // MT_EPI_GELU_BWD
            if (row < p.m) {
              const __nv_bfloat16* ap = p.aux + (long long)row * p.ld_aux + col0;
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                if (col0 + 8 * v < p.n) {
                  const uint4 av = *reinterpret_cast<const uint4*>(ap + 8 * v);
                  const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const float2 f = unpack_bf16x2(aw[q]);
                    x[8 * v + 2 * q] *= gelu_tanh_grad(f.x);
                    x[8 * v + 2 * q + 1] *= gelu_tanh_grad(f.y);
                  }
                }
              }
            }
          }
          reuse_wait<C::kEpiBufs>(lane);
          stage_bf16_wide(stg + bi * 4096, lane, x);
          flush_piece(&tmap_d, stg + bi * 4096, lane, col0, row0, b, false);
          bi = (bi + 1) % C::kEpiBufs;
        }
      }
      uint32_t rn[32];
      if (parts == nullptr && c_begin < BN / 32) tmem_ld_32x32b_x32(tmem_row + c_begin * 32, rn);
#pragma unroll 1
      for (int c = c_begin; c < BN / 32; ++c) {
        const int col0 = nb * BN + c * 32;
        if (col0 >= p.n) break;
        float x[32];
        if (parts == nullptr) {
          if (!kLdPipe && c > c_begin) tmem_ld_32x32b_x32(tmem_row + c * 32, rn);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(rn[j]);
          if (kLdPipe && c + 1 < BN / 32 && col0 + 32 < p.n) tmem_ld_32x32b_x32(tmem_row + (c + 1) * 32, rn);
        } else {  // split-K tail: fixed-order sum of all splits' partials (see the 64-column path)
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] = 0.f;
          for (int sp = 0; sp < p.splits; ++sp) {
            const float* q = parts + (size_t)sp * 2 * (128 * BN) + c * 32;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v = __ldcg(reinterpret_cast<const float4*>(q + 4 * j));
              x[4 * j] += v.x;
              x[4 * j + 1] += v.y;
              x[4 * j + 2] += v.z;
              x[4 * j + 3] += v.w;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] *= alpha;
        if (f32) {
          reuse_wait<C::kEpiBufs>(lane);
          stage_f32(stg + bi * 4096, lane, x);
          flush_piece(&tmap_d, stg + bi * 4096, lane, col0, row0, b, ep == MT_EPI_ACCUM_F32, p.store_policy);
          bi = (bi + 1) % C::kEpiBufs;
          continue;
        }
        if (ep == MT_EPI_STORE_BF16 || ep == MT_EPI_BIAS_GELU) {
          if (p.bias != nullptr) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if (col0 + 8 * v < p.n) {
                const uint4 bv = __ldg(reinterpret_cast<const uint4*>(p.bias + col0 + 8 * v));
                const uint32_t bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float2 f = unpack_bf16x2(bw[q]);
                  x[8 * v + 2 * q] += f.x;
                  x[8 * v + 2 * q + 1] += f.y;
                }
              }
            }
          }
          if (ep == MT_EPI_BIAS_GELU) {
            // pre-activation (bf16) goes to aux; GeLU is applied to the rounded value the backward sees
            reuse_wait<C::kEpiBufs>(lane);
            stage_bf16(stg + bi * 4096, lane, x);
            flush_piece(&tmap_aux, stg + bi * 4096, lane, col0, row0, 0, false);
            bi = (bi + 1) % C::kEpiBufs;
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float2 pr = unpack_bf16x2(pack_bf16x2(x[j], x[j + 1]));
              x[j] = gelu_tanh(pr.x);
              x[j + 1] = gelu_tanh(pr.y);
            }
          }
        } else {  // MT_EPI_GELU_BWD: D = acc * gelu'(aux)
          if (row < p.m) {
            const __nv_bfloat16* ap = p.aux + (long long)row * p.ld_aux + col0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if (col0 + 8 * v < p.n) {
                const uint4 av = *reinterpret_cast<const uint4*>(ap + 8 * v);
                const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float2 f = unpack_bf16x2(aw[q]);
                  x[8 * v + 2 * q] *= gelu_tanh_grad(f.x);
                  x[8 * v + 2 * q + 1] *= gelu_tanh_grad(f.y);
                }
              }
            }
          }
        }
        reuse_wait<C::kEpiBufs>(lane);
        stage_bf16(stg + bi * 4096, lane, x);
        flush_piece(&tmap_d, stg + bi * 4096, lane, col0, row0, b, false);
        bi = (bi + 1) % C::kEpiBufs;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair)
          tmem_release_arrive(smem_u32(&bars[2 * C::kStages + 2 + acc]));  // the leader's tmem_empty
        else
          mbar_arrive(smem_u32(&bars[2 * C::kStages + 2 + acc]));
      }
      ++it;
      if (kAR && p.ar_group_cols > 0) {
        // bulk groups of the tile issued after `unpublished` (64-column bf16 pieces when BN % 64 == 0)
        if (unpublished >= 0) ar_publish<(BN % 64 == 0) ? BN / 64 : BN / 32>(p, unpublished, lane);
        unpublished = w;
      }
    }
    if (kAR && p.ar_group_cols > 0 && unpublished >= 0) ar_publish<0>(p, unpublished, lane);
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  if (kPair)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (kPair)
      tmem_dealloc_pair<C::kTmemCols>(tmem_base);
    else
      tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  return fn;
}

// 3-D tensor map: dims (inner, outer, batch) with element size `esize`, box (box_inner, box_outer, 1).
bool make_map_ex(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t batch, uint64_t ld,
                 uint64_t batch_stride, uint32_t box_inner, uint32_t box_outer, bool f32, CUtensorMapSwizzle swz) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const uint64_t es = f32 ? 4 : 2;
  cuuint64_t dims[3] = {inner, outer, batch};
  uint64_t bs = batch_stride;
  if (batch <= 1) bs = (ld * outer + 7) / 8 * 8;
  if (bs == 0) bs = 8;
  cuuint64_t strides[2] = {ld * es, bs * es};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Operand map: bf16, 128B swizzle, box (64, box_outer).
bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t batch, uint64_t ld,
              uint64_t batch_stride, uint32_t box_outer) {
  return make_map_ex(map, base, inner, outer, batch, ld, batch_stride, 64, box_outer, false,
                     CU_TENSOR_MAP_SWIZZLE_128B);
}

// Epilogue store map: 32 x 32 pieces; bf16 rows are 64 B (64B swizzle), fp32 rows 128 B (128B swizzle).
bool make_store_map(CUtensorMap* map, const void* base, uint64_t n, uint64_t m, uint64_t batch, uint64_t ld,
                    uint64_t batch_stride, bool f32, bool wide = false) {
  if (wide && !f32)  // 64 x 32 bf16 pieces (128 B rows)
    return make_map_ex(map, base, n, m, batch, ld, batch_stride, 64, 32, false, CU_TENSOR_MAP_SWIZZLE_128B);
  return make_map_ex(map, base, n, m, batch, ld, batch_stride, 32, 32, f32,
                     f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

constexpr size_t kSplitCounterBytes = 64 * 1024;  // arrival counters at the head of the workspace

bool split_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MT_GEMM_SPLITK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Shortest K (in 64-wide k-blocks) the split-K tail is used for. Measured per shape on B200
// (tools/gemm_split_ab.sh): +4-7% at K >= 20480 (320+ k-blocks), neutral at K = 12288 (192), and a
// loss below — -5% at K = 9216, -11% at K = 6144, up to -40% at K = 1536 (the TP=8 projection) —
// because the partial-tile round trip does not shrink with K while the tail work it spreads does.
int split_min_kblocks() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MT_GEMM_SPLIT_MINK");
    v = e ? std::max(1, atoi(e)) : 256;
  }
  return v;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// kAR: the fused TP all-reduce variant (only the K-major x K-major row-parallel forward GEMMs use it;
// a separate instantiation so the plain kernels keep their register budget).
template <int BN, bool kAMN, bool kBMN, bool kPair, bool kAR = false>
int launch(const mt_gemm_args& a, cudaStream_t stream) {
  using C = Cfg<BN, kPair>;
  CUtensorMap ma, mb;
  const int m = (int)a.m, n = (int)a.n, k = (int)a.k, batch = (int)a.batch;
  bool ok = kAMN ? make_map(&ma, a.a, m, k, batch, a.lda, a.a_batch_stride, 64)
                 : make_map(&ma, a.a, k, m, batch, a.lda, a.a_batch_stride, kBM);
  ok = ok && (kBMN ? make_map(&mb, a.b, n, k, batch, a.ldb, a.b_batch_stride, 64)
                   : make_map(&mb, a.b, k, n, batch, a.ldb, a.b_batch_stride, C::kBRows));
  const bool f32 = a.epilogue == MT_EPI_STORE_F32 || a.epilogue == MT_EPI_ACCUM_F32;
  CUtensorMap md, maux;
  ok = ok && make_store_map(&md, a.d, n, m, batch, a.ldd, a.d_batch_stride, f32, BN % 64 == 0);
  if (a.epilogue == MT_EPI_BIAS_GELU)
    ok = ok && make_store_map(&maux, a.aux, n, m, 1, a.ld_aux, 0, false, BN % 64 == 0);
  else
    maux = md;
  if (!ok) return 1;
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.batch = batch;
  p.mblocks = (m + C::kTileM - 1) / C::kTileM;
  p.nblocks = (n + BN - 1) / BN;
  p.kblocks = (k + kBK - 1) / kBK;
  p.total_tiles = p.mblocks * p.nblocks * batch;
  // split-K tail (whole-tile work first; the last partial wave's tiles split over idle units)
  const int cap_units = (a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms()) / (kPair ? 2 : 1);
  p.full_tiles = p.total_tiles;
  p.splits = 1;
  p.work_items = p.total_tiles;
  if (a.causal == MT_CAUSAL_NONE && a.workspace != nullptr && a.allreduce == nullptr && split_enabled() &&
      p.kblocks >= split_min_kblocks()) {
    const int units = std::max(1, cap_units);
    const int full = (p.total_tiles / units) * units, tail = p.total_tiles - full;
    if (full > 0 && tail > 0 && tail * 2 <= units) {
      const int splits = std::min({units / tail, p.kblocks / 4, 8});
      const size_t need = kSplitCounterBytes + (size_t)tail * splits * 2 * 128 * BN * sizeof(float);
      if (splits >= 2 && (size_t)a.workspace_bytes >= need && tail * 2 * (int)sizeof(int) <= kSplitCounterBytes - 64) {
        p.full_tiles = full;
        p.splits = splits;
        p.work_items = full + tail * splits;
        p.split_cnt = static_cast<int*>(a.workspace);
        p.split_ws = reinterpret_cast<float*>(static_cast<char*>(a.workspace) + kSplitCounterBytes);
      }
    }
  }
  p.alpha = a.alpha;
  p.epilogue = a.epilogue;
  p.causal = a.causal;
  // Raster so the larger operand is streamed once: concurrently resident CTAs then share the tile
  // of the larger operand, and the smaller operand stays L2-resident across the sweep (e.g. the
  // wgrad of fc1, M = 4h/t >> N = h, would otherwise re-read its 200 MB A operand per n-block).
  p.n_fastest = (m > n) ? 1 : 0;
  // L2 eviction hints on the operand loads (streamed operand evict_first, re-read one evict_last):
  // ~2% faster for the n-fastest wgrad GEMMs; with the dynamic tile scheduler also 1-2% faster for
  // the m-fastest GEMMs up to K = 16384 (fc1 / QKV forward at K = 12288) but 2-4% slower at
  // K = 49152 (tools/hints_dyn_ab.sh), so those keep plain loads. MT_GEMM_HINTS=0/1 forces.
  static const int hints = [] {
    const char* e = getenv("MT_GEMM_HINTS");
    return e ? atoi(e) : -1;
  }();
  static const bool shortk_hints = [] {  // MT_GEMM_SHORTK_HINTS=0: plain loads for every m-fastest GEMM (A/B)
    const char* e = getenv("MT_GEMM_SHORTK_HINTS");
    return !(e && e[0] == '0');
  }();
  const bool short_k = shortk_hints && a.causal == MT_CAUSAL_NONE && p.kblocks <= 256;
  p.hints = hints >= 0 ? hints : ((p.n_fastest || short_k) ? 1 : 0);
  // (direct register->global fp32 stores were measured 8% slower than smem staging + TMA store)
  p.d_bf16 = static_cast<__nv_bfloat16*>(a.d);
  p.d_f32 = static_cast<float*>(a.d);
  p.ldd = a.ldd;
  p.d_batch_stride = a.d_batch_stride;
  p.bias = static_cast<const __nv_bfloat16*>(a.bias);
  p.aux = static_cast<__nv_bfloat16*>(a.aux);
  p.ld_aux = a.ld_aux;
  // fp32 outputs (wgrad) are written once and never re-read by this GEMM: evict_first keeps the
  // re-read operand tiles in L2 (tools/gemm_one.py wg_mm_f32: 1864 -> 1832 us); MT_GEMM_STORE_HINT=0 disables
  static const int store_hint = [] {
    const char* e = getenv("MT_GEMM_STORE_HINT");
    return e ? atoi(e) : 1;
  }();
  p.store_policy = (store_hint == 1) ? kEvictFirst : (store_hint == 2 ? kEvictLast : 0);
  if (a.allreduce != nullptr) {
    // column-group mode: column blocks complete in raster order only when m-blocks vary fastest
    mt_gemm_allreduce& ar = *a.allreduce;
    if (ar.ranks < 2 || ar.ranks > 8 || ar.rank < 0 || ar.rank >= ar.ranks || ar.groups < 1 || ar.groups > 64 ||
        !ar.d_multicast || !ar.group_counters || !ar.counter_multicast || p.n_fastest)
      return 1;
    p.ar_group_cnt = ar.group_counters;
    p.ar_group_cols = (p.nblocks + ar.groups - 1) / ar.groups;
    ar.geom[0] = BN;
    ar.geom[1] = C::kTileM;
    ar.geom[2] = kPair ? 1 : 0;
    ar.geom[3] = p.n_fastest;
    ar.geom[4] = p.mblocks;
    ar.geom[5] = p.nblocks;
    ar.geom[6] = p.m;
    ar.geom[7] = p.n;
    ar.group_cols = p.ar_group_cols;
    ar.units = (long long)p.total_tiles * (kPair ? 2 : 1);
  }
  auto kern = gemm_sm100_kernel<BN, kAMN, kBMN, kPair, kAR>;
  // the dynamic shared-memory opt-in is per device: one bit per device that has it, set by any thread
  // (setting it twice is harmless), so one context per GPU per host thread works in one process
  static std::atomic<uint64_t> attr_devices{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 2;
  const uint64_t bit = uint64_t{1} << (dev & 63);
  if (!(attr_devices.load(std::memory_order_acquire) & bit)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes) != cudaSuccess)
      return 2;
    attr_devices.fetch_or(bit, std::memory_order_release);
  }
  // dynamic tile scheduler: the ticket counter is the last int of the workspace's counter block
  static const bool dyn_sched = [] {
    const char* e = getenv("MT_GEMM_DYNAMIC");
    return !(e && e[0] == '0');
  }();
  auto set_sched = [&](int units) {
    if (!dyn_sched || a.workspace == nullptr) return;
    p.tile_ctr = static_cast<int*>(a.workspace) + kSplitCounterBytes / sizeof(int) - 1;
    p.sched_fetches = std::max(0, p.work_items - units) + std::min(units, p.work_items);
  };
  if (!kPair) {
    const int cap = a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms();
    const int grid = p.work_items < cap ? p.work_items : cap;
    set_sched(grid);
    kern<<<grid, kThreads, C::kSmemBytes, stream>>>(ma, mb, md, maux, p);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  const int cap = a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms();
  const int pairs = std::max(1, std::min(p.work_items, cap / 2));
  set_sched(pairs);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, md, maux, p) != cudaSuccess) return 2;
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

template <int BN, bool kPair>
int dispatch_major(const mt_gemm_args& a, cudaStream_t s) {
  if (a.a_mn_major)
    return a.allreduce != nullptr ? 1
           : a.b_mn_major        ? launch<BN, true, true, kPair>(a, s)
                                 : launch<BN, true, false, kPair>(a, s);
  if (a.allreduce != nullptr) return a.b_mn_major ? 1 : launch<BN, false, false, kPair, true>(a, s);
  return a.b_mn_major ? launch<BN, false, true, kPair>(a, s) : launch<BN, false, false, kPair>(a, s);
}

bool pair_enabled();

bool use_pair(const mt_gemm_args& a, int bn) {
  return pair_enabled() && a.m >= 256 && (bn == 128 || bn == 192 || bn == 256);
}

// Tile width: N <= 64/128 and the head dim 160 map directly; otherwise pick the width whose last
// wave of (pair) tiles is fullest, weighted by the measured per-tile rate of narrower tiles
// (tools/gemm_ab.sh: BN 192 and 128 run at 87% and 68% of BN 256's rate, so 256 nearly always wins;
// the last-wave loss, e.g. N = 12288 at M = 2048 -> 384 tiles = 5.19 waves of 74 pairs, is left to
// a split-K tail).
int choose_block_n(const mt_gemm_args& a) {
  if (a.n <= 64) return 64;
  if (a.n <= 128) return 128;
  if (a.n == 160) return 160;
  const int units = pair_enabled() && a.m >= 256 ? num_sms() / 2 : num_sms();
  const int tile_m = pair_enabled() && a.m >= 256 ? 256 : 128;
  const long long mblocks = (a.m + tile_m - 1) / tile_m;
  const int cand[3] = {256, 192, 128};
  const double weight[3] = {1.0, 0.87, 0.68};  // measured per-tile rates relative to BN = 256 (B200)
  int best = 256;
  double best_eff = -1.0;
  for (int i = 0; i < 3; ++i) {
    const long long tiles = mblocks * ((a.n + cand[i] - 1) / cand[i]) * a.batch;
    const long long waves = (tiles + units - 1) / units;
    const double eff = weight[i] * double(tiles) / double(waves * units);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = cand[i];
    }
  }
  return best;
}

bool pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MT_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

}  // namespace
}  // namespace mt

extern "C" int mt_gemm_launches_per_call(void) { return 1; }

extern "C" int mt_gemm_allreduce_reduce_groups(const mt_gemm_allreduce* ar, int64_t ldd, uint32_t* group_counters,
                                               const uint32_t* counter_local, uint32_t base, int32_t ctas,
                                               void* stream) {
  if (ar == nullptr || group_counters == nullptr || counter_local == nullptr || ctas < 1 || ar->group_cols <= 0 ||
      ar->ranks < 2 || ar->geom[6] % ar->ranks != 0 || ar->timeout_ns == 0)
    return 1;
  mt::ArGroupParams p{};
  p.mc = static_cast<__nv_bfloat16*>(ar->d_multicast);
  p.group_cnt = group_counters;
  p.counter_mc = ar->counter_multicast;
  p.counter_local = counter_local;
  p.base = base;
  p.rank = ar->rank;
  p.ranks = ar->ranks;
  p.group_cols = (int)ar->group_cols;
  p.bn = (int)ar->geom[0];
  p.units_per_block = ar->geom[2] ? 2 : 1;
  p.mblocks = (int)ar->geom[4];
  p.m = (int)ar->geom[6];
  p.n = (int)ar->geom[7];
  p.groups = ((int)ar->geom[5] + p.group_cols - 1) / p.group_cols;
  p.ldd = ldd;
  p.err = ar->error_flag;
  p.timeout_ns = ar->timeout_ns;
  mt::allreduce_group_kernel<<<ctas, mt::kReduceThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int mt_gemm_allreduce_wait(const mt_gemm_allreduce* ar, const uint32_t* counter_local, uint32_t target,
                                      void* stream) {
  if (ar == nullptr || counter_local == nullptr || ar->timeout_ns == 0) return 1;
  mt::allreduce_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(counter_local, target, ar->error_flag,
                                                                            ar->timeout_ns);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int mt_gemm(const mt_gemm_args* args, void* stream) {
  if (args == nullptr) return 1;
  const mt_gemm_args& a = *args;
  if (a.m <= 0 || a.n <= 0 || a.k <= 0 || a.batch <= 0) return 1;
  if (a.a == nullptr || a.b == nullptr || a.d == nullptr) return 1;
  if ((a.n % 8) != 0 || (a.lda % 8) != 0 || (a.ldb % 8) != 0 || (a.ldd % 8) != 0) return 1;
  if ((a.a_batch_stride % 8) != 0 || (a.b_batch_stride % 8) != 0 || (a.d_batch_stride % 8) != 0) return 1;
  if ((reinterpret_cast<uintptr_t>(a.a) | reinterpret_cast<uintptr_t>(a.b) | reinterpret_cast<uintptr_t>(a.d)) & 15)
    return 1;
  if ((a.epilogue == MT_EPI_BIAS_GELU || a.epilogue == MT_EPI_GELU_BWD) && (a.aux == nullptr || a.ld_aux % 8))
    return 1;
  if (a.epilogue == MT_EPI_BIAS_GELU && a.bias == nullptr) return 1;
  if ((a.epilogue == MT_EPI_BIAS_GELU || a.epilogue == MT_EPI_GELU_BWD) && a.batch != 1) return 1;
  if (a.allreduce != nullptr && (a.epilogue != MT_EPI_STORE_BF16 || a.batch != 1 || a.causal != MT_CAUSAL_NONE))
    return 1;
  if (a.epilogue < 0 || a.epilogue > MT_EPI_ACCUM_F32 || a.causal < 0 || a.causal > MT_CAUSAL_K_GE_M) return 1;
  int bn = a.block_n;
  if (bn == 0) bn = mt::choose_block_n(a);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // 2-CTA 256-row tiles whenever M fills them; 1-CTA 128-row tiles otherwise.
  const bool pair = mt::use_pair(a, bn);
  switch (bn) {
    case 64:
      return mt::dispatch_major<64, false>(a, s);
    case 128:
      return pair ? mt::dispatch_major<128, true>(a, s) : mt::dispatch_major<128, false>(a, s);
    case 160:
      return mt::dispatch_major<160, false>(a, s);
    case 192:
      return pair ? mt::dispatch_major<192, true>(a, s) : mt::dispatch_major<192, false>(a, s);
    case 256:
      return pair ? mt::dispatch_major<256, true>(a, s) : mt::dispatch_major<256, false>(a, s);
    default:
      return 1;
  }
}
