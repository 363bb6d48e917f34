// Fused causal attention (flash-style) on tcgen05 for sm_100a: the scaled-masked-softmax attention of
// the tensor-sliced layer (Megatron's fused scale-mask-softmax) without the
// [s x s] score / probability round trips through HBM.
//
// Forward, one CTA per (head, 128-query block), 256 threads:
//   warp 0      TMA producer: Q once, then K_j / V_j blocks (double-buffered)
//   warp 1      MMA issuer  : S_j = Q K_j^T into one of two TMEM score buffers (S_{j+1} overlaps the
//                             softmax of S_j), then O += P_j V_j into the TMEM output accumulator
//   warp 2      TMEM allocator
//   warps 4..7  softmax     : one query row per thread; online softmax in the log2 domain with a lazy
//                             rescale of O (only when the running max grows by > 8, i.e. 256x),
//                             attention dropout from the shared counter-based mask
//                             (include/curator/dropout.hpp), P_j written to smem as the bf16 A
//                             operand of the PV MMA; final O / l -> bf16 ctx, and the row LSE.
// Semantics match the unfused path: P = dropout(softmax(alpha * Q K^T)) with alpha = 1/sqrt(hd),
// ctx = P V, lse = log-sum-exp of alpha * Q K^T (natural log), causal (j <= i).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "curator/dropout.hpp"
#include "sm100_ptx.cuh"

namespace mt {
namespace {

constexpr int kAttnThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;

template <int HD>
struct AttnCfg {
  static constexpr int kChunks = (HD + 63) / 64;    // 64-wide head-dim chunks (128 B rows, SW128)
  static constexpr int kTileBytes = kChunks * 16384;  // 128 rows x kChunks x 128 B
  static constexpr int kPBytes = 2 * 16384;           // P: 128 x 128 bf16 (two 64-col chunks)
  // smem: Q, K[2], V[kVBuf], P
  static constexpr int kVBuf = (HD > 128) ? 1 : 2;
  static constexpr int kSmem = 1024 + kTileBytes * (1 + 2 + kVBuf) + kPBytes + 512;
  static constexpr uint32_t kTmemCols = 512;  // S0 [0,128), S1 [128,256), O [256, 256+HD)
  static constexpr uint32_t kOCol = 256;
};

struct AttnParams {
  int seq, nqb;           // sequence length, number of 128-row query blocks
  int heads;              // heads handled by this launch (grid.y)
  long long head_base;    // global (microbatch row, head) id of head 0 (dropout element index)
  float alpha_log2;       // alpha * log2(e)
  uint64_t seed;
  uint32_t thresh16;
  float drop_scale;       // 1 / (1 - p)
  __nv_bfloat16* out;     // ctx: row i, head h at out + i * ld_out + h * out_head_stride
  long long ld_out, out_head_stride;
  float* lse;             // [heads][seq]
  int group_heads;        // attn_fwd2_kernel: heads per launch-order group (as the one-kernel backward)
  int balanced;           // attn_fwd2_kernel: pair query blocks (p, nqb - 1 - p) instead of (2p, 2p + 1)
  uint32_t* mask;         // optional attention-dropout keep bits [heads][seq][seq / 32] (bit c % 32 of word
                          // c / 32 = score (row, c) kept); written for the causal blocks only
};

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Row r's 16-byte chunk j (of 8 bf16) inside a 128-row, 128 B-per-row SW128 tile.
__device__ __forceinline__ uint32_t sw128_addr(uint32_t base, uint32_t r, uint32_t j) {
  return base + r * 128 + ((j ^ (r & 7)) << 4);
}

// Attention-dropout stream in Weyl form (curator::dropout_bits(site, g) = splitmix64(site + g*gamma)):
// consecutive groups of 4 scores are one 64-bit add apart.
__device__ __forceinline__ uint64_t drop_weyl_attn(uint64_t site, uint64_t group) {
  return site + (group + 1) * curator::kSplitMixGamma;
}
// pv[t] = keep_t ? e[t] : 0 for the 8 scores of groups (z, z + gamma) (16-bit field t & 3 >= thresh16).
// Returns the 8 keep bits (bit t = score t kept).
__device__ __forceinline__ uint32_t drop_select8(uint64_t z, uint32_t thresh16, const float (&e)[8], float (&pv)[8]) {
  uint32_t keep = 0;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    uint64_t b = z + (uint64_t)g * curator::kSplitMixGamma;
    b = (b ^ (b >> 30)) * 0xbf58476d1ce4e5b9ull;
    b = (b ^ (b >> 27)) * 0x94d049bb133111ebull;
    b ^= b >> 31;
    const uint32_t lo = (uint32_t)b, hi = (uint32_t)(b >> 32);
    const uint32_t u[4] = {lo & 0xffffu, lo >> 16, hi & 0xffffu, hi >> 16};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool k = u[q] >= thresh16;
      pv[4 * g + q] = k ? e[4 * g + q] : 0.f;
      keep |= (k ? 1u : 0u) << (4 * g + q);
    }
  }
  return keep;
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  using C = AttnCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK = sQ + C::kTileBytes;                 // 2 buffers
  const uint32_t sV = sK + 2 * C::kTileBytes;             // kVBuf buffers
  const uint32_t sP = sV + C::kVBuf * C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kTileBytes * (3 + C::kVBuf) + C::kPBytes);
  // barriers
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2] S_j ready in TMEM
  uint64_t* s_free = bars + 11;  // [2] softmax finished reading S buffer
  uint64_t* p_full = bars + 13;  // P_j in smem (and O rescaled)
  uint64_t* o_done = bars + 14;  // PV_j complete (P smem free, O stable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const uint32_t warp = warp_id(), lane = lane_id();
  // grid (heads, blocks): the launch order runs every head's heaviest block (most kv blocks) first, so
  // the last CTAs to start are the light ones (a head-major order left heavy CTAs for the tail)
  const int qb = p.nqb - 1 - (int)blockIdx.y;
  const int head = blockIdx.x;
  const int nkv = qb + 1;                       // causal: kv blocks 0..qb

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    mbar_init(smem_u32(q_full), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(k_full + i), 1);
      mbar_init(smem_u32(k_empty + i), 1);
      mbar_init(smem_u32(v_full + i), 1);
      mbar_init(smem_u32(v_empty + i), 1);
      mbar_init(smem_u32(s_full + i), 1);
      mbar_init(smem_u32(s_free + i), 4);
    }
    mbar_init(smem_u32(p_full), 4);
    mbar_init(smem_u32(o_done), 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(smem_u32(q_full), C::kTileBytes);
      for (int c = 0; c < C::kChunks; ++c) tma_load_3d(sQ + c * 16384, &tq, smem_u32(q_full), c * 64, qb * 128, head);
      for (int j = 0; j < nkv; ++j) {
        const int kb = j & 1, kph = (j >> 1) & 1;
        mbar_wait(smem_u32(k_empty + kb), kph ^ 1);
        mbar_arrive_expect_tx(smem_u32(k_full + kb), C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(sK + kb * C::kTileBytes + c * 16384, &tk, smem_u32(k_full + kb), c * 64, j * 128, head);
        const int vb = C::kVBuf == 2 ? (j & 1) : 0;
        const int vph = C::kVBuf == 2 ? ((j >> 1) & 1) : (j & 1);
        mbar_wait(smem_u32(v_empty + vb), vph ^ 1);
        mbar_arrive_expect_tx(smem_u32(v_full + vb), C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(sV + vb * C::kTileBytes + c * 16384, &tv, smem_u32(v_full + vb), c * 64, j * 128, head);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, 0, 0);  // Q (K-major) x K_j (K-major)
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, HD, 0, 1);   // P (K-major) x V_j (MN-major)
      mbar_wait(smem_u32(q_full), 0);
      auto issue_s = [&](int j) {
        const int kb = j & 1;
        mbar_wait(smem_u32(k_full + kb), (j >> 1) & 1);
        mbar_wait(smem_u32(s_free + kb), ((j >> 1) & 1) ^ 1);  // softmax done with S_{j-2}
        tc_fence_after();
        const uint32_t d = tmem + kb * 128;
#pragma unroll
        for (int kk = 0; kk < C::kChunks * 4; ++kk) {
          if (kk * 16 >= HD) break;
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16(d, umma_desc_sw128(sQ + off, 16, 1024), umma_desc_sw128(sK + kb * C::kTileBytes + off, 16, 1024),
                    idesc_s, kk > 0 ? 1u : 0u);
        }
        tc_commit(smem_u32(k_empty + kb));
        tc_commit(smem_u32(s_full + kb));
      };
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        // O += P_j V_j once softmax has written P_j
        mbar_wait(smem_u32(p_full), j & 1);
        const int vb = C::kVBuf == 2 ? (j & 1) : 0;
        const int vph = C::kVBuf == 2 ? ((j >> 1) & 1) : (j & 1);
        mbar_wait(smem_u32(v_full + vb), vph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 kv positions
          const uint32_t a = sP + (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t b = sV + vb * C::kTileBytes + kk * 2048;
          umma_bf16(tmem + C::kOCol, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16384, 1024), idesc_o,
                    (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(smem_u32(v_empty + vb));
        tc_commit(smem_u32(o_done));
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax / epilogue
    const uint32_t quad = warp - 4;
    const int r = quad * 32 + lane;  // row within the query block (TMEM lane)
    const int qrow = qb * 128 + r;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    float m2 = -INFINITY;  // running (possibly stale) max, log2 domain
    float l = 0.f;         // running sum of exp2(s - m2) over valid, undropped probabilities
    const uint64_t row_idx = ((uint64_t)(p.head_base + head) * p.seq + qrow) * (uint64_t)p.seq;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(smem_u32(s_full + sb), (j >> 1) & 1);
      tc_fence_after();
      float sv[128];
      {
        uint32_t u[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + sb * 128 + c * 32, u[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int t = 0; t < 32; ++t) sv[c * 32 + t] = __uint_as_float(u[c][t]) * p.alpha_log2;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(s_free + sb));
      const bool diag = (j == qb);
      // 8 independent partial maxima (no 128-long dependency chain)
      float pm[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = -INFINITY;
#pragma unroll
      for (int t = 0; t < 128; ++t) {
        if (diag && t > r) sv[t] = -INFINITY;
        pm[t & 7] = fmaxf(pm[t & 7], sv[t]);
      }
      const float bmax = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      // lazy rescale: move the reference max only when it grows by more than 8 (2^8 headroom)
      float corr = 1.f;
      bool rescale = false;
      if (bmax > m2 + 8.f || m2 == -INFINITY) {
        const float mnew = fmaxf(bmax, m2);
        corr = (m2 == -INFINITY) ? 0.f : ex2(m2 - mnew);
        rescale = (m2 != -INFINITY);
        m2 = mnew;
      }
      // probabilities, row sum (8 partial sums) and the dropped bf16 P row, all before waiting on PV_{j-1}
      float ps[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) ps[k] = 0.f;
      uint32_t packed[64];
      const uint64_t col_idx = row_idx + (uint64_t)j * 128;
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        uint32_t keep = 0xffu;
        if (p.thresh16) {
          keep = 0;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const uint64_t bits = curator::dropout_bits(p.seed, (col_idx + g * 8 + h2 * 4) >> 2);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (((bits >> (16 * q)) & 0xffffu) >= p.thresh16) keep |= 1u << (4 * h2 + q);
          }
        }
        float pv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float e = ex2(sv[g * 8 + t] - m2);  // exp2(-inf) = 0 for masked columns
          ps[t] += e;
          pv[t] = ((keep >> t) & 1u) ? e : 0.f;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) packed[g * 4 + t] = pack_bf16x2(pv[2 * t], pv[2 * t + 1]);
      }
      l = l * corr + (((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7])));
      // P buffer and O: wait for PV_{j-1}
      if (j > 0) mbar_wait(smem_u32(o_done), (j - 1) & 1);
      tc_fence_after();
      if (__any_sync(0xffffffffu, rescale)) {
        // O *= corr (rows that did not rescale multiply by 1)
        for (int c = 0; c * 32 < HD; ++c) {
          uint32_t u[32];
          tmem_ld_32x32b_x32(lane_base + C::kOCol + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) u[t] = __float_as_uint(__uint_as_float(u[t]) * corr);
          tmem_st_32x32b_x32(lane_base + C::kOCol + c * 32, u);
        }
        tmem_st_wait();
      }
#pragma unroll
      for (int g = 0; g < 16; ++g)
        st_shared_v4(sw128_addr(sP + (g >> 3) * 16384, r, g & 7), packed[g * 4], packed[g * 4 + 1], packed[g * 4 + 2],
                     packed[g * 4 + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(p_full));
    }
    // epilogue: O / l * dropout scale -> bf16 ctx ; lse
    mbar_wait(smem_u32(o_done), (nkv - 1) & 1);
    tc_fence_after();
    const float inv = p.drop_scale / l;
    __nv_bfloat16* orow = p.out + (long long)qrow * p.ld_out + (long long)head * p.out_head_stride;
    for (int c = 0; c * 32 < HD; ++c) {
      uint32_t u[32];
      tmem_ld_32x32b_x32(lane_base + C::kOCol + c * 32, u);
      tmem_ld_wait();
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        *reinterpret_cast<uint4*>(orow + c * 32 + v * 8) =
            make_uint4(pack_bf16x2(__uint_as_float(u[8 * v]) * inv, __uint_as_float(u[8 * v + 1]) * inv),
                       pack_bf16x2(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv),
                       pack_bf16x2(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv),
                       pack_bf16x2(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv));
      }
    }
    p.lse[(long long)head * p.seq + qrow] = (m2 + __log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem);
}

// ---------------------------------------------------------------- forward, two query tiles per CTA
// attn_fwd2_kernel<HD> (HD <= 128): one CTA per (head, pair of consecutive 128-row query blocks
// qa = 2p, qb = 2p + 1), 384 threads:
//   warp 0        TMA producer: Q_a, Q_b once; then K_j, V_j through a 3-slot ring (K_j, V_j and
//                 K_{j+1} resident together), shared by both query tiles
//   warp 1        MMA issuer:  S_x = Q_x K_j^T into S_x's TMEM columns; O_x += P_x V_j
//   warp 2        TMEM allocator (S_a [0,128), S_b [128,256), O_a [256,384), O_b [384,512))
//   warps 4..7    softmax of tile a, warps 8..11 softmax of tile b (one row per thread)
// The two softmax warpgroups alternate with the tensor core (while one computes exps and the
// dropout mask of block j, the MMAs of the other tile run), which is what the single-tile kernel
// lacked (it was latency-bound, 0.63 ms for the GPT-3 layer's forward attention). Each row's block
// is read from TMEM in two 64-column halves (max, then exp / mask / pack) to stay within the 170
// registers a 384-thread CTA allows. Semantics are attn_fwd_kernel's (online softmax with lazy
// rescale, counter-based attention dropout, lse in natural log).
template <int HD>
struct Fwd2Cfg {
  static constexpr int kChunks = (HD + 63) / 64;
  static constexpr int kTileBytes = kChunks * 16384;
  static constexpr int kPBytes = 2 * 16384;
  static constexpr int kRing = 3;
  static constexpr int kSmem = 1024 + kTileBytes * (2 + kRing) + 2 * kPBytes + 256;
  static_assert(kSmem <= 232448, "fwd2 shared memory");
  static_assert(HD <= 128, "fwd2 TMEM layout holds two 128-column accumulators");
};
constexpr int kFwd2Threads = 384;

template <int HD>
__global__ void __launch_bounds__(kFwd2Threads, 1)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  using C = Fwd2Cfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem);                    // 2 tiles
  const uint32_t sR = sQ + 2 * C::kTileBytes;            // ring of kRing tiles
  const uint32_t sP = sR + C::kRing * C::kTileBytes;     // 2 P tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kTileBytes * (2 + C::kRing) + 2 * C::kPBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* r_full = bars + 1;   // [3]
  uint64_t* r_empty = bars + 4;  // [3]
  uint64_t* s_full = bars + 7;   // [2] S_x of the current block in TMEM
  uint64_t* p_full = bars + 9;   // [2] P_x in smem (S_x read, O_x rescaled)
  uint64_t* o_done = bars + 11;  // [2] PV_x complete (P_x smem free, O_x stable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const uint32_t warp = warp_id(), lane = lane_id();
  // 1-D grid in groups of group_heads heads, heaviest pairs of every head of a group first: no tail of
  // heavy CTAs, and the CTAs in flight share a few heads' K / V blocks in L2
  const int npair = p.nqb / 2, per_group = p.group_heads * npair;
  const int grp = (int)blockIdx.x / per_group, within = (int)blockIdx.x - grp * per_group;
  const int gh = min(p.group_heads, p.heads - grp * p.group_heads);
  const int pair = npair - 1 - within / gh;
  const int head = grp * p.group_heads + within % gh;
  // tile a, tile b: adjacent query blocks (the heaviest pairs first keep a many-wave launch balanced),
  // or — when the launch is under two waves (e.g. 12 heads at TP=8) and the heaviest adjacent pair
  // alone would set the kernel's length — a heavy block with a light one, so every CTA carries about
  // the same number of key blocks
  const int q_lo = p.balanced ? pair : 2 * pair, q_hi = p.balanced ? p.nqb - 1 - pair : 2 * pair + 1;
  const int nkv = q_hi + 1;                           // kv blocks 0..q_hi (tile a uses 0..q_lo)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    mbar_init(smem_u32(q_full), 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(smem_u32(r_full + i), 1);
      mbar_init(smem_u32(r_empty + i), 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(smem_u32(s_full + x), 1);
      mbar_init(smem_u32(p_full + x), 4);
      mbar_init(smem_u32(o_done + x), 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(smem_u32(q_full), 2 * C::kTileBytes);
      for (int x = 0; x < 2; ++x)
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(sQ + x * C::kTileBytes + c * 16384, &tq, smem_u32(q_full), c * 64, (x ? q_hi : q_lo) * 128,
                      head);
      for (int t = 0; t < 2 * nkv; ++t) {  // K_0, V_0, K_1, V_1, ...
        const int slot = t % 3, ph = (t / 3) & 1;
        mbar_wait(smem_u32(r_empty + slot), ph ^ 1);
        mbar_arrive_expect_tx(smem_u32(r_full + slot), C::kTileBytes);
        const CUtensorMap* m = (t & 1) ? &tv : &tk;
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(sR + slot * C::kTileBytes + c * 16384, m, smem_u32(r_full + slot), c * 64, (t >> 1) * 128, head);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, 0, 0);  // Q (K-major) x K_j (K-major)
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, HD, 0, 1);   // P (K-major) x V_j (MN-major)
      auto slot_of = [](int t) { return t % 3; };
      auto wait_item = [&](int t) { mbar_wait(smem_u32(r_full + t % 3), (t / 3) & 1); };
      auto issue_s = [&](int x, int j) {
        const uint32_t kbase = sR + slot_of(2 * j) * C::kTileBytes;
        const uint32_t qbase = sQ + x * C::kTileBytes;
        const uint32_t d = tmem + x * 128;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16(d, umma_desc_sw128(qbase + off, 16, 1024), umma_desc_sw128(kbase + off, 16, 1024), idesc_s,
                    kk > 0 ? 1u : 0u);
        }
        tc_commit(smem_u32(s_full + x));
      };
      auto issue_pv = [&](int x, int j) {
        mbar_wait(smem_u32(p_full + x), j & 1);
        tc_fence_after();
        const uint32_t vbase = sR + slot_of(2 * j + 1) * C::kTileBytes;
        const uint32_t pbase = sP + x * C::kPBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 kv positions
          umma_bf16(tmem + 256 + x * 128, umma_desc_sw128(pbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    umma_desc_sw128(vbase + kk * 2048, 16384, 1024), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(smem_u32(o_done + x));
      };
      mbar_wait(smem_u32(q_full), 0);
      wait_item(0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      tc_commit(smem_u32(r_empty + slot_of(0)));
      for (int j = 0; j < nkv; ++j) {
        const bool a_here = j <= q_lo, a_next = j + 1 <= q_lo, b_next = j + 1 < nkv;
        wait_item(2 * j + 1);  // V_j
        if (a_here) issue_pv(0, j);
        if (b_next) {
          wait_item(2 * j + 2);  // K_{j+1}
          tc_fence_after();
        }
        // S_a(j+1): softmax a finished reading S_a(j) before it wrote P_a(j) (waited in issue_pv)
        if (a_next) issue_s(0, j + 1);
        issue_pv(1, j);
        tc_commit(smem_u32(r_empty + slot_of(2 * j + 1)));  // V_j consumed by both tiles
        if (b_next) {
          issue_s(1, j + 1);
          tc_commit(smem_u32(r_empty + slot_of(2 * j + 2)));  // K_{j+1} consumed
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax (two warpgroups)
    const int x = (int)(warp - 4) / 4;  // 0: tile a, 1: tile b
    const uint32_t quad = (warp - 4) & 3;
    const int r = quad * 32 + lane;
    const int qblk = x ? q_hi : q_lo;
    const int qrow = qblk * 128 + r;
    const int nblk = qblk + 1;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    const uint32_t s_col = x * 128, o_col = 256 + x * 128;
    const uint32_t pbuf = sP + x * C::kPBytes;
    float m2 = -INFINITY;  // running (lazily updated) max, log2 domain
    float l = 0.f;         // running sum of exp2(s - m2) over valid scores (dropped ones included)
    const uint64_t row_idx = ((uint64_t)(p.head_base + head) * p.seq + qrow) * (uint64_t)p.seq;
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(smem_u32(s_full + x), j & 1);
      tc_fence_after();
      const bool diag = (j == qblk);
      // pass 1: block max over the two 64-column halves (the causal mask only on the diagonal block:
      // the off-diagonal blocks take a branch-free path — the kernel is integer-ALU bound)
      auto block_max = [&](auto diag_tag) {
        constexpr bool kDiag = decltype(diag_tag)::value;
        float bm = -INFINITY;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t u[64];
          tmem_ld_32x32b_x32(lane_base + s_col + h * 64, *reinterpret_cast<uint32_t(*)[32]>(u));
          tmem_ld_32x32b_x32(lane_base + s_col + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
          tmem_ld_wait();
          float pm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int t = 0; t < 64; ++t) {
            const float v = (kDiag && h * 64 + t > r) ? -INFINITY : __uint_as_float(u[t]);
            pm[t & 3] = fmaxf(pm[t & 3], v);
          }
          bm = fmaxf(bm, fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])));
        }
        return bm;
      };
      float bmax = diag ? block_max(std::true_type{}) : block_max(std::false_type{});
      bmax *= p.alpha_log2;
      float corr = 1.f;
      bool rescale = false;
      if (bmax > m2 + 8.f || m2 == -INFINITY) {  // lazy rescale (2^8 headroom), as attn_fwd_kernel
        const float mnew = fmaxf(bmax, m2);
        corr = (m2 == -INFINITY) ? 0.f : ex2(m2 - mnew);
        rescale = (m2 != -INFINITY);
        m2 = mnew;
      }
      // P_x smem and O_x: PV_x(j-1) must be done
      if (j > 0) mbar_wait(smem_u32(o_done + x), (j - 1) & 1);
      tc_fence_after();
      if (__any_sync(0xffffffffu, rescale)) {
        for (int c = 0; c * 32 < HD; ++c) {
          uint32_t u[32];
          tmem_ld_32x32b_x32(lane_base + o_col + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) u[t] = __float_as_uint(__uint_as_float(u[t]) * corr);
          tmem_st_32x32b_x32(lane_base + o_col + c * 32, u);
        }
        tmem_st_wait();
      }
      // pass 2: exps, row sum, dropout, bf16 P_x straight into smem; the keep bits of the block go to
      // the optional mask buffer (the backward then reads them instead of re-hashing)
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
      uint64_t z = drop_weyl_attn(p.seed, (row_idx + (uint64_t)j * 128) >> 2);
      uint32_t kw[4] = {0u, 0u, 0u, 0u};
      auto block_exp = [&](auto diag_tag) {
        constexpr bool kDiag = decltype(diag_tag)::value;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t u[64];
          tmem_ld_32x32b_x32(lane_base + s_col + h * 64, *reinterpret_cast<uint32_t(*)[32]>(u));
          tmem_ld_32x32b_x32(lane_base + s_col + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
          tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < 8; ++g) {  // 8 chunks of 8 columns
            float e[8], pv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const int col = h * 64 + g * 8 + t;
              const float sv = (kDiag && col > r) ? -INFINITY : __uint_as_float(u[g * 8 + t]);
              e[t] = ex2(fmaf(sv, p.alpha_log2, -m2));  // exp2(-inf) = 0 for masked columns
              ps[t & 3] += e[t];
            }
            if (p.thresh16) {
              const uint32_t keep = drop_select8(z, p.thresh16, e, pv);
              kw[(h * 64 + g * 8) >> 5] |= keep << ((g * 8) & 31);
            } else {
#pragma unroll
              for (int t = 0; t < 8; ++t) pv[t] = e[t];
            }
            z += 2 * curator::kSplitMixGamma;
            st_shared_v4(sw128_addr(pbuf + h * 16384, r, g), pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]),
                         pack_bf16x2(pv[4], pv[5]), pack_bf16x2(pv[6], pv[7]));
          }
        }
      };
      if (diag)
        block_exp(std::true_type{});
      else
        block_exp(std::false_type{});
      if (p.mask != nullptr && p.thresh16)
        *reinterpret_cast<uint4*>(p.mask + ((size_t)head * p.seq + qrow) * (p.seq >> 5) + j * 4) =
            make_uint4(kw[0], kw[1], kw[2], kw[3]);
      l = l * corr + ((ps[0] + ps[1]) + (ps[2] + ps[3]));
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(p_full + x));  // also: S_x read (the next S_x may overwrite it)
    }
    // epilogue: O / l * dropout scale -> bf16 ctx ; lse
    mbar_wait(smem_u32(o_done + x), (nblk - 1) & 1);
    tc_fence_after();
    const float inv = p.drop_scale / l;
    __nv_bfloat16* orow = p.out + (long long)qrow * p.ld_out + (long long)head * p.out_head_stride;
    for (int c = 0; c * 32 < HD; ++c) {
      uint32_t u[32];
      tmem_ld_32x32b_x32(lane_base + o_col + c * 32, u);
      tmem_ld_wait();
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        *reinterpret_cast<uint4*>(orow + c * 32 + v * 8) =
            make_uint4(pack_bf16x2(__uint_as_float(u[8 * v]) * inv, __uint_as_float(u[8 * v + 1]) * inv),
                       pack_bf16x2(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv),
                       pack_bf16x2(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv),
                       pack_bf16x2(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv));
      }
    }
    p.lse[(long long)head * p.seq + qrow] = (m2 + __log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- backward
// D[h][i] = sum_d dO[i][h][d] * O[i][h][d]   (= sum_j P_drop dP_drop, the softmax-backward row term)
__global__ void attn_bwd_rowdot_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
                                       long long ld, int hd, int heads, int seq, float* __restrict__ D) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= heads * seq) return;
  const int h = warp / seq, i = warp - h * seq;
  const __nv_bfloat16* a = dout + (long long)i * ld + (long long)h * hd;
  const __nv_bfloat16* b = out + (long long)i * ld + (long long)h * hd;
  float acc = 0.f;
  for (int d = lane * 2; d < hd; d += 64) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + d));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(b + d));
    acc += x.x * y.x + x.y * y.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) D[(long long)h * seq + i] = acc;
}

// Same D with coalesced rows: consecutive threads take consecutive 16-byte chunks of a token row (all
// heads of row i are contiguous), TPR = hd / 8 lanes per (head, row) reduce with shuffles. hd 64 / 128.
template <int TPR>
__global__ void __launch_bounds__(256) attn_bwd_rowdot_vec_kernel(const uint4* __restrict__ dout,
                                                                  const uint4* __restrict__ out, long long ld_vec,
                                                                  int heads, int seq, float* __restrict__ D) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_row = heads * TPR;
  const long long i = t / per_row;
  const int c = (int)(t - i * per_row);
  float acc = 0.f;
  if (i < seq) {
    const uint4 x = __ldg(dout + i * ld_vec + c), y = __ldg(out + i * ld_vec + c);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 a = unpack_bf16x2(xs[q]), b = unpack_bf16x2(ys[q]);
      acc = fmaf(a.x, b.x, fmaf(a.y, b.y, acc));
    }
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (i < seq && (c & (TPR - 1)) == 0) D[(long long)(c / TPR) * seq + i] = acc;
}

// D for every (head, row): the coalesced kernel for hd 64 / 128, the warp-per-row kernel otherwise.
void launch_rowdot(const void* dout, const void* out, long long ld, int hd, int heads, int seq, float* D,
                   cudaStream_t s) {
  const long long threads = (long long)seq * heads * (hd / 8);
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  const bool vec_ok = (ld % 8 == 0) && ((reinterpret_cast<uintptr_t>(dout) | reinterpret_cast<uintptr_t>(out)) % 16 == 0);
  if (vec_ok && hd == 128)
    attn_bwd_rowdot_vec_kernel<16><<<blocks, 256, 0, s>>>(static_cast<const uint4*>(dout), static_cast<const uint4*>(out),
                                                          ld / 8, heads, seq, D);
  else if (vec_ok && hd == 64)
    attn_bwd_rowdot_vec_kernel<8><<<blocks, 256, 0, s>>>(static_cast<const uint4*>(dout), static_cast<const uint4*>(out),
                                                         ld / 8, heads, seq, D);
  else
    attn_bwd_rowdot_kernel<<<(heads * seq + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dout),
                                                                 static_cast<const __nv_bfloat16*>(out), ld, hd, heads,
                                                                 seq, D);
}

struct AttnBwdParams {
  int seq, nqb, heads;
  long long head_base;
  float alpha, alpha_log2;
  uint64_t seed;
  uint32_t thresh16;
  float drop_scale;
  const float* lse;  // [heads][seq]
  const float* D;    // [heads][seq]
  __nv_bfloat16* dq; // dqkv: row i, head h: + i * ld_dq + h * 3hd (+0 Q, +hd K, +2hd V)
  long long ld_dq;
  const uint32_t* mask;  // keep bits written by the forward ([heads][seq][seq/32]); nullptr: re-hash
  int group_heads;       // one-kernel backward: heads per launch-order group (see attn_bwd2_kernel)
};


template <int HD>
struct BwdCfg {
  static constexpr int kChunks = (HD + 63) / 64;
  static constexpr int kTileBytes = kChunks * 16384;
  static constexpr int kMBytes = 2 * 16384;  // one 128 x 128 bf16 tile (P or dS)
  static constexpr int kHDP = (HD + 31) / 32 * 32;
};

// Keep bits of 8 consecutive attention-score elements starting at idx (idx % 4 == 0).
__device__ __forceinline__ uint32_t keep8(uint64_t seed, uint64_t idx, uint32_t thresh16) {
  if (thresh16 == 0) return 0xffu;
  uint32_t m = 0;
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const uint64_t bits = curator::dropout_bits(seed, (idx + h2 * 4) >> 2);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (((bits >> (16 * q)) & 0xffffu) >= thresh16) m |= 1u << (4 * h2 + q);
  }
  return m;
}

// Keep bits of the 8 scores (qrow, col .. col + 7) of `head` (col % 8 == 0): from the forward's mask
// buffer when present (one load instead of two SplitMix64 evaluations), else the counter-based hash.
__device__ __forceinline__ uint32_t keep8_bwd(const AttnBwdParams& p, int head, int qrow, int col, uint64_t idx) {
  if (p.thresh16 == 0) return 0xffu;
  if (p.mask != nullptr)
    return (__ldg(p.mask + ((size_t)head * p.seq + qrow) * (p.seq >> 5) + (col >> 5)) >> (col & 31)) & 0xffu;
  return keep8(p.seed, idx, p.thresh16);
}

// Issue a 128 x N x K (K = 16 * ksteps) MMA chain with both operands given as smem descriptor generators.
template <class FA, class FB>
__device__ __forceinline__ void mma_chain(uint32_t d, uint32_t idesc, int ksteps, bool accumulate, FA fa, FB fb) {
  for (int kk = 0; kk < ksteps; ++kk) umma_bf16(d, fa(kk), fb(kk), idesc, (accumulate || kk > 0) ? 1u : 0u);
}

// K-major operand of `rows` x K in 64-wide SW128 chunks of 16 KB: k-step kk of 16 elements.
__device__ __forceinline__ uint64_t kmaj(uint32_t base, int kk) {
  return umma_desc_sw128(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
}
// MN-major operand (rows = k, 128 B of the MN dim per row, 64-wide chunks 16 KB apart): k-step kk.
__device__ __forceinline__ uint64_t mnmaj(uint32_t base, int kk) {
  return umma_desc_sw128(base + kk * 2048, 16384, 1024);
}

// dK, dV for one (head, 128-key block j): loop over query blocks i >= j. NH softmax warpgroups split
// each block row's 128 columns (the backward has no row reduction), NH = 2: 384 threads.
template <int HD, int NH>
__global__ void __launch_bounds__(128 + 128 * NH, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                         const AttnBwdParams p) {
  using C = BwdCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sK = smem_u32(smem), sV = sK + C::kTileBytes, sQ = sV + C::kTileBytes, sO = sQ + C::kTileBytes;
  // P_drop and dS share one 128 x 128 smem tile: dS is written after the dV MMA has consumed P
  const uint32_t sP = sO + C::kTileBytes, sS = sP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * C::kTileBytes + C::kMBytes);
  uint64_t* kv_full = bars + 0;
  uint64_t* qo_full = bars + 1;
  uint64_t* qo_empty = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* p_full = bars + 4;   // softmax wrote P_drop (and finished reading S)
  uint64_t* dp_full = bars + 5;
  uint64_t* ds_full = bars + 6;
  uint64_t* blk_done = bars + 7; // dV and dK MMAs of the block done (P / dS smem free)
  uint64_t* pv_done = bars + 8;  // dV MMA done (P consumed; the tile can take dS)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int jb = (int)blockIdx.y;  // key block; jb = 0 has the most query blocks (grid: heads, key blocks)
  const int head = blockIdx.x;
  const int i0 = jb, nblk = p.nqb - jb;
  constexpr uint32_t kDV = 0, kDK = C::kHDP, kSC = 2 * C::kHDP;
  // dP gets its own TMEM columns when they fit (head dim <= 128): the dP MMA then runs while the
  // softmax warps still work on S; for head dim 160 it reuses the S columns after S is consumed.
  constexpr bool kSepDP = 2 * C::kHDP + 256 <= 512;
  constexpr uint32_t kDPc = kSepDP ? kSC + 128 : kSC;

  if (warp == 0 && lane == 0) {
    for (auto* b : {&tq, &tk, &tv, &tdo}) tma_prefetch_desc(b);
    for (int i = 0; i < 9; ++i) mbar_init(smem_u32(bars + i), (i == 4 || i == 6) ? 4 * NH : 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(smem_u32(kv_full), 2 * C::kTileBytes);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_3d(sK + c * 16384, &tk, smem_u32(kv_full), c * 64, jb * 128, head);
        tma_load_3d(sV + c * 16384, &tv, smem_u32(kv_full), c * 64, jb * 128, head);
      }
      for (int b = 0; b < nblk; ++b) {
        const int ib = i0 + b;
        mbar_wait(smem_u32(qo_empty), (b & 1) ^ 1);
        mbar_arrive_expect_tx(smem_u32(qo_full), 2 * C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(sQ + c * 16384, &tq, smem_u32(qo_full), c * 64, ib * 128, head);
          tma_load_3d(sO + c * 16384, &tdo, smem_u32(qo_full), c * 64, ib * 128, head);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_acc = umma_idesc_bf16(128, HD, 1, 1);
      constexpr int kd = (HD + 15) / 16;  // k-steps over the head dim
      mbar_wait(smem_u32(kv_full), 0);
      for (int b = 0; b < nblk; ++b) {
        const int ph = b & 1;
        mbar_wait(smem_u32(qo_full), ph);
        if (b > 0) mbar_wait(smem_u32(blk_done), ph ^ 1);  // previous block's dV/dK done (P, dS free)
        tc_fence_after();
        // S = Q_i K_j^T
        mma_chain(tmem + kSC, id_s, kd, false, [&](int kk) { return kmaj(sQ, kk); }, [&](int kk) { return kmaj(sK, kk); });
        tc_commit(smem_u32(s_full));
        // dP = dO_i V_j^T
        if (!kSepDP) mbar_wait(smem_u32(p_full), ph);  // aliased with S: wait until S is consumed
        tc_fence_after();
        mma_chain(tmem + kDPc, id_s, kd, false, [&](int kk) { return kmaj(sO, kk); }, [&](int kk) { return kmaj(sV, kk); });
        tc_commit(smem_u32(dp_full));
        if (kSepDP) {
          mbar_wait(smem_u32(p_full), ph);
          tc_fence_after();
        }
        // dV += P_drop^T dO_i
        mma_chain(tmem + kDV, id_acc, 8, b > 0, [&](int kk) { return mnmaj(sP, kk); }, [&](int kk) { return mnmaj(sO, kk); });
        tc_commit(smem_u32(pv_done));
        // dK += dS^T Q_i
        mbar_wait(smem_u32(ds_full), ph);
        tc_fence_after();
        mma_chain(tmem + kDK, id_acc, 8, b > 0, [&](int kk) { return mnmaj(sS, kk); }, [&](int kk) { return mnmaj(sQ, kk); });
        tc_commit(smem_u32(qo_empty));
        tc_commit(smem_u32(blk_done));
      }
    }
  } else if (warp >= 4) {
    constexpr int CW = 128 / NH;  // score columns per thread
    const uint32_t quad = (warp - 4) & 3;
    const int hf = (int)(warp - 4) >> 2;
    const int col0 = hf * CW;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    for (int b = 0; b < nblk; ++b) {
      const int ib = i0 + b, ph = b & 1;
      const int qrow = ib * 128 + r;
      const float lse2 = p.lse[(long long)head * p.seq + qrow] * kLog2e;
      const float Di = p.D[(long long)head * p.seq + qrow];
      const uint64_t row_idx = ((uint64_t)(p.head_base + head) * p.seq + qrow) * (uint64_t)p.seq + (uint64_t)jb * 128;
      const bool diag = (ib == jb);
      // the block's 128 keep bits in one 16-byte load, issued before the S wait so its latency hides
      uint4 mw = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      if (p.mask != nullptr && p.thresh16)
        mw = __ldg(reinterpret_cast<const uint4*>(p.mask + ((size_t)head * p.seq + qrow) * (p.seq >> 5)) + jb);
      mbar_wait(smem_u32(s_full), ph);
      tc_fence_after();
      float pr[CW];
      auto probs = [&](auto diag_tag) {  // the causal mask only on the diagonal block (branch-free elsewhere)
        constexpr bool kDiag = decltype(diag_tag)::value;
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) {
          uint32_t u[32];
          tmem_ld_32x32b_x32(lane_base + kSC + col0 + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int col = col0 + c * 32 + t;
            pr[c * 32 + t] = (kDiag && col > r) ? 0.f : ex2(__uint_as_float(u[t]) * p.alpha_log2 - lse2);
          }
        }
      };
      if (diag)
        probs(std::true_type{});
      else
        probs(std::false_type{});
      if (b > 0) mbar_wait(smem_u32(blk_done), ph ^ 1);  // P / dS smem free
#pragma unroll
      for (int gl = 0; gl < CW / 8; ++gl) {
        const int g = col0 / 8 + gl;
        const uint32_t keep = keep8_bwd(p, head, qrow, jb * 128 + g * 8, row_idx + g * 8);
        float v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) v[t] = ((keep >> t) & 1u) ? pr[gl * 8 + t] : 0.f;
        st_shared_v4(sw128_addr(sP + (g >> 3) * 16384, r, g & 7), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                     pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(p_full));
      mbar_wait(smem_u32(dp_full), ph);
      mbar_wait(smem_u32(pv_done), ph);  // the P tile is free for dS
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + kDPc + col0 + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int cc = col0 + c * 32 + g * 8;
          const uint32_t keep = keep8_bwd(p, head, qrow, jb * 128 + cc, row_idx + cc);
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const float dp = ((keep >> t) & 1u) ? __uint_as_float(u[g * 8 + t]) * p.drop_scale : 0.f;
            v[t] = pr[c * 32 + g * 8 + t] * (dp - Di);
          }
          const int gg = cc / 8;
          st_shared_v4(sw128_addr(sS + (gg >> 3) * 16384, r, gg & 7), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                       pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
    }
    // epilogue: dV = scale * acc, dK = alpha * acc -> dqkv (V and K slots) of key rows jb*128 + r
    mbar_wait(smem_u32(blk_done), (nblk - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* base = p.dq + (long long)(jb * 128 + r) * p.ld_dq + (long long)head * 3 * HD;
    for (int which = (NH == 2 ? hf : 0); which < (NH == 2 ? hf + 1 : 2); ++which) {
      const float sc = which == 0 ? p.drop_scale : p.alpha;
      __nv_bfloat16* dst = base + (which == 0 ? 2 * HD : HD);
      const uint32_t col = which == 0 ? kDV : kDK;
      for (int c = 0; c * 32 < HD; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + col + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int v = 0; v < 4; ++v)
          *reinterpret_cast<uint4*>(dst + c * 32 + v * 8) =
              make_uint4(pack_bf16x2(__uint_as_float(u[8 * v]) * sc, __uint_as_float(u[8 * v + 1]) * sc),
                         pack_bf16x2(__uint_as_float(u[8 * v + 2]) * sc, __uint_as_float(u[8 * v + 3]) * sc),
                         pack_bf16x2(__uint_as_float(u[8 * v + 4]) * sc, __uint_as_float(u[8 * v + 5]) * sc),
                         pack_bf16x2(__uint_as_float(u[8 * v + 6]) * sc, __uint_as_float(u[8 * v + 7]) * sc));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- backward, one kernel (hd <= 128)
// attn_bwd2_kernel<HD>: one CTA per (head, 128-key block j), heaviest first, looping over the query
// blocks i >= j. Per block: S = Q_i K_j^T and dP = dO_i V_j^T in TMEM; the softmax warpgroup forms
// P (from S, lse and the forward's keep bits) and dS = P~ (dP' - D) into ONE shared smem tile (dS
// after the dV MMA consumed P); dV += P^T dO_i, dK += dS^T Q_i accumulate in TMEM, and dQ_i's partial
// dS K_j (in dP's TMEM columns once dP was read) is added into an fp32 dQ accumulator with vector
// red.global.add — so the dQ pass of attn_bwd_dq_kernel (which recomputed S, dP and the softmax
// backward) disappears. Q_i / dO_i are double-buffered; S(i+1) is issued as soon as S(i) was read.
// TMEM: dV [0,128), dK [128,256), S [256,384), dP / dQ partial [384,512).
template <int HD>
struct Bwd2Cfg {
  static constexpr int kChunks = (HD + 63) / 64;
  static constexpr int kTileBytes = kChunks * 16384;
  static constexpr int kTBytes = 2 * 16384;  // P / dS tile: 128 x 128 bf16
  static constexpr int kSmem = 1024 + kTileBytes * 6 + kTBytes + 256;
  static_assert(HD <= 128, "bwd2 TMEM layout");
  static_assert(kSmem <= 232448, "bwd2 shared memory");
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

template <int HD, int NH>
__global__ void __launch_bounds__(128 + 128 * NH, 1)
    attn_bwd2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                     const AttnBwdParams p, float* __restrict__ dq_acc) {
  using C = Bwd2Cfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sK = smem_u32(smem), sV = sK + C::kTileBytes;
  const uint32_t sQ0 = sV + C::kTileBytes;           // Q slots 0, 1
  const uint32_t sO0 = sQ0 + 2 * C::kTileBytes;      // dO slots 0, 1
  const uint32_t sT = sO0 + 2 * C::kTileBytes;       // P, then dS
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * C::kTileBytes + C::kTBytes);
  uint64_t* kv_full = bars + 0;
  uint64_t* qo_full = bars + 1;   // [2]
  uint64_t* qo_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* s_free = bars + 6;    // unused since the pipelined order (p_full(i) implies S(i) was read)
  uint64_t* dp_full = bars + 7;
  uint64_t* p_full = bars + 8;    // 4 warps wrote P
  uint64_t* pv_done = bars + 9;   // dV MMA consumed P (the tile can take dS)
  uint64_t* ds_full = bars + 10;  // 4 warps wrote dS
  uint64_t* mma_done = bars + 11; // dK and dQ-partial MMAs done (tile free, dQ partial in TMEM)
  uint64_t* dq_free = bars + 12;  // 4 warps drained the dQ partial (dP columns free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);
  const uint32_t warp = warp_id(), lane = lane_id();
  // Launch order (1-D grid): groups of group_heads heads; inside a group every head's heaviest key block
  // (jb = 0: most query blocks) first, the light ones last. Heavy-first avoids a tail of heavy CTAs;
  // the grouping keeps the CTAs in flight on a few heads, so the fp32 dQ accumulator rows they add
  // into (and the heads' Q / dO blocks) stay in L2 instead of spanning all heads at once.
  const int per_group = p.group_heads * p.nqb;
  const int grp = (int)blockIdx.x / per_group, within = (int)blockIdx.x - grp * per_group;
  const int gh = min(p.group_heads, p.heads - grp * p.group_heads);  // heads in this (last) group
  const int jb = within / gh;
  const int head = grp * p.group_heads + (within - jb * gh);
  const int nblk = p.nqb - jb;
  constexpr uint32_t kDV = 0, kDK = 128, kSC = 256, kDP = 384;

  if (warp == 0 && lane == 0) {
    for (auto* b : {&tq, &tk, &tv, &tdo}) tma_prefetch_desc(b);
    for (int i = 0; i < 13; ++i) {
      const bool four = (bars + i == s_free) || (bars + i == p_full) || (bars + i == ds_full) || (bars + i == dq_free);
      mbar_init(smem_u32(bars + i), four ? 4 * NH : 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(smem_u32(kv_full), 2 * C::kTileBytes);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_3d(sK + c * 16384, &tk, smem_u32(kv_full), c * 64, jb * 128, head);
        tma_load_3d(sV + c * 16384, &tv, smem_u32(kv_full), c * 64, jb * 128, head);
      }
      for (int b = 0; b < nblk; ++b) {
        const int slot = b & 1, ib = jb + b;
        mbar_wait(smem_u32(qo_empty + slot), ((b >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(smem_u32(qo_full + slot), 2 * C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(sQ0 + slot * C::kTileBytes + c * 16384, &tq, smem_u32(qo_full + slot), c * 64, ib * 128, head);
          tma_load_3d(sO0 + slot * C::kTileBytes + c * 16384, &tdo, smem_u32(qo_full + slot), c * 64, ib * 128, head);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_acc = umma_idesc_bf16(128, HD, 1, 1);
      constexpr uint32_t id_dq = umma_idesc_bf16(128, HD, 0, 1);
      constexpr int kd = HD / 16;
      auto sQ = [&](int b) { return sQ0 + (b & 1) * C::kTileBytes; };
      auto sO = [&](int b) { return sO0 + (b & 1) * C::kTileBytes; };
      auto issue_s = [&](int b) {
        mma_chain(tmem + kSC, id_s, kd, false, [&](int kk) { return kmaj(sQ(b), kk); },
                  [&](int kk) { return kmaj(sK, kk); });
        tc_commit(smem_u32(s_full));
      };
      auto issue_dp = [&](int b) {
        mma_chain(tmem + kDP, id_s, kd, false, [&](int kk) { return kmaj(sO(b), kk); },
                  [&](int kk) { return kmaj(sV, kk); });
        tc_commit(smem_u32(dp_full));
      };
      mbar_wait(smem_u32(kv_full), 0);
      mbar_wait(smem_u32(qo_full), 0);
      tc_fence_after();
      issue_s(0);
      for (int b = 0; b < nblk; ++b) {
        const int ph = b & 1;
        // dV += P^T dO_i
        mbar_wait(smem_u32(p_full), ph);
        tc_fence_after();
        mma_chain(tmem + kDV, id_acc, 8, b > 0, [&](int kk) { return mnmaj(sT, kk); },
                  [&](int kk) { return mnmaj(sO(b), kk); });
        tc_commit(smem_u32(pv_done));
        // S(i+1): the softmax warps read S(i) before they wrote P(i)
        if (b + 1 < nblk) {
          mbar_wait(smem_u32(qo_full + ((b + 1) & 1)), ((b + 1) >> 1) & 1);
          tc_fence_after();
          issue_s(b + 1);
        }
        // dP(i) once the previous block's dQ partial left the shared columns (drained while dV(i) ran)
        if (b > 0) {
          mbar_wait(smem_u32(dq_free), ph ^ 1);
          tc_fence_after();
        }
        issue_dp(b);
        // dK += dS^T Q_i ; dQ partial = dS K_j into dP's columns (dP read before dS was written)
        mbar_wait(smem_u32(ds_full), ph);
        tc_fence_after();
        mma_chain(tmem + kDK, id_acc, 8, b > 0, [&](int kk) { return mnmaj(sT, kk); },
                  [&](int kk) { return mnmaj(sQ(b), kk); });
        mma_chain(tmem + kDP, id_dq, 8, false, [&](int kk) { return kmaj(sT, kk); },
                  [&](int kk) { return mnmaj(sK, kk); });
        tc_commit(smem_u32(mma_done));
        tc_commit(smem_u32(qo_empty + (b & 1)));
      }
    }
  } else if (warp >= 4) {
    // NH column halves: warpgroup hf (warps 4 + 4 hf .. 7 + 4 hf) owns columns [hf * CW, (hf + 1) * CW)
    // of every block row (the softmax backward has no row reduction: D_i and lse_i are precomputed),
    // so with NH = 2 two warpgroups share each block's exp / mask / dS work and the dQ drain.
    constexpr int CW = 128 / NH;          // score columns per thread
    constexpr int QW = HD / NH;           // dQ / dV / dK columns per thread
    const uint32_t quad = (warp - 4) & 3;
    const int hf = (int)(warp - 4) >> 2;
    const int col0 = hf * CW, g0 = col0 / 8;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    // Software-pipelined per block i (the tensor core and the softmax warps overlap):
    //   write P(i) -> [dV(i) MMA | drain dQ(i-1)] -> dP(i) MMA -> dS(i) -> [dK(i), dQ(i) MMAs | P(i+1) exps]
    uint32_t pp[CW / 2];  // the row's probabilities, packed bf16 pairs (fp32 spilled at 255 registers)
    uint4 mw, mw_nx;      // the block's 128 keep bits from the forward (current, next block)
    float Di = 0.f, D_nx = 0.f, lse_nx = 0.f;
    // the per-row operands of block b (lse, D, keep bits): issued one block ahead so their L2 latency
    // is off the softmax warps' critical path
    auto prefetch = [&](int b) {
      const int qrow = (jb + b) * 128 + r;
      lse_nx = p.lse[(long long)head * p.seq + qrow];
      D_nx = p.D[(long long)head * p.seq + qrow];
      mw_nx = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      if (p.mask != nullptr && p.thresh16)
        mw_nx = __ldg(reinterpret_cast<const uint4*>(p.mask + ((size_t)head * p.seq + qrow) * (p.seq >> 5)) + jb);
    };
    // exps of block b into pp (S(b) in TMEM), its keep bits and row term (prefetch(b) issued before)
    auto load_block = [&](int b) {
      const int ib = jb + b;
      const int qrow = ib * 128 + r;
      const float lse2 = lse_nx * kLog2e;
      Di = D_nx;
      mw = mw_nx;
      if (p.mask == nullptr && p.thresh16 != 0) {
        const uint64_t row_idx = ((uint64_t)(p.head_base + head) * p.seq + qrow) * (uint64_t)p.seq + (uint64_t)jb * 128;
        uint32_t kw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t w = 0;
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if ((4 * q + g) >= g0 && (4 * q + g) < g0 + CW / 8)
              w |= keep8(p.seed, row_idx + (4 * q + g) * 8, p.thresh16) << (8 * g);
          kw[q] = w;
        }
        mw = make_uint4(kw[0], kw[1], kw[2], kw[3]);
      }
      mbar_wait(smem_u32(s_full), b & 1);
      tc_fence_after();
      auto probs = [&](auto diag_tag) {
        constexpr bool kDiag = decltype(diag_tag)::value;
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) {
          uint32_t u[32];
          tmem_ld_32x32b_x32(lane_base + kSC + col0 + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            const int col = col0 + c * 32 + t;
            const float a = (kDiag && col > r) ? 0.f : ex2(__uint_as_float(u[t]) * p.alpha_log2 - lse2);
            const float b2 = (kDiag && col + 1 > r) ? 0.f : ex2(__uint_as_float(u[t + 1]) * p.alpha_log2 - lse2);
            pp[(c * 32 + t) >> 1] = pack_bf16x2(a, b2);
          }
        }
      };
      if (ib == jb)
        probs(std::true_type{});
      else
        probs(std::false_type{});
      tc_fence_before();
    };
    // TMEM -> registers -> fp32 vector atomics: this half of dQ_i's partial (block b)
    auto drain = [&](int b) {
      const int qrow = (jb + b) * 128 + r;
      float* dst = dq_acc + ((size_t)head * p.seq + qrow) * HD + hf * QW;
#pragma unroll
      for (int c = 0; c < QW / 32; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + kDP + hf * QW + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          red_add_v4(dst + c * 32 + 4 * v, __uint_as_float(u[4 * v]), __uint_as_float(u[4 * v + 1]),
                     __uint_as_float(u[4 * v + 2]), __uint_as_float(u[4 * v + 3]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(dq_free));
    };
    prefetch(0);
    load_block(0);
    for (int b = 0; b < nblk; ++b) {
      const int ph = b & 1;
      const uint32_t kw[4] = {mw.x, mw.y, mw.z, mw.w};  // byte g = keep bits of the 8 columns of group g
      if (b + 1 < nblk) prefetch(b + 1);
      // P (dropped, unscaled) into the tile once the previous block's dK / dQ MMAs have read dS from it
      if (b > 0) mbar_wait(smem_u32(mma_done), ph ^ 1);
#pragma unroll
      for (int gl = 0; gl < CW / 8; ++gl) {
        const int g = g0 + gl;
        const uint32_t kb = kw[g >> 2] >> ((g & 3) * 8);
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w[q] = pp[gl * 4 + q] & (((kb >> (2 * q)) & 1u) * 0xffffu | ((kb >> (2 * q + 1)) & 1u) * 0xffff0000u);
        st_shared_v4(sw128_addr(sT + (g >> 3) * 16384, r, g & 7), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(p_full));
      // the previous block's dQ partial leaves TMEM while the dV MMA runs; dP(i) is issued after it
      if (b > 0) {
        tc_fence_after();
        drain(b - 1);
      }
      // dS = P~ (dP' - D) once dP is in TMEM and the dV MMA has consumed P from the tile
      mbar_wait(smem_u32(dp_full), ph);
      mbar_wait(smem_u32(pv_done), ph);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + kDP + col0 + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int gl = c * 4 + g, gg = g0 + gl;  // 8-column chunk index 0..15
          const uint32_t kb = kw[gg >> 2] >> ((gg & 3) * 8);
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 pr = unpack_bf16x2(pp[gl * 4 + q]);
            const float d0 = ((kb >> (2 * q)) & 1u) ? __uint_as_float(u[g * 8 + 2 * q]) * p.drop_scale : 0.f;
            const float d1 = ((kb >> (2 * q + 1)) & 1u) ? __uint_as_float(u[g * 8 + 2 * q + 1]) * p.drop_scale : 0.f;
            w[q] = pack_bf16x2(pr.x * (d0 - Di), pr.y * (d1 - Di));
          }
          st_shared_v4(sw128_addr(sT + (gg >> 3) * 16384, r, gg & 7), w[0], w[1], w[2], w[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
      // the next block's exps while dK(i) and dQ(i) run on the tensor core
      if (b + 1 < nblk) load_block(b + 1);
    }
    mbar_wait(smem_u32(mma_done), (nblk - 1) & 1);
    tc_fence_after();
    drain(nblk - 1);
    // epilogue: dV = scale * acc, dK = alpha * acc -> dqkv (V and K slots) of key rows jb*128 + r
    // (NH = 2: warpgroup 0 writes dV, warpgroup 1 dK)
    __nv_bfloat16* base = p.dq + (long long)(jb * 128 + r) * p.ld_dq + (long long)head * 3 * HD;
    for (int which = (NH == 2 ? hf : 0); which < (NH == 2 ? hf + 1 : 2); ++which) {
      const float sc = which == 0 ? p.drop_scale : p.alpha;
      __nv_bfloat16* dst = base + (which == 0 ? 2 * HD : HD);
      const uint32_t col = which == 0 ? kDV : kDK;
      for (int c = 0; c * 32 < HD; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + col + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int v = 0; v < 4; ++v)
          *reinterpret_cast<uint4*>(dst + c * 32 + v * 8) =
              make_uint4(pack_bf16x2(__uint_as_float(u[8 * v]) * sc, __uint_as_float(u[8 * v + 1]) * sc),
                         pack_bf16x2(__uint_as_float(u[8 * v + 2]) * sc, __uint_as_float(u[8 * v + 3]) * sc),
                         pack_bf16x2(__uint_as_float(u[8 * v + 4]) * sc, __uint_as_float(u[8 * v + 5]) * sc),
                         pack_bf16x2(__uint_as_float(u[8 * v + 6]) * sc, __uint_as_float(u[8 * v + 7]) * sc));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// dQ (bf16, into dqkv's Q slots) = alpha * the fp32 accumulator [heads][seq][HD]; 8 values per thread.
__global__ void dq_finalize_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq, long long ld_dq,
                                   int hd, int heads, int seq, float alpha) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // 8-value group
  const long long groups = (long long)heads * seq * (hd / 8);
  if (i >= groups) return;
  const int per_row = hd / 8;
  const long long row = i / per_row;  // head * seq + q
  const int g = (int)(i - row * per_row);
  const int h = (int)(row / seq), q = (int)(row - (long long)h * seq);
  const float4 a = *reinterpret_cast<const float4*>(acc + row * hd + g * 8);
  const float4 b = *reinterpret_cast<const float4*>(acc + row * hd + g * 8 + 4);
  *reinterpret_cast<uint4*>(dq + (long long)q * ld_dq + (long long)h * 3 * hd + g * 8) =
      make_uint4(pack_bf16x2(a.x * alpha, a.y * alpha), pack_bf16x2(a.z * alpha, a.w * alpha),
                 pack_bf16x2(b.x * alpha, b.y * alpha), pack_bf16x2(b.z * alpha, b.w * alpha));
}

// dQ for one (head, 128-query block i): loop over key blocks j <= i.
template <int HD, int NH>
__global__ void __launch_bounds__(128 + 128 * NH, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                       const AttnBwdParams p) {
  using C = BwdCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem), sO = sQ + C::kTileBytes, sK = sO + C::kTileBytes, sV = sK + C::kTileBytes;
  const uint32_t sS = sV + C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * C::kTileBytes + C::kMBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 2;
  uint64_t* sd_full = bars + 3;  // S and dP in TMEM
  uint64_t* ds_full = bars + 4;
  uint64_t* blk_done = bars + 5;  // dQ MMA of the block done (dS smem and TMEM S/dP free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int ib = p.nqb - 1 - (int)blockIdx.y;  // heaviest query blocks of every head first
  const int head = blockIdx.x;
  const int nblk = ib + 1;
  constexpr uint32_t kDQ = 0, kSC = 256, kDP = 384;

  if (warp == 0 && lane == 0) {
    for (auto* b : {&tq, &tk, &tv, &tdo}) tma_prefetch_desc(b);
    for (int i = 0; i < 6; ++i) mbar_init(smem_u32(bars + i), i == 4 ? 4 * NH : 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(smem_u32(q_full), 2 * C::kTileBytes);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_3d(sQ + c * 16384, &tq, smem_u32(q_full), c * 64, ib * 128, head);
        tma_load_3d(sO + c * 16384, &tdo, smem_u32(q_full), c * 64, ib * 128, head);
      }
      for (int j = 0; j < nblk; ++j) {
        mbar_wait(smem_u32(kv_empty), (j & 1) ^ 1);
        mbar_arrive_expect_tx(smem_u32(kv_full), 2 * C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(sK + c * 16384, &tk, smem_u32(kv_full), c * 64, j * 128, head);
          tma_load_3d(sV + c * 16384, &tv, smem_u32(kv_full), c * 64, j * 128, head);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_dq = umma_idesc_bf16(128, HD, 0, 1);
      constexpr int kd = (HD + 15) / 16;
      mbar_wait(smem_u32(q_full), 0);
      for (int j = 0; j < nblk; ++j) {
        const int ph = j & 1;
        mbar_wait(smem_u32(kv_full), ph);
        if (j > 0) mbar_wait(smem_u32(blk_done), ph ^ 1);
        tc_fence_after();
        mma_chain(tmem + kSC, id_s, kd, false, [&](int kk) { return kmaj(sQ, kk); }, [&](int kk) { return kmaj(sK, kk); });
        mma_chain(tmem + kDP, id_s, kd, false, [&](int kk) { return kmaj(sO, kk); }, [&](int kk) { return kmaj(sV, kk); });
        tc_commit(smem_u32(sd_full));
        mbar_wait(smem_u32(ds_full), ph);
        tc_fence_after();
        // dQ += dS K_j   (dS K-major over kv; K_j MN-major: n = head dim, k = kv)
        mma_chain(tmem + kDQ, id_dq, 8, j > 0, [&](int kk) { return kmaj(sS, kk); }, [&](int kk) { return mnmaj(sK, kk); });
        tc_commit(smem_u32(kv_empty));
        tc_commit(smem_u32(blk_done));
      }
    }
  } else if (warp >= 4) {
    constexpr int CW = 128 / NH;  // score columns per thread (NH warpgroups split each block row)
    const uint32_t quad = (warp - 4) & 3;
    const int hf = (int)(warp - 4) >> 2;
    const int col0 = hf * CW;
    const int r = quad * 32 + lane;
    const int qrow = ib * 128 + r;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    const float lse2 = p.lse[(long long)head * p.seq + qrow] * kLog2e;
    const float Di = p.D[(long long)head * p.seq + qrow];
    for (int j = 0; j < nblk; ++j) {
      const int ph = j & 1;
      const bool diag = (j == ib);
      const uint64_t row_idx = ((uint64_t)(p.head_base + head) * p.seq + qrow) * (uint64_t)p.seq + (uint64_t)j * 128;
      mbar_wait(smem_u32(sd_full), ph);
      tc_fence_after();
      if (j > 0) mbar_wait(smem_u32(blk_done), ph ^ 1);  // dS smem free (previous dQ MMA done)
      auto dscores = [&](auto diag_tag) {  // the causal mask only on the diagonal block
        constexpr bool kDiag = decltype(diag_tag)::value;
#pragma unroll
        for (int c = col0 / 32; c < (col0 + CW) / 32; ++c) {
          uint32_t us[32], ud[32];
          tmem_ld_32x32b_x32(lane_base + kSC + c * 32, us);
          tmem_ld_32x32b_x32(lane_base + kDP + c * 32, ud);
          tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t keep = keep8_bwd(p, head, qrow, j * 128 + c * 32 + g * 8, row_idx + c * 32 + g * 8);
            float v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const int col = c * 32 + g * 8 + t;
              const float pr =
                  (kDiag && col > r) ? 0.f : ex2(__uint_as_float(us[g * 8 + t]) * p.alpha_log2 - lse2);
              const float dp = ((keep >> t) & 1u) ? __uint_as_float(ud[g * 8 + t]) * p.drop_scale : 0.f;
              v[t] = pr * (dp - Di);
            }
            const int gg = c * 4 + g;
            st_shared_v4(sw128_addr(sS + (gg >> 3) * 16384, r, gg & 7), pack_bf16x2(v[0], v[1]),
                         pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
          }
        }
      };
      if (diag)
        dscores(std::true_type{});
      else
        dscores(std::false_type{});
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
    }
    mbar_wait(smem_u32(blk_done), (nblk - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* dst = p.dq + (long long)qrow * p.ld_dq + (long long)head * 3 * HD;
    for (int c = hf; c * 32 < HD; c += NH) {
      uint32_t u[32];
      tmem_ld_32x32b_x32(lane_base + kDQ + c * 32, u);
      tmem_ld_wait();
      const float sc = p.alpha;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        *reinterpret_cast<uint4*>(dst + c * 32 + v * 8) =
            make_uint4(pack_bf16x2(__uint_as_float(u[8 * v]) * sc, __uint_as_float(u[8 * v + 1]) * sc),
                       pack_bf16x2(__uint_as_float(u[8 * v + 2]) * sc, __uint_as_float(u[8 * v + 3]) * sc),
                       pack_bf16x2(__uint_as_float(u[8 * v + 4]) * sc, __uint_as_float(u[8 * v + 5]) * sc),
                       pack_bf16x2(__uint_as_float(u[8 * v + 6]) * sc, __uint_as_float(u[8 * v + 7]) * sc));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode() {
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

// Dynamic shared-memory opt-in, once per (kernel, device) (one context per GPU per host thread).
template <auto kKern>
bool set_smem_once(int bytes) {
  static std::atomic<uint64_t> done{0};  // one instance per kernel (template argument = the kernel)
  auto kern = kKern;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const uint64_t bit = uint64_t{1} << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  done.fetch_or(bit, std::memory_order_release);
  return true;
}

// Per-head [seq x hd] bf16 operand: dims (hd, seq, heads), row stride ld, head stride hs; box (64, 128).
bool head_map(CUtensorMap* m, const void* base, int hd, int seq, int heads, long long ld, long long hs) {
  EncodeFn enc = encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)hd, (cuuint64_t)seq, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)hs * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
int launch_fwd(const void* qkv, long long ld_qkv, int heads, int seq, long long head_base, float alpha,
               uint64_t seed, uint32_t thresh16, float drop_scale, void* out, long long ld_out, float* lse,
               uint32_t* mask, cudaStream_t s) {
  (void)mask;  // the single-tile kernel re-hashes in the backward
  using C = AttnCfg<HD>;
  CUtensorMap mq, mk, mv;
  const auto* q = static_cast<const uint16_t*>(qkv);
  if (!head_map(&mq, q, HD, seq, heads, ld_qkv, 3 * HD) || !head_map(&mk, q + HD, HD, seq, heads, ld_qkv, 3 * HD) ||
      !head_map(&mv, q + 2 * HD, HD, seq, heads, ld_qkv, 3 * HD))
    return 1;
  AttnParams p{};
  p.seq = seq;
  p.nqb = seq / 128;
  p.heads = heads;
  p.head_base = head_base;
  p.alpha_log2 = alpha * kLog2e;
  p.seed = seed;
  p.thresh16 = thresh16;
  p.drop_scale = drop_scale;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.ld_out = ld_out;
  p.out_head_stride = HD;
  p.lse = lse;
  if (!set_smem_once<attn_fwd_kernel<HD>>(C::kSmem)) return 2;
  attn_fwd_kernel<HD><<<dim3(heads, p.nqb), kAttnThreads, C::kSmem, s>>>(mq, mk, mv, p);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int attn_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      n <= 0)
    n = 148;
  return n;
}

template <int HD>
int launch_fwd2(const void* qkv, long long ld_qkv, int heads, int seq, long long head_base, float alpha,
                uint64_t seed, uint32_t thresh16, float drop_scale, void* out, long long ld_out, float* lse,
                uint32_t* mask, cudaStream_t s) {
  using C = Fwd2Cfg<HD>;
  CUtensorMap mq, mk, mv;
  const auto* q = static_cast<const uint16_t*>(qkv);
  if (!head_map(&mq, q, HD, seq, heads, ld_qkv, 3 * HD) || !head_map(&mk, q + HD, HD, seq, heads, ld_qkv, 3 * HD) ||
      !head_map(&mv, q + 2 * HD, HD, seq, heads, ld_qkv, 3 * HD))
    return 1;
  AttnParams p{};
  p.seq = seq;
  p.nqb = seq / 128;
  p.heads = heads;
  p.head_base = head_base;
  p.alpha_log2 = alpha * kLog2e;
  p.seed = seed;
  p.thresh16 = thresh16;
  p.drop_scale = drop_scale;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.ld_out = ld_out;
  p.out_head_stride = HD;
  p.lse = lse;
  p.mask = mask;
  if (!set_smem_once<attn_fwd2_kernel<HD>>(C::kSmem)) return 2;
  {
    // measured: grouping halves the forward's DRAM reads but its 8 pairs per head leave group tails
    // (GPT-3 layer 273 us ungrouped vs 286-303 us in groups of 4-12), so one group by default
    const char* e = getenv("MT_ATTN_FWD_GROUP_HEADS");
    const int g = e ? atoi(e) : 0;
    p.group_heads = (g <= 0 || g > heads) ? heads : g;
    // MT_ATTN_FWD_BALANCED=0/1 forces the pairing; default: balanced pairs when the CTAs fit one wave
    // (GPT-3 TP=8, 12 heads: 87.7 -> 74.2 us; from 24 heads on adjacent pairs win: 92 vs 130 us,
    // profiles/r02_attn_balanced_ab.log)
    const char* b = getenv("MT_ATTN_FWD_BALANCED");
    p.balanced = b && b[0] ? (b[0] == '1') : (heads * (p.nqb / 2) <= attn_sm_count());
  }
  attn_fwd2_kernel<HD><<<heads * (p.nqb / 2), kFwd2Threads, C::kSmem, s>>>(mq, mk, mv, p);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// Softmax warpgroups of the fused backward kernels (MT_ATTN_BWD_WG, default 2: column halves; read per
// call so tests can switch it).
int bwd2_halves() {
  const char* e = getenv("MT_ATTN_BWD_WG");
  return (e && e[0] == '1') ? 1 : 2;
}

template <int HD>
int launch_bwd(const void* qkv, long long ld_qkv, const void* ctx, const void* dctx, long long ld_ctx, int heads,
               int seq, long long head_base, float alpha, uint64_t seed, uint32_t thresh16, float drop_scale,
               const float* lse, float* D, void* dqkv, const uint32_t* mask, float* dq_acc, cudaStream_t s) {
  using C = BwdCfg<HD>;
  const auto* q = static_cast<const uint16_t*>(qkv);
  CUtensorMap mq, mk, mv, mdo;
  if (!head_map(&mq, q, HD, seq, heads, ld_qkv, 3 * HD) || !head_map(&mk, q + HD, HD, seq, heads, ld_qkv, 3 * HD) ||
      !head_map(&mv, q + 2 * HD, HD, seq, heads, ld_qkv, 3 * HD) ||
      !head_map(&mdo, dctx, HD, seq, heads, ld_ctx, HD))
    return 1;
  launch_rowdot(dctx, ctx, ld_ctx, HD, heads, seq, D, s);
  AttnBwdParams p{};
  p.seq = seq;
  p.nqb = seq / 128;
  p.heads = heads;
  p.head_base = head_base;
  p.alpha = alpha;
  p.alpha_log2 = alpha * kLog2e;
  p.seed = seed;
  p.thresh16 = thresh16;
  p.drop_scale = drop_scale;
  p.lse = lse;
  p.D = D;
  p.dq = static_cast<__nv_bfloat16*>(dqkv);
  p.ld_dq = ld_qkv;
  p.mask = mask;
  {
    // groups of 8 heads for launches of >= 5 waves: DRAM 1.80 -> 0.50 GB, 582 -> 550 us (GPT-3 layer,
    // 96 heads; 48 heads 288 -> 284 us); shorter launches get group tails (24 heads: 157 -> 181 us),
    // so they keep one group (profiles/r02_attn_group_ab.log, r02_attn_group_tp8_ab.log)
    const char* e = getenv("MT_ATTN_GROUP_HEADS");  // 0: one group (all heads)
    const int g = e ? atoi(e) : (heads * p.nqb >= 5 * attn_sm_count() ? 8 : 0);
    p.group_heads = (g <= 0 || g > heads) ? heads : g;
  }
  constexpr int kSmemKV = 1024 + 4 * C::kTileBytes + C::kMBytes + 256;
  constexpr int kSmemQ = 1024 + 4 * C::kTileBytes + C::kMBytes + 256;
  if constexpr (HD <= 128) {
    if (dq_acc != nullptr) {  // one kernel: dK, dV and dQ (fp32 vector atomics), then the bf16 dQ
      using C2 = Bwd2Cfg<HD>;
      if (cudaMemsetAsync(dq_acc, 0, (size_t)heads * seq * HD * sizeof(float), s) != cudaSuccess) return 2;
      if (bwd2_halves() == 2) {
        if (!set_smem_once<attn_bwd2_kernel<HD, 2>>(C2::kSmem)) return 2;
        attn_bwd2_kernel<HD, 2><<<heads * p.nqb, 384, C2::kSmem, s>>>(mq, mk, mv, mdo, p, dq_acc);
      } else {
        if (!set_smem_once<attn_bwd2_kernel<HD, 1>>(C2::kSmem)) return 2;
        attn_bwd2_kernel<HD, 1><<<heads * p.nqb, 256, C2::kSmem, s>>>(mq, mk, mv, mdo, p, dq_acc);
      }
      const long long groups = (long long)heads * seq * (HD / 8);
      dq_finalize_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, s>>>(dq_acc, p.dq, p.ld_dq, HD, heads, seq, alpha);
      return cudaGetLastError() == cudaSuccess ? 0 : 2;
    }
  }
  if (bwd2_halves() == 2) {
    if (!set_smem_once<attn_bwd_dkdv_kernel<HD, 2>>(kSmemKV) || !set_smem_once<attn_bwd_dq_kernel<HD, 2>>(kSmemQ))
      return 2;
    attn_bwd_dkdv_kernel<HD, 2><<<dim3(heads, p.nqb), 384, kSmemKV, s>>>(mq, mk, mv, mdo, p);
    attn_bwd_dq_kernel<HD, 2><<<dim3(heads, p.nqb), 384, kSmemQ, s>>>(mq, mk, mv, mdo, p);
  } else {
    if (!set_smem_once<attn_bwd_dkdv_kernel<HD, 1>>(kSmemKV) || !set_smem_once<attn_bwd_dq_kernel<HD, 1>>(kSmemQ))
      return 2;
    attn_bwd_dkdv_kernel<HD, 1><<<dim3(heads, p.nqb), 256, kSmemKV, s>>>(mq, mk, mv, mdo, p);
    attn_bwd_dq_kernel<HD, 1><<<dim3(heads, p.nqb), 256, kSmemQ, s>>>(mq, mk, mv, mdo, p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace

// Fused causal attention backward for `heads` heads of one microbatch row: from qkv, the forward's
// ctx (O), its gradient dctx (dO) and the saved lse, writes dQ, dK, dV into dqkv (same layout as
// qkv). D is a [heads][seq] fp32 scratch. mask: the forward's dropout keep bits, or nullptr (the
// kernels re-derive them from the counter-based stream). dq_acc: [heads][seq][hd] fp32 scratch enabling
// the one-kernel backward for hd <= 128 (nullptr or MT_ATTN_BWD2=0: the dK/dV + dQ kernel pair).
// Returns 0 ok, 1 unsupported shape, 2 CUDA error.
int attention_bwd(const void* qkv, long long ld_qkv, const void* ctx, const void* dctx, long long ld_ctx, int heads,
                  int seq, int hd, long long head_base, float alpha, uint64_t seed, uint32_t thresh16,
                  float drop_scale, const float* lse, float* D, void* dqkv, const uint32_t* mask, float* dq_acc,
                  cudaStream_t s) {
  if (seq % 128 != 0 || seq <= 0) return 1;
  // MT_ATTN_BWD2=0 selects the deterministic kernel pair (the one-kernel backward adds dQ partials with
  // fp32 atomics, whose order varies between runs); read per call so tests can switch it
  const char* bwd2_env = getenv("MT_ATTN_BWD2");
  const bool one_kernel = !(bwd2_env && bwd2_env[0] == '0');
  if (!one_kernel) dq_acc = nullptr;
  switch (hd) {
    case 64:
      return launch_bwd<64>(qkv, ld_qkv, ctx, dctx, ld_ctx, heads, seq, head_base, alpha, seed, thresh16, drop_scale,
                            lse, D, dqkv, mask, dq_acc, s);
    case 128:
      return launch_bwd<128>(qkv, ld_qkv, ctx, dctx, ld_ctx, heads, seq, head_base, alpha, seed, thresh16, drop_scale,
                             lse, D, dqkv, mask, dq_acc, s);
    case 160:
      return launch_bwd<160>(qkv, ld_qkv, ctx, dctx, ld_ctx, heads, seq, head_base, alpha, seed, thresh16, drop_scale,
                             lse, D, dqkv, mask, nullptr, s);
    default:
      return 1;
  }
}

// Fused causal attention forward for `heads` heads of one microbatch row:
// qkv [seq][heads][3][hd] (row stride ld_qkv), out ctx [seq][heads][hd] (row stride ld_out),
// lse [heads][seq]. mask (optional, [heads][seq][seq/32] uint32): receives the dropout keep bits of
// the causal blocks (two-tile kernel only; returns *mask_written = 1 then). Returns 0 ok, 1
// unsupported shape, 2 CUDA error.
int attention_fwd(const void* qkv, long long ld_qkv, int heads, int seq, int hd, long long head_base, float alpha,
                  uint64_t seed, uint32_t thresh16, float drop_scale, void* out, long long ld_out, float* lse,
                  uint32_t* mask, int* mask_written, cudaStream_t s) {
  if (seq % 128 != 0 || seq <= 0) return 1;
  static const bool two_tiles = [] {
    const char* e = getenv("MT_ATTN_FWD2");
    return !(e && e[0] == '0');
  }();
  const bool fwd2 = two_tiles && (seq / 128) % 2 == 0;
  if (mask_written) *mask_written = (fwd2 && mask != nullptr && (hd == 64 || hd == 128)) ? 1 : 0;
  switch (hd) {
    case 64:
      return fwd2 ? launch_fwd2<64>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out,
                                    lse, mask, s)
                  : launch_fwd<64>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out,
                                   lse, mask, s);
    case 128:
      return fwd2 ? launch_fwd2<128>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out,
                                     lse, mask, s)
                  : launch_fwd<128>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out,
                                    lse, mask, s);
    case 160:
      return launch_fwd<160>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out, lse,
                             mask, s);
    default:
      return 1;
  }
}

// D[h][i] = dout_i . out_i per head (the softmax-backward row term; attention_sm100.cu's rowdot kernel)
void attn_rowdot(const void* dout, const void* out, long long ld, int hd, int heads, int seq, float* D, cudaStream_t s) {
  launch_rowdot(dout, out, ld, hd, heads, seq, D, s);
}

}  // namespace mt
