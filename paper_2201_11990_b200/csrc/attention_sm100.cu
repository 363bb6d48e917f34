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

#include <cstdint>
#include <cstdio>
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
  const int qb = p.nqb - 1 - (int)blockIdx.x;  // heaviest (most kv blocks) first
  const int head = blockIdx.y;
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

// dK, dV for one (head, 128-key block j): loop over query blocks i >= j.
template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1)
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
  const int jb = p.nqb - 1 - (int)blockIdx.x;  // key block (heaviest = first column of queries: jb = 0)
  const int head = blockIdx.y;
  const int i0 = jb, nblk = p.nqb - jb;
  constexpr uint32_t kDV = 0, kDK = C::kHDP, kSC = 2 * C::kHDP;
  // dP gets its own TMEM columns when they fit (head dim <= 128): the dP MMA then runs while the
  // softmax warps still work on S; for head dim 160 it reuses the S columns after S is consumed.
  constexpr bool kSepDP = 2 * C::kHDP + 256 <= 512;
  constexpr uint32_t kDPc = kSepDP ? kSC + 128 : kSC;

  if (warp == 0 && lane == 0) {
    for (auto* b : {&tq, &tk, &tv, &tdo}) tma_prefetch_desc(b);
    for (int i = 0; i < 9; ++i) mbar_init(smem_u32(bars + i), (i == 4 || i == 6) ? 4 : 1);
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
    const uint32_t quad = warp - 4;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    for (int b = 0; b < nblk; ++b) {
      const int ib = i0 + b, ph = b & 1;
      const int qrow = ib * 128 + r;
      const float lse2 = p.lse[(long long)head * p.seq + qrow] * kLog2e;
      const float Di = p.D[(long long)head * p.seq + qrow];
      const uint64_t row_idx = ((uint64_t)(p.head_base + head) * p.seq + qrow) * (uint64_t)p.seq + (uint64_t)jb * 128;
      const bool diag = (ib == jb);
      mbar_wait(smem_u32(s_full), ph);
      tc_fence_after();
      float pr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + kSC + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int col = c * 32 + t;
          pr[col] = (diag && col > r) ? 0.f : ex2(__uint_as_float(u[t]) * p.alpha_log2 - lse2);
        }
      }
      if (b > 0) mbar_wait(smem_u32(blk_done), ph ^ 1);  // P / dS smem free
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        const uint32_t keep = keep8(p.seed, row_idx + g * 8, p.thresh16);
        float v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) v[t] = ((keep >> t) & 1u) ? pr[g * 8 + t] : 0.f;
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
      for (int c = 0; c < 4; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(lane_base + kDPc + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t keep = keep8(p.seed, row_idx + c * 32 + g * 8, p.thresh16);
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int col = c * 32 + g * 8 + t;
            const float dp = ((keep >> t) & 1u) ? __uint_as_float(u[g * 8 + t]) * p.drop_scale : 0.f;
            v[t] = pr[col] * (dp - Di);
          }
          const int gg = c * 4 + g;
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
    for (int which = 0; which < 2; ++which) {
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

// dQ for one (head, 128-query block i): loop over key blocks j <= i.
template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1)
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
  const int ib = p.nqb - 1 - (int)blockIdx.x;
  const int head = blockIdx.y;
  const int nblk = ib + 1;
  constexpr uint32_t kDQ = 0, kSC = 256, kDP = 384;

  if (warp == 0 && lane == 0) {
    for (auto* b : {&tq, &tk, &tv, &tdo}) tma_prefetch_desc(b);
    for (int i = 0; i < 6; ++i) mbar_init(smem_u32(bars + i), i == 4 ? 4 : 1);
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
    const uint32_t quad = warp - 4;
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
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t us[32], ud[32];
        tmem_ld_32x32b_x32(lane_base + kSC + c * 32, us);
        tmem_ld_32x32b_x32(lane_base + kDP + c * 32, ud);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t keep = keep8(p.seed, row_idx + c * 32 + g * 8, p.thresh16);
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int col = c * 32 + g * 8 + t;
            const float pr = (diag && col > r) ? 0.f : ex2(__uint_as_float(us[g * 8 + t]) * p.alpha_log2 - lse2);
            const float dp = ((keep >> t) & 1u) ? __uint_as_float(ud[g * 8 + t]) * p.drop_scale : 0.f;
            v[t] = pr * (dp - Di);
          }
          const int gg = c * 4 + g;
          st_shared_v4(sw128_addr(sS + (gg >> 3) * 16384, r, gg & 7), pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                       pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
    }
    mbar_wait(smem_u32(blk_done), (nblk - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* dst = p.dq + (long long)qrow * p.ld_dq + (long long)head * 3 * HD;
    for (int c = 0; c * 32 < HD; ++c) {
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
               cudaStream_t s) {
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
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return 2;
    attr = true;
  }
  attn_fwd_kernel<HD><<<dim3(p.nqb, heads), kAttnThreads, C::kSmem, s>>>(mq, mk, mv, p);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

template <int HD>
int launch_bwd(const void* qkv, long long ld_qkv, const void* ctx, const void* dctx, long long ld_ctx, int heads,
               int seq, long long head_base, float alpha, uint64_t seed, uint32_t thresh16, float drop_scale,
               const float* lse, float* D, void* dqkv, cudaStream_t s) {
  using C = BwdCfg<HD>;
  const auto* q = static_cast<const uint16_t*>(qkv);
  CUtensorMap mq, mk, mv, mdo;
  if (!head_map(&mq, q, HD, seq, heads, ld_qkv, 3 * HD) || !head_map(&mk, q + HD, HD, seq, heads, ld_qkv, 3 * HD) ||
      !head_map(&mv, q + 2 * HD, HD, seq, heads, ld_qkv, 3 * HD) ||
      !head_map(&mdo, dctx, HD, seq, heads, ld_ctx, HD))
    return 1;
  const int rows = heads * seq;
  attn_bwd_rowdot_kernel<<<(rows + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dctx),
                                                         static_cast<const __nv_bfloat16*>(ctx), ld_ctx, HD, heads, seq,
                                                         D);
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
  constexpr int kSmemKV = 1024 + 4 * C::kTileBytes + C::kMBytes + 256;
  constexpr int kSmemQ = 1024 + 4 * C::kTileBytes + C::kMBytes + 256;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_bwd_dkdv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemKV) !=
            cudaSuccess ||
        cudaFuncSetAttribute(attn_bwd_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemQ) !=
            cudaSuccess)
      return 2;
    attr = true;
  }
  attn_bwd_dkdv_kernel<HD><<<dim3(p.nqb, heads), kAttnThreads, kSmemKV, s>>>(mq, mk, mv, mdo, p);
  attn_bwd_dq_kernel<HD><<<dim3(p.nqb, heads), kAttnThreads, kSmemQ, s>>>(mq, mk, mv, mdo, p);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace

// Fused causal attention backward for `heads` heads of one microbatch row: from qkv, the forward's
// ctx (O), its gradient dctx (dO) and the saved lse, writes dQ, dK, dV into dqkv (same layout as
// qkv). D is a [heads][seq] fp32 scratch. Returns 0 ok, 1 unsupported shape, 2 CUDA error.
int attention_bwd(const void* qkv, long long ld_qkv, const void* ctx, const void* dctx, long long ld_ctx, int heads,
                  int seq, int hd, long long head_base, float alpha, uint64_t seed, uint32_t thresh16,
                  float drop_scale, const float* lse, float* D, void* dqkv, cudaStream_t s) {
  if (seq % 128 != 0 || seq <= 0) return 1;
  switch (hd) {
    case 64:
      return launch_bwd<64>(qkv, ld_qkv, ctx, dctx, ld_ctx, heads, seq, head_base, alpha, seed, thresh16, drop_scale,
                            lse, D, dqkv, s);
    case 128:
      return launch_bwd<128>(qkv, ld_qkv, ctx, dctx, ld_ctx, heads, seq, head_base, alpha, seed, thresh16, drop_scale,
                             lse, D, dqkv, s);
    case 160:
      return launch_bwd<160>(qkv, ld_qkv, ctx, dctx, ld_ctx, heads, seq, head_base, alpha, seed, thresh16, drop_scale,
                             lse, D, dqkv, s);
    default:
      return 1;
  }
}

// Fused causal attention forward for `heads` heads of one microbatch row:
// qkv [seq][heads][3][hd] (row stride ld_qkv), out ctx [seq][heads][hd] (row stride ld_out),
// lse [heads][seq]. Returns 0 ok, 1 unsupported shape, 2 CUDA error.
int attention_fwd(const void* qkv, long long ld_qkv, int heads, int seq, int hd, long long head_base, float alpha,
                  uint64_t seed, uint32_t thresh16, float drop_scale, void* out, long long ld_out, float* lse,
                  cudaStream_t s) {
  if (seq % 128 != 0 || seq <= 0) return 1;
  switch (hd) {
    case 64:
      return launch_fwd<64>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out, lse, s);
    case 128:
      return launch_fwd<128>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out, lse,
                             s);
    case 160:
      return launch_fwd<160>(qkv, ld_qkv, heads, seq, head_base, alpha, seed, thresh16, drop_scale, out, ld_out, lse,
                             s);
    default:
      return 1;
  }
}

// D[h][i] = dout_i . out_i per head (the softmax-backward row term; attention_sm100.cu's rowdot kernel)
void attn_rowdot(const void* dout, const void* out, long long ld, int hd, int heads, int seq, float* D, cudaStream_t s) {
  const int rows = heads * seq;
  attn_bwd_rowdot_kernel<<<(rows + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dout),
                                                         static_cast<const __nv_bfloat16*>(out), ld, hd, heads, seq, D);
}

}  // namespace mt
