// HBM-bound kernels of the tensor-sliced transformer layer (sm_100a).
//
// All kernels move bf16 in 16-byte vectors (8 elements per thread per access), reduce with warp
// shuffles, and keep row data in registers between the passes of a row reduction, so every
// element is read from HBM once and written once. Column reductions (bias / LayerNorm parameter
// gradients) are two-stage and deterministic: per-split partials in a workspace, then a fixed-order
// sum into the fp32 gradient accumulator.
//
// Layer math restated from PAPER.md:133-150 (Megatron tensor slicing) — the reference has no
// implementation of it; the CPU restatement the tests compare against is oracle/layer_oracle.cpp.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "curator/dropout.hpp"
#include "kernels.cuh"

namespace mt {
namespace {

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[j]);
    const float2 p = __bfloat1622float2(h);
    f[2 * j] = p.x;
    f[2 * j + 1] = p.y;
  }
}
// bf16x8 unpack the compiler may not CSE across passes (re-unpacking costs 8 ALU ops; keeping the
// floats costs 8 registers per vector).
__device__ __forceinline__ void unpack8_v(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t lo, hi;
    asm volatile("shl.b32 %0, %2, 16; and.b32 %1, %2, 0xffff0000;" : "=r"(lo), "=r"(hi) : "r"(w[j]));
    f[2 * j] = __uint_as_float(lo);
    f[2 * j + 1] = __uint_as_float(hi);
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum over the block; `red` is >= 32 floats of shared memory, reused across calls.
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : 0.f;
  return warp_sum(t);
}

// Dropout stream in Weyl form: curator::dropout_bits(site, g) = splitmix64(site + g * gamma) =
// sm64_final(weyl(site, g)) with weyl = site + (g + 1) * gamma, so consecutive groups of 4 elements
// are one 64-bit add apart (the softmax kernels walk their row's groups without a 64-bit multiply
// per group).
__device__ __forceinline__ uint64_t drop_weyl(uint64_t site, uint64_t group) {
  return site + (group + 1) * curator::kSplitMixGamma;
}
__device__ __forceinline__ uint64_t sm64_final(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// o[j] = keep_j ? x[j] * mul : 0 for the 8 elements of groups (z, z + gamma): keep_j is the 16-bit
// field j & 3 of the group's 64 bits >= thresh16, compared and selected directly.
__device__ __forceinline__ void drop_scale8(uint64_t z, uint32_t thresh16, const float (&x)[8], float mul,
                                            float (&o)[8]) {
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const uint64_t b = sm64_final(z + (uint64_t)g * curator::kSplitMixGamma);
    const uint32_t lo = (uint32_t)b, hi = (uint32_t)(b >> 32);
    const uint32_t u[4] = {lo & 0xffffu, lo >> 16, hi & 0xffffu, hi >> 16};
#pragma unroll
    for (int q = 0; q < 4; ++q) o[4 * g + q] = u[q] >= thresh16 ? x[4 * g + q] * mul : 0.f;
  }
}

// Drop mask for 8 consecutive elements starting at idx (idx % 4 == 0): two SplitMix64 groups
// (include/curator/dropout.hpp).
__device__ __forceinline__ uint32_t keep_mask8(uint64_t seed, uint64_t idx, uint32_t thresh16) {
  if (thresh16 == 0) return 0xffu;
  uint32_t m = 0;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const uint64_t bits = curator::dropout_bits(seed, (idx >> 2) + g);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (((bits >> (16 * q)) & 0xffffu) >= thresh16) m |= 1u << (4 * g + q);
  }
  return m;
}

// ------------------------------------------------------------------ LayerNorm
// One CTA per row; the row stays in registers as packed bf16 (4 regs per 8 elements) and is
// re-unpacked in each pass (unpack8_v), keeping ~half the registers of an fp32 copy.
template <int VPT>
__global__ void __launch_bounds__(1024) ln_fwd_kernel(const uint4* __restrict__ x, const uint4* __restrict__ gamma,
                                                     const uint4* __restrict__ beta, uint4* __restrict__ y,
                                                     float* __restrict__ mean, float* __restrict__ rstd, int nvec,
                                                     float inv_h, float eps) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const uint4* xr = x + row * nvec;
  uint4 raw[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = i * blockDim.x + threadIdx.x;
    raw[i] = idx < nvec ? xr[idx] : make_uint4(0, 0, 0, 0);  // zero bf16 = 0.0: neutral for the sum
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    float v[8];
    unpack8_v(raw[i], v);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  const float mu = block_sum(s, red) * inv_h;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = i * blockDim.x + threadIdx.x;
    if (idx < nvec) {
      float v[8];
      unpack8_v(raw[i], v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = v[j] - mu;
        sq += d * d;
      }
    }
  }
  const float rs = rsqrtf(block_sum(sq, red) * inv_h + eps);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = i * blockDim.x + threadIdx.x;
    if (idx < nvec) {
      float v[8], g[8], b[8], o[8];
      unpack8_v(raw[i], v);
      unpack8(gamma[idx], g);
      unpack8(beta[idx], b);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[j] - mu) * rs * g[j] + b[j];
      y[row * nvec + idx] = pack8(o);
    }
  }
  if (threadIdx.x == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

template <int VPT>
__global__ void __launch_bounds__(1024) ln_bwd_dx_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ x,
                                                        const uint4* __restrict__ gamma, const float* __restrict__ mean,
                                                        const float* __restrict__ rstd, const uint4* __restrict__ resid,
                                                        uint4* __restrict__ dx, int nvec, float inv_h) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const float mu = mean[row], rs = rstd[row];
  uint4 rdy[VPT], rx[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = i * blockDim.x + threadIdx.x;
    const bool in = idx < nvec;
    rdy[i] = in ? dy[row * nvec + idx] : make_uint4(0, 0, 0, 0);
    rx[i] = in ? x[row * nvec + idx] : make_uint4(0, 0, 0, 0);
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = i * blockDim.x + threadIdx.x;
    if (idx < nvec) {
      float d[8], xv[8], gm[8];
      unpack8_v(rdy[i], d);
      unpack8_v(rx[i], xv);
      unpack8(gamma[idx], gm);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = d[j] * gm[j];
        s1 += g;
        s2 += g * ((xv[j] - mu) * rs);
      }
    }
  }
  const float m1 = block_sum(s1, red) * inv_h;
  const float m2 = block_sum(s2, red) * inv_h;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = i * blockDim.x + threadIdx.x;
    if (idx < nvec) {
      float d[8], xv[8], gm[8], o[8];
      unpack8_v(rdy[i], d);
      unpack8_v(rx[i], xv);
      unpack8(gamma[idx], gm);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = rs * (d[j] * gm[j] - m1 - (xv[j] - mu) * rs * m2);
      if (resid != nullptr) {
        float r[8];
        unpack8(resid[row * nvec + idx], r);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += r[j];
      }
      dx[row * nvec + idx] = pack8(o);
    }
  }
}

// ------------------------------------------------------------------ column reductions
// Stage 1: block (32 x 8): threadIdx.x -> 8-column vector, threadIdx.y -> row lane.
// Each (blockIdx.y) split covers rows [split*rows_per, ...). Partials -> ws[out][split][col].
constexpr int kColTY = 8;
constexpr int kColU = 4;

enum ColOp { kColSum = 0, kColLnParams = 1, kColDropout = 2 };

template <int OP>
__global__ void __launch_bounds__(256) colsum_stage1(const uint4* __restrict__ a, long long lda_vec,
                                                     const uint4* __restrict__ xin, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, uint4* __restrict__ out_dz,
                                                     float* __restrict__ ws, int rows, int nvec, int rows_per,
                                                     uint64_t seed, uint32_t thresh16, float scale,
                                                     uint64_t elem_offset = 0, const uint8_t* __restrict__ keep_in = nullptr) {
  constexpr int NO = OP == kColLnParams ? 2 : 1;
  __shared__ float part[NO][kColTY][32][9];
  const int cv = blockIdx.x * 32 + threadIdx.x;
  const int split = blockIdx.y;
  const int r0 = split * rows_per, r1 = min(rows, r0 + rows_per);
  float acc[NO][8];
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[o][j] = 0.f;
  if (cv < nvec) {
    // kColU rows per thread in flight (loads first, then the same in-order accumulation)
    for (int rb = r0 + threadIdx.y; rb < r1; rb += kColU * kColTY) {
      uint4 va[kColU], vx[kColU];
#pragma unroll
      for (int u = 0; u < kColU; ++u) {
        const int r = rb + u * kColTY;
        if (r < r1) {
          va[u] = a[(long long)r * lda_vec + cv];
          if (OP == kColLnParams) vx[u] = xin[(long long)r * nvec + cv];
        }
      }
#pragma unroll
      for (int u = 0; u < kColU; ++u) {
        const int r = rb + u * kColTY;
        if (r >= r1) break;
        float v[8];
        unpack8(va[u], v);
        if (OP == kColSum) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[0][j] += v[j];
        } else if (OP == kColLnParams) {
          float xv[8];
          unpack8(vx[u], xv);
          const float mu = mean[r], rs = rstd[r];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc[0][j] += v[j] * ((xv[j] - mu) * rs);
            acc[1][j] += v[j];
          }
        } else {
          const uint64_t idx = elem_offset + ((uint64_t)r * nvec + cv) * 8;
          const uint32_t keep = keep_in != nullptr ? (uint32_t)keep_in[(long long)r * nvec + cv]
                                                   : keep_mask8(seed, idx, thresh16);
          float o[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = ((keep >> j) & 1u) ? v[j] * scale : 0.f;
          const uint4 packed = pack8(o);
          out_dz[(long long)r * nvec + cv] = packed;
          float ob[8];
          unpack8(packed, ob);  // bias grad of the stored (bf16) dz
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[0][j] += ob[j];
        }
      }
    }
  }
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int j = 0; j < 8; ++j) part[o][threadIdx.y][threadIdx.x][j] = acc[o][j];
  __syncthreads();
  // 256 threads reduce 32 vectors x 8 lanes = 256 outputs per op (fixed order over threadIdx.y)
  const int t = threadIdx.y * 32 + threadIdx.x;
  const int vec = t >> 3, lane = t & 7;
  const int col = (blockIdx.x * 32 + vec) * 8 + lane;
  if (blockIdx.x * 32 + vec < nvec) {
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      float s = 0.f;
#pragma unroll
      for (int y = 0; y < kColTY; ++y) s += part[o][y][vec][lane];
      ws[((size_t)o * gridDim.y + split) * (size_t)nvec * 8 + col] = s;
    }
  }
}

// Stage 2: block (32 columns x 8 split lanes); lane y sums splits y, y+8, ... of its column, then a
// fixed-order shared-memory reduction over the 8 lanes (deterministic; many blocks even when the
// number of splits is large, e.g. the per-CTA partials of the fused LayerNorm backward).
__global__ void __launch_bounds__(256) colsum_stage2(const float* __restrict__ ws, float* __restrict__ out0,
                                                     float* __restrict__ out1, int n, int splits, int accumulate) {
  __shared__ float red[2][8][33];
  const int col = blockIdx.x * 32 + threadIdx.x;
  const int y = threadIdx.y;
  float s0 = 0.f, s1 = 0.f;
  if (col < n) {
#pragma unroll 4
    for (int sp = y; sp < splits; sp += 8) {
      s0 += ws[(size_t)sp * n + col];
      if (out1 != nullptr) s1 += ws[((size_t)splits + sp) * n + col];
    }
  }
  red[0][y][threadIdx.x] = s0;
  red[1][y][threadIdx.x] = s1;
  __syncthreads();
  if (y == 0 && col < n) {
    float t0 = 0.f, t1 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      t0 += red[0][k][threadIdx.x];
      t1 += red[1][k][threadIdx.x];
    }
    out0[col] = accumulate ? out0[col] + t0 : t0;
    if (out1 != nullptr) out1[col] = accumulate ? out1[col] + t1 : t1;
  }
}

int col_splits(int rows) {
  static int per = 0;
  if (per == 0) {
    const char* e = getenv("MT_COL_ROWS_PER_SPLIT");
    per = e ? std::max(8, atoi(e)) : 64;
  }
  int s = rows / per;
  return s < 1 ? 1 : (s > 64 ? 64 : s);
}

// ------------------------------------------------------------------ bias + dropout + residual
// 2-D grid: blockIdx.y = row, x covers the row's 8-element vectors (no 64-bit div/mod per element).
__global__ void __launch_bounds__(256) bias_dropout_residual_kernel(const uint4* __restrict__ z,
                                                                    const uint4* __restrict__ bias,
                                                                    const uint4* __restrict__ resid,
                                                                    uint4* __restrict__ out, int nvec_row,
                                                                    uint64_t seed, uint32_t thresh16, float scale,
                                                                    uint64_t elem_offset, uint8_t* __restrict__ keep_out) {
  const int cv = blockIdx.x * blockDim.x + threadIdx.x;
  if (cv >= nvec_row) return;
  const size_t v = (size_t)blockIdx.y * nvec_row + cv;
  float a[8], b[8], r[8], o[8];
  unpack8(z[v], a);
  unpack8(bias[cv], b);
  unpack8(resid[v], r);
  const uint32_t keep = keep_mask8(seed, elem_offset + (uint64_t)v * 8, thresh16);
  if (keep_out != nullptr) keep_out[v] = (uint8_t)keep;
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = r[j] + (((keep >> j) & 1u) ? (a[j] + b[j]) * scale : 0.f);
  out[v] = pack8(o);
}

// ------------------------------------------------------------------ causal softmax
// One warp per score row; the row's bf16 vectors stay packed in registers (4 regs per 8 scores)
// and are unpacked on the fly in each pass, which keeps the backward at ~half the registers of an
// fp32 copy and lets 3-4 CTAs share an SM. exp is exp2 of log2e-prescaled values (one FFMA + MUFU).
constexpr float kLog2e = 1.4426950408889634f;

// exp2 that the compiler may not CSE across passes (volatile): recomputing it in the second pass is
// cheaper than keeping a row's worth of fp32 probabilities live in registers.
__device__ __forceinline__ float ex2_recompute(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One warp per score row (VPL 8-score vectors per lane). The row's causal tail (columns > i) and the
// lanes past it are set to -inf, so the passes need no per-element causal checks:
//   max   on packed bf16x2 (one HMNMX2 per two scores; exact, the scores are bf16),
//   exp2  once per score in fp32 (kept in registers for rows up to 2048 columns), summed,
//   P     = keep ? e * (scale / sum) : 0, packed to bf16.
// ~13 instructions per score vs ~21 for three unpacking passes with a recomputed exp (the kernel was
// issue-bound at 0.39 of HBM roofline, ncu profiles/r02_hbm_ncu.md).
template <int VPL>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const uint4* __restrict__ S, uint4* __restrict__ P,
                                                          float* __restrict__ lse, int rows_total, int seq,
                                                          long long head_base, uint64_t seed, uint32_t thresh16,
                                                          float scale) {
  constexpr bool kKeep = VPL <= 8;  // fp32 exps stay in registers (64 per lane at most)
  constexpr uint32_t kNegInf2 = 0xff80ff80u;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows_total) return;
  const int bh = warp / seq, i = warp - bh * seq;
  const int nvec_row = seq >> 3;
  const uint4* srow = S + (size_t)warp * nvec_row;
  uint4* prow = P + (size_t)warp * nvec_row;
  const int nvalid = i + 1, nvec = (nvalid + 7) >> 3, nfull = nvalid >> 3, rem = nvalid & 7;
  uint4 raw[VPL];
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    const int v = lane + 32 * t;
    raw[t] = v < nvec ? srow[v] : make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
    if (v == nfull && rem != 0) {  // causal tail: scores j >= rem of the row's last vector -> -inf
      uint32_t w[4] = {raw[t].x, raw[t].y, raw[t].z, raw[t].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (2 * q >= rem) w[q] = kNegInf2;
        else if (2 * q + 1 >= rem) w[q] = (w[q] & 0xffffu) | 0xff800000u;
      }
      raw[t] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  __nv_bfloat162 m2v = __halves2bfloat162(__ushort_as_bfloat16(0xff80), __ushort_as_bfloat16(0xff80));
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    const uint32_t w[4] = {raw[t].x, raw[t].y, raw[t].z, raw[t].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) m2v = __hmax2(m2v, *reinterpret_cast<const __nv_bfloat162*>(&w[q]));
  }
  const float mx = warp_max(fmaxf(__low2float(m2v), __high2float(m2v)));
  const float mx2 = mx * kLog2e;
  float e[kKeep ? VPL : 1][8];
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < VPL; ++t) {
    if (lane + 32 * t < nvec) {
      float x[8];
      unpack8_v(raw[t], x);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float ej = ex2_recompute(fmaf(x[j], kLog2e, -mx2));  // exp2(-inf) = 0 on the causal tail
        sum += ej;
        if constexpr (kKeep) e[t][j] = ej;
      }
    }
  }
  sum = warp_sum(sum);
  const float inv = scale / sum;
  const uint64_t base_idx = ((uint64_t)(head_base + bh) * seq + i) * (uint64_t)seq;
  // this lane's first group; its later vectors are 32 * 2 groups further each
  uint64_t z = drop_weyl(seed, (base_idx >> 2) + 2 * (uint64_t)lane);
  const uint64_t z_step = 64 * curator::kSplitMixGamma;
#pragma unroll
  for (int t = 0; t < VPL; ++t, z += z_step) {
    const int v = lane + 32 * t;
    if (v < nvec) {
      float x[8], o[8];
      if constexpr (kKeep) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = e[t][j];
      } else {
        unpack8_v(raw[t], x);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = ex2_recompute(fmaf(x[j], kLog2e, -mx2));
      }
      if (thresh16 != 0) {
        drop_scale8(z, thresh16, x, inv, o);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = x[j] * inv;
      }
      prow[v] = pack8(o);
    }
  }
  const int zend = min(seq, (i / 256 + 1) * 256) >> 3;
  for (int v = nvec + lane; v < zend; v += 32) prow[v] = make_uint4(0, 0, 0, 0);
  if (lane == 0) lse[warp] = mx + logf(sum);
}

__global__ void __launch_bounds__(256) softmax_bwd_rowdot_kernel(const uint4* __restrict__ S,
                                                                  const float* __restrict__ lse,
                                                                  const float* __restrict__ D, uint4* __restrict__ dP,
                                                                  int rows_total, int seq, long long head_base,
                                                                  uint64_t seed, uint32_t thresh16, float scale,
                                                                  float alpha) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows_total) return;
  const int bh = warp / seq, i = warp - bh * seq;
  const int nvec_row = seq >> 3;
  const uint4* srow = S + (size_t)warp * nvec_row;
  uint4* drow = dP + (size_t)warp * nvec_row;
  const int nvalid = i + 1, nvec = (nvalid + 7) >> 3, nfull = nvalid >> 3, rem = nvalid & 7;
  const float l2 = lse[warp] * kLog2e;
  const float dot = D[warp];
  const uint64_t base_idx = ((uint64_t)(head_base + bh) * seq + i) * (uint64_t)seq;
  uint64_t z = drop_weyl(seed, (base_idx >> 2) + 2 * (uint64_t)lane);  // Weyl state of this lane's groups
  for (int v = lane; v < nvec; v += 32, z += 64 * curator::kSplitMixGamma) {
    const uint32_t valid = v < nfull ? 0xffu : (1u << rem) - 1u;
    float sv[8], g[8], gk[8], o[8];
    unpack8(srow[v], sv);
    unpack8(drow[v], g);
    if (thresh16 != 0) {
      drop_scale8(z, thresh16, g, scale, gk);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) gk[j] = g[j] * scale;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float y = ex2_recompute(fmaf(sv[j], kLog2e, -l2));
      o[j] = ((valid >> j) & 1u) ? alpha * y * (gk[j] - dot) : 0.f;
    }
    drow[v] = pack8(o);
  }
  const int zend = min(seq, (i / 256 + 1) * 256) >> 3;
  for (int v = nvec + lane; v < zend; v += 32) drow[v] = make_uint4(0, 0, 0, 0);
}

// ------------------------------------------------------------------ loss, init
__global__ void mse_loss_kernel(const uint4* __restrict__ y, const uint4* __restrict__ t, uint4* __restrict__ dy,
                                float* __restrict__ loss, long long nvec, float inv_n) {
  __shared__ float red[32];
  float acc = 0.f;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nvec; v += (long long)gridDim.x * blockDim.x) {
    float a[8], b[8], o[8];
    unpack8(y[v], a);
    unpack8(t[v], b);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = a[j] - b[j];
      acc += 0.5f * d * d;
      o[j] = d * inv_n;
    }
    dy[v] = pack8(o);
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(loss, acc * inv_n);
}

__global__ void fill_normal_kernel(__nv_bfloat16* __restrict__ out, long long rows, long long cols,
                                   long long global_cols, long long row0, long long col0, uint64_t key, float mean,
                                   float std) {
  const long long n = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols, c = e - r * cols;
    const uint64_t gidx = (uint64_t)(row0 + r) * (uint64_t)global_cols + (uint64_t)(col0 + c);
    const float z = (float)curator::normal_at(key, gidx);
    out[e] = __float2bfloat16_rn(mean + std * z);
  }
}

__global__ void fill_zero_kernel(float* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0.f;
}

int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  const long long cap = 148LL * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}


}  // namespace

// ------------------------------------------------------------------ launchers
#define MT_VPT_DISPATCH(VPT_NEEDED, LAUNCH) \
  do {                                      \
    if ((VPT_NEEDED) <= 1) {                \
      LAUNCH(1);                            \
    } else if ((VPT_NEEDED) <= 2) {         \
      LAUNCH(2);                            \
    } else if ((VPT_NEEDED) <= 4) {         \
      LAUNCH(4);                            \
    } else if ((VPT_NEEDED) <= 8) {         \
      LAUNCH(8);                            \
    } else if ((VPT_NEEDED) <= 12) {        \
      LAUNCH(12);                           \
    } else {                                \
      LAUNCH(16);                           \
    }                                       \
  } while (0)

// Threads per row: enough that each holds <= 2 vectors (16 elements) up to h = 16384 (<= 1024
// threads), so the row fits in a few registers per thread.
static void row_launch_shape(int h, int& threads, int& vpt) {
  const int nvec = h / 8;
  threads = (((nvec + 1) / 2 + 31) / 32) * 32;
  if (threads > 1024) threads = 1024;
  vpt = (nvec + threads - 1) / threads;
}

// TMA-fed persistent row kernels (rows_sm100.cu); MT_ROW_KERNELS=0 selects the per-row kernels.
static bool row_kernels_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MT_ROW_KERNELS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

void ln_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows, int h,
            float eps, cudaStream_t s) {
  if (row_kernels_enabled() && ln_fwd_rows(x, gamma, beta, y, mean, rstd, rows, h, eps, s)) return;
  int threads, vpt;
  row_launch_shape(h, threads, vpt);
#define L(V)                                                                                                   \
  ln_fwd_kernel<V><<<rows, threads, 0, s>>>((const uint4*)x, (const uint4*)gamma, (const uint4*)beta, (uint4*)y, \
                                            mean, rstd, h / 8, 1.f / h, eps)
  MT_VPT_DISPATCH(vpt, L);
#undef L
}

void ln_bwd_dx(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
               const void* resid, void* dx, int rows, int h, cudaStream_t s) {
  int threads, vpt;
  row_launch_shape(h, threads, vpt);
#define L(V)                                                                                                     \
  ln_bwd_dx_kernel<V><<<rows, threads, 0, s>>>((const uint4*)dy, (const uint4*)x, (const uint4*)gamma, mean, rstd, \
                                               (const uint4*)resid, (uint4*)dx, h / 8, 1.f / h)
  MT_VPT_DISPATCH(vpt, L);
#undef L
}

size_t colsum_workspace_floats(int rows, int n) {
  return std::max((size_t)2 * col_splits(rows) * n, (size_t)2 * row_kernel_ctas(rows) * n);
}

void colsum_partials(const float* ws, float* out0, float* out1, int n, int splits, bool accumulate, cudaStream_t s) {
  colsum_stage2<<<(n + 31) / 32, dim3(32, 8), 0, s>>>(ws, out0, out1, n, splits, accumulate);
}

int ln_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd, const void* resid,
            void* dx, float* dgamma, float* dbeta, int rows, int h, float* ws, bool accumulate, cudaStream_t s) {
  if (row_kernels_enabled() &&
      ln_bwd_rows(dy, x, gamma, mean, rstd, resid, dx, dgamma, dbeta, rows, h, ws, accumulate, s))
    return 2;
  // parameter grads first: dx may overwrite x in place (the vocab head does that)
  ln_bwd_params(dy, x, mean, rstd, dgamma, dbeta, rows, h, ws, accumulate, s);
  ln_bwd_dx(dy, x, gamma, mean, rstd, resid, dx, rows, h, s);
  return 3;
}

int bias_dropout_residual_ln(const void* z, const void* bias, const void* resid, void* out, const void* gamma,
                              const void* beta, void* y, float* mean, float* rstd, int rows, int h, float eps,
                              uint64_t seed, uint32_t thresh16, float scale, uint64_t elem_offset, cudaStream_t s,
                              uint8_t* keep_out) {
  if (thresh16 == 0) keep_out = nullptr;
  if (row_kernels_enabled() && bdr_ln_rows(z, bias, resid, out, gamma, beta, y, mean, rstd, rows, h, eps, seed,
                                           thresh16, scale, elem_offset, s, keep_out))
    return 1;
  bias_dropout_residual(z, bias, resid, out, rows, h, seed, thresh16, scale, s, elem_offset, keep_out);
  if (gamma != nullptr) ln_fwd(out, gamma, beta, y, mean, rstd, rows, h, eps, s);
  return gamma != nullptr ? 2 : 1;
}

void ln_bwd_params(const void* dy, const void* x, const float* mean, const float* rstd, float* dgamma, float* dbeta,
                   int rows, int h, float* ws, bool accumulate, cudaStream_t s) {
  const int nvec = h / 8, splits = col_splits(rows);
  dim3 grid((nvec + 31) / 32, splits), block(32, kColTY);
  colsum_stage1<kColLnParams><<<grid, block, 0, s>>>((const uint4*)dy, nvec, (const uint4*)x, mean, rstd, nullptr, ws,
                                                     rows, nvec, (rows + splits - 1) / splits, 0, 0, 1.f);
  colsum_stage2<<<(h + 31) / 32, dim3(32, 8), 0, s>>>(ws, dgamma, dbeta, h, splits, accumulate);
}

void bias_grad(const void* x, float* dbias, int rows, int n, long long ldx, float* ws, bool accumulate,
               cudaStream_t s) {
  const int nvec = n / 8, splits = col_splits(rows);
  dim3 grid((nvec + 31) / 32, splits), block(32, kColTY);
  colsum_stage1<kColSum><<<grid, block, 0, s>>>((const uint4*)x, ldx / 8, nullptr, nullptr, nullptr, nullptr, ws, rows,
                                                nvec, (rows + splits - 1) / splits, 0, 0, 1.f);
  colsum_stage2<<<(n + 31) / 32, dim3(32, 8), 0, s>>>(ws, dbias, nullptr, n, splits, accumulate);
}

void dropout_bwd_bias_grad(const void* dy, void* dz, float* dbias, int rows, int h, uint64_t seed, uint32_t thresh16,
                           float scale, float* ws, bool accumulate, cudaStream_t s, uint64_t elem_offset,
                           const uint8_t* keep_in) {
  if (thresh16 == 0) keep_in = nullptr;
  const int nvec = h / 8, splits = col_splits(rows);
  dim3 grid((nvec + 31) / 32, splits), block(32, kColTY);
  colsum_stage1<kColDropout><<<grid, block, 0, s>>>((const uint4*)dy, nvec, nullptr, nullptr, nullptr, (uint4*)dz, ws,
                                                    rows, nvec, (rows + splits - 1) / splits, seed, thresh16, scale,
                                                    elem_offset, keep_in);
  colsum_stage2<<<(h + 31) / 32, dim3(32, 8), 0, s>>>(ws, dbias, nullptr, h, splits, accumulate);
}

void bias_dropout_residual(const void* z, const void* bias, const void* resid, void* out, int rows, int h,
                           uint64_t seed, uint32_t thresh16, float scale, cudaStream_t s, uint64_t elem_offset,
                           uint8_t* keep_out) {
  const int nvec_row = h / 8;
  dim3 grid((nvec_row + 255) / 256, rows);
  bias_dropout_residual_kernel<<<grid, 256, 0, s>>>((const uint4*)z, (const uint4*)bias, (const uint4*)resid,
                                                    (uint4*)out, nvec_row, seed, thresh16, scale, elem_offset,
                                                    keep_out);
}

#define MT_VPL_DISPATCH(SEQ, LAUNCH) \
  do {                               \
    const int need = ((SEQ) + 255) / 256; \
    if (need <= 1) LAUNCH(1);        \
    else if (need <= 2) LAUNCH(2);   \
    else if (need <= 4) LAUNCH(4);   \
    else if (need <= 8) LAUNCH(8);   \
    else LAUNCH(16);                 \
  } while (0)

void softmax_fwd(const void* S, void* P, float* lse, int batch_heads, int seq, long long head_base, uint64_t seed,
                 uint32_t thresh16, float scale, cudaStream_t s) {
  const int rows = batch_heads * seq;
  const int blocks = (rows + 7) / 8;
#define L(V)                                                                                                     \
  softmax_fwd_kernel<V><<<blocks, 256, 0, s>>>((const uint4*)S, (uint4*)P, lse, rows, seq, head_base, seed, thresh16, \
                                               scale)
  MT_VPL_DISPATCH(seq, L);
#undef L
}

void softmax_bwd_rowdot(const void* S, const float* lse, const float* D, void* dP, int batch_heads, int seq,
                        long long head_base, uint64_t seed, uint32_t thresh16, float scale, float alpha,
                        cudaStream_t s) {
  const int rows = batch_heads * seq;
  softmax_bwd_rowdot_kernel<<<(rows + 7) / 8, 256, 0, s>>>((const uint4*)S, lse, D, (uint4*)dP, rows, seq, head_base,
                                                           seed, thresh16, scale, alpha);
}


void mse_loss(const void* y, const void* t, void* dy, float* loss, long long n, cudaStream_t s, long long n_total) {
  const long long nvec = n / 8;
  mse_loss_kernel<<<grid_for(nvec, 256), 256, 0, s>>>((const uint4*)y, (const uint4*)t, (uint4*)dy, loss, nvec,
                                                      1.f / (float)(n_total > 0 ? n_total : n));
}

void fill_normal(void* out, long long rows, long long cols, long long global_cols, long long row0, long long col0,
                 uint64_t key, float mean, float std, cudaStream_t s) {
  fill_normal_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>((__nv_bfloat16*)out, rows, cols, global_cols, row0,
                                                                col0, key, mean, std);
}

void fill_zero_f32(float* p, size_t n, cudaStream_t s) {
  fill_zero_kernel<<<grid_for((long long)n, 256), 256, 0, s>>>(p, n);
}

}  // namespace mt
