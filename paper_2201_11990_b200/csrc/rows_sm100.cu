// Row-wise HBM-bound kernels of the layer (LayerNorm forward / backward, bias + dropout + residual
// [+ LayerNorm]) as persistent, TMA-fed pipelines: one 512-thread CTA per SM walks its rows while
// the bulk-copy engine (cp.async.bulk, mbarrier completion) streams the next rows' inputs into a
// 2-3 deep shared-memory ring, so HBM reads are always in flight without spending registers on them
// (the previous one-CTA-per-row kernels stalled on every row's load -> reduce -> store chain and ran
// at 2.6-3.4 TB/s). Outputs are written with coalesced 16-byte stores.
//
// The LayerNorm backward also accumulates the gamma / beta gradient partials of its rows in registers
// (each thread owns fixed columns) and writes one partial per CTA, so dy and x are read once instead
// of twice; colsum_stage2 sums the per-CTA partials (deterministic order).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <utility>

#include "curator/dropout.hpp"
#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace mt {
namespace {

constexpr int kRowThreads = 512;
constexpr int kRowSmemBudget = 200 * 1024;

__device__ __forceinline__ void bulk_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void unpack8f(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 p = unpack_bf16x2(w[q]);
    f[2 * q] = p.x;
    f[2 * q + 1] = p.y;
  }
}
__device__ __forceinline__ uint4 pack8f(const float (&f)[8]) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                    pack_bf16x2(f[6], f[7]));
}

__device__ __forceinline__ float row_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red may still be read by the previous reduction
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = l < (int)(blockDim.x >> 5) ? red[l] : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// Two row sums with one pair of barriers (same shuffle / slot order as row_sum, so bit-identical).
__device__ __forceinline__ float2 row_sum2(float a, float b, float2* red2) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red2 may still be read by the previous reduction
  if (l == 0) red2[w] = make_float2(a, b);
  __syncthreads();
  float2 t = l < (int)(blockDim.x >> 5) ? red2[l] : make_float2(0.f, 0.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
    t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
  }
  return t;
}

__device__ __forceinline__ uint32_t keep_mask8_rows(uint64_t seed, uint64_t idx, uint32_t thresh16) {
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

// Ring of `stages` x `nin` row buffers + one mbarrier per stage. Thread 0 issues the loads. With a
// split row (kSplit = 2) each CTA's buffers hold its half of the row's columns (col_off bytes in).
struct Ring {
  uint8_t* buf;
  uint64_t* bar;
  int stages, nin;
  uint32_t row_bytes;  // bytes of this CTA's part of a row
  size_t row_stride;   // bytes of a whole row in global memory
  uint32_t col_off;    // byte offset of this CTA's part within the row
  __device__ uint8_t* slot(int s, int i) const { return buf + ((size_t)s * nin + i) * row_bytes; }
  __device__ void issue(int s, const void* const* src, long long row) const {
    const uint32_t b = smem_u32(&bar[s]);
    mbar_arrive_expect_tx(b, (uint32_t)nin * row_bytes);
    for (int i = 0; i < nin; ++i)
      bulk_load_1d(smem_u32(slot(s, i)), static_cast<const uint8_t*>(src[i]) + (size_t)row * row_stride + col_off,
                   row_bytes, b);
  }
};

// Exchange of per-row partials between the two CTAs of a cluster that split every row's columns: each
// CTA stores its pair of floats into the peer's slot with st.async, which completes the transaction on
// the peer's mbarrier for that slot (4 slots rotate over the rows: a slot is rewritten only after the
// peer has passed three later exchanges, long after it read the slot).
constexpr int kXSlots = 4;
struct RowXchg {
  float2* slot;   // [kXSlots], written by the peer
  uint64_t* bar;  // [kXSlots], one arrival (the local expect_tx) + 8 transaction bytes
};

__device__ __forceinline__ RowXchg make_xchg(uint8_t* base) {
  RowXchg x;
  x.bar = reinterpret_cast<uint64_t*>(base);
  x.slot = reinterpret_cast<float2*>(base + kXSlots * sizeof(uint64_t));
  if (threadIdx.x == 0) {
    for (int i = 0; i < kXSlots; ++i) mbar_init(smem_u32(&x.bar[i]), 1);
    fence_barrier_init();
  }
  return x;
}

// Returns (part 0's value, part 1's value) for row iteration k: this CTA's `mine` and the peer's.
__device__ __forceinline__ void xchg_row(const RowXchg& x, int k, uint32_t part, float2 mine, float2& p0, float2& p1) {
  const int i = k & (kXSlots - 1);
  const uint32_t bar = smem_u32(&x.bar[i]);
  if (threadIdx.x == 0) {
    uint32_t rslot, rbar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rslot) : "r"(smem_u32(&x.slot[i])), "r"(part ^ 1u));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar), "r"(part ^ 1u));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(rslot),
                 "f"(mine.x), "f"(mine.y), "r"(rbar)
                 : "memory");
    mbar_arrive_expect_tx(bar, 8);
  }
  mbar_wait(bar, (k / kXSlots) & 1);
  const float2 peer = x.slot[i];
  p0 = part == 0 ? mine : peer;
  p1 = part == 0 ? peer : mine;
}

// LayerNorm statistics of a row from shifted sums s1 = sum(x - c), s2 = sum((x - c)^2) over n values.
// Split rows: each part has its own shift (its first element); the halves' (mean, M2) are combined in
// part order (Chan et al.), so both CTAs compute the same bits.
template <int kSplit>
__device__ __forceinline__ void ln_stats(const RowXchg& x, int k, uint32_t part, float c, float s1, float s2,
                                         float inv_h, float eps, float& mu, float& rs) {
  if constexpr (kSplit == 1) {
    const float md = s1 * inv_h;
    mu = c + md;
    rs = rsqrtf(fmaxf(s2 * inv_h - md * md, 0.f) + eps);
  } else {
    const float inv_n = 2.f * inv_h;  // values per part = h / 2
    const float md = s1 * inv_n;
    float2 a, b;
    xchg_row(x, k, part, make_float2(c + md, s2 - s1 * md), a, b);
    const float d = b.x - a.x;
    mu = 0.5f * (a.x + b.x);
    const float m2 = a.y + b.y + d * d * (0.25f / inv_h);  // n0 n1 / n = h / 4
    rs = rsqrtf(fmaxf(m2 * inv_h, 0.f) + eps);
  }
}

__device__ __forceinline__ Ring make_ring(uint8_t* smem, int stages, int nin, uint32_t row_bytes, size_t row_stride,
                                          uint32_t col_off) {
  Ring r;
  r.buf = smem;
  r.bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * nin * row_bytes);
  r.stages = stages;
  r.nin = nin;
  r.row_bytes = row_bytes;
  r.row_stride = row_stride;
  r.col_off = col_off;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&r.bar[s]), 1);
    fence_barrier_init();
  }
  return r;
}

// Where a CTA sits: `unit` walks rows unit, unit + units, ...; `part` is its half of each row's columns.
template <int kSplit>
struct RowPlace {
  uint32_t part;
  int unit, units, nvh;  // nvh: this CTA's vectors (8 bf16) per row
  __device__ RowPlace(int nvec) {
    part = kSplit == 2 ? cluster_ctarank() : 0u;
    unit = (int)blockIdx.x / kSplit;
    units = (int)gridDim.x / kSplit;
    nvh = nvec / kSplit;
  }
  __device__ int rows_of(int rows) const { return rows > unit ? (rows - 1 - unit) / units + 1 : 0; }
  __device__ long long row(int k) const { return unit + (long long)k * units; }
  __device__ int col0() const { return (int)part * nvh; }  // first vector of this CTA's columns
};

// smem bytes after the ring: its mbarriers, then (split rows) the exchange slots
constexpr size_t kRingTail = 256;

// Forward row kernels: every thread owns the fixed vectors v = tid + i*T (i < VPT) of every row (of its
// half of every row when kSplit = 2: a cluster of two CTAs splits each row's columns, which halves the
// registers and ring bytes per CTA for the wide rows — h = 20480 spilled otherwise), so the per-column
// parameters (gamma, beta, bias) are loaded once per CTA into registers, each row is unpacked from smem
// into fp32 registers once, and the LayerNorm needs a single block reduction per row (+ one exchange
// with the peer CTA): shifted sums s1 = sum(x - c), s2 = sum((x - c)^2) around c = the first element
// (mean = c + s1/n, var = s2/n - (s1/n)^2, robust to a large row mean). The ring slot is handed back to
// the bulk-copy engine right after that reduction (all reads of the row happened before it).
template <int VPT>
__device__ __forceinline__ void load_params(const uint4* __restrict__ p, uint4 (&out)[VPT], int nvh, int T) {
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int v = (int)threadIdx.x + i * T;
    out[i] = v < nvh ? __ldg(p + v) : make_uint4(0, 0, 0, 0);
  }
}

template <int T, int VPT, int kSplit>
__global__ void __launch_bounds__(T) ln_fwd_rows_kernel(const uint4* __restrict__ x, const uint4* __restrict__ gamma,
                                                        const uint4* __restrict__ beta, uint4* __restrict__ y,
                                                        float* __restrict__ mean, float* __restrict__ rstd, int rows,
                                                        int nvec, float inv_h, float eps, int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red2[32];
  const RowPlace<kSplit> pl(nvec);
  const int nvh = pl.nvh, col0 = pl.col0();
  const Ring ring = make_ring(smem, stages, 1, (uint32_t)nvh * 16, (size_t)nvec * 16, (uint32_t)col0 * 16);
  const RowXchg xg = make_xchg(smem + (size_t)stages * nvh * 16 + 64);
  if constexpr (kSplit == 2) cluster_sync(); else __syncthreads();
  const void* src[1] = {x};
  uint4 gp[VPT], bp[VPT];
  load_params<VPT>(gamma + col0, gp, nvh, T);
  load_params<VPT>(beta + col0, bp, nvh, T);
  const int nk = pl.rows_of(rows);
  if (threadIdx.x == 0)
    for (int k = 0; k < min(stages, nk); ++k) ring.issue(k, src, pl.row(k));
  for (int k = 0; k < nk; ++k) {
    const int s = k % stages;
    const long long row = pl.row(k);
    mbar_wait(smem_u32(&ring.bar[s]), (k / stages) & 1);
    const uint4* xs = reinterpret_cast<const uint4*>(ring.slot(s, 0));
    uint4 xp[VPT];  // the row stays packed (bf16) in registers: 4 registers per 8 values
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int v = (int)threadIdx.x + i * T;
      xp[i] = v < nvh ? xs[v] : make_uint4(0, 0, 0, 0);
    }
    const float c = __uint_as_float(reinterpret_cast<const uint32_t*>(xs)[0] << 16);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      if ((int)threadIdx.x + i * T < nvh) {
        float o[8];
        unpack8f(xp[i], o);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = o[j] - c;
          s1 += d;
          s2 = fmaf(d, d, s2);
        }
      }
    }
    // the reduction is also the barrier after which every thread has read slot s: refill it now
    const float2 t = row_sum2(s1, s2, red2);
    if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, pl.row(k + stages));
    float mu, rs;
    ln_stats<kSplit>(xg, k, pl.part, c, t.x, t.y, inv_h, eps, mu, rs);
    const float nmr = -mu * rs;
    uint4* yr = y + row * nvec + col0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int v = (int)threadIdx.x + i * T;
      if (v < nvh) {
        float o[8], g[8], b[8], r[8];
        unpack8f(xp[i], o);
        unpack8f(gp[i], g);
        unpack8f(bp[i], b);
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = fmaf(fmaf(o[j], rs, nmr), g[j], b[j]);
        yr[v] = pack8f(r);
      }
    }
    if (threadIdx.x == 0 && pl.part == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  }
  if constexpr (kSplit == 2) cluster_sync();  // the peer's last exchange into this CTA's smem has landed
}

// out = resid + dropout(z + bias) (written), then optionally y = LayerNorm(out) from the same registers.
template <int T, int VPT, bool kLN, int kSplit>
__global__ void __launch_bounds__(T)
    bdr_ln_rows_kernel(const uint4* __restrict__ z, const uint4* __restrict__ bias, const uint4* __restrict__ resid,
                       uint4* __restrict__ out, const uint4* __restrict__ gamma, const uint4* __restrict__ beta,
                       uint4* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int rows, int nvec,
                       float inv_h, float eps, uint64_t seed, uint32_t thresh16, float scale, uint64_t elem_offset,
                       int stages, uint8_t* __restrict__ keep_out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red2[32];
  const RowPlace<kSplit> pl(nvec);
  const int nvh = pl.nvh, col0 = pl.col0();
  const Ring ring = make_ring(smem, stages, 2, (uint32_t)nvh * 16, (size_t)nvec * 16, (uint32_t)col0 * 16);
  const RowXchg xg = make_xchg(smem + (size_t)stages * 2 * nvh * 16 + 64);
  if constexpr (kSplit == 2) cluster_sync(); else __syncthreads();
  const void* src[2] = {z, resid};
  uint4 bi[VPT], gp[kLN ? VPT : 1], bp[kLN ? VPT : 1];
  load_params<VPT>(bias + col0, bi, nvh, T);
  if constexpr (kLN) {
    load_params<VPT>(gamma + col0, gp, nvh, T);
    load_params<VPT>(beta + col0, bp, nvh, T);
  }
  const int nk = pl.rows_of(rows);
  if (threadIdx.x == 0)
    for (int k = 0; k < min(stages, nk); ++k) ring.issue(k, src, pl.row(k));
  for (int k = 0; k < nk; ++k) {
    const int s = k % stages;
    const long long row = pl.row(k);
    mbar_wait(smem_u32(&ring.bar[s]), (k / stages) & 1);
    const uint4* zs = reinterpret_cast<const uint4*>(ring.slot(s, 0));
    const uint4* rs_ = reinterpret_cast<const uint4*>(ring.slot(s, 1));
    uint4 ob[VPT];  // the stored (bf16) residual stream, which is what the LayerNorm sees
    uint4* outr = out + row * nvec + col0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int v = (int)threadIdx.x + i * T;
      ob[i] = make_uint4(0, 0, 0, 0);
      if (v < nvh) {
        float a[8], b[8], r[8], o[8];
        unpack8f(zs[v], a);
        unpack8f(bi[i], b);
        unpack8f(rs_[v], r);
        const uint32_t keep =
            keep_mask8_rows(seed, elem_offset + ((uint64_t)row * nvec + col0 + v) * 8, thresh16);
        if (keep_out != nullptr) keep_out[row * nvec + col0 + v] = (uint8_t)keep;  // coalesced bytes
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = r[j] + (((keep >> j) & 1u) ? (a[j] + b[j]) * scale : 0.f);
        ob[i] = pack8f(o);
        outr[v] = ob[i];
      }
    }
    if constexpr (!kLN) {
      __syncthreads();  // every thread read slot s
      if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, pl.row(k + stages));
      continue;
    } else {
      // shift: the part's first output element (thread 0 owns its vector 0); broadcast through smem
      __shared__ float c_sh;
      if (threadIdx.x == 0) c_sh = __uint_as_float(ob[0].x << 16);
      float s1 = 0.f, s2 = 0.f;
      __syncthreads();
      const float c = c_sh;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if ((int)threadIdx.x + i * T < nvh) {
          float o[8];
          unpack8f(ob[i], o);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float d = o[j] - c;
            s1 += d;
            s2 = fmaf(d, d, s2);
          }
        }
      }
      const float2 t = row_sum2(s1, s2, red2);  // also: every thread finished reading slot s
      if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, pl.row(k + stages));
      float mu, rs;
      ln_stats<kSplit>(xg, k, pl.part, c, t.x, t.y, inv_h, eps, mu, rs);
      const float nmr = -mu * rs;
      uint4* yr = y + row * nvec + col0;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = (int)threadIdx.x + i * T;
        if (v < nvh) {
          float o[8], g[8], b[8], r[8];
          unpack8f(ob[i], o);
          unpack8f(gp[i], g);
          unpack8f(bp[i], b);
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] = fmaf(fmaf(o[j], rs, nmr), g[j], b[j]);
          yr[v] = pack8f(r);
        }
      }
      if (threadIdx.x == 0 && pl.part == 0) {
        mean[row] = mu;
        rstd[row] = rs;
      }
    }
  }
  if constexpr (kSplit == 2) cluster_sync();
}

// LayerNorm backward: dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)) [+ resid], and the
// per-unit partial sums of dgamma = sum(dy * xhat), dbeta = sum(dy) over this unit's rows
// (ws[0][unit][col], ws[1][unit][col]). MAXV = vectors per thread (ceil(nvh / 512)). Split rows: the
// two row sums are exchanged with the peer CTA and added in part order.
template <int MAXV, int kSplit>
__global__ void __launch_bounds__(kRowThreads, 1)
    ln_bwd_rows_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ x, const uint4* __restrict__ gamma,
                       const float* __restrict__ mean, const float* __restrict__ rstd, const uint4* __restrict__ resid,
                       uint4* __restrict__ dx, float* __restrict__ ws, int rows, int nvec, float inv_h, int stages,
                       int nin) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red2[32];
  const RowPlace<kSplit> pl(nvec);
  const int nvh = pl.nvh, col0 = pl.col0();
  // nin == 3: the residual-gradient rows are streamed through the ring too (when they fit in smem)
  const Ring ring = make_ring(smem, stages, nin, (uint32_t)nvh * 16, (size_t)nvec * 16, (uint32_t)col0 * 16);
  const RowXchg xg = make_xchg(smem + (size_t)stages * nin * nvh * 16 + 64);
  if constexpr (kSplit == 2) cluster_sync(); else __syncthreads();
  const void* src[3] = {dy, x, resid};
  float dg[MAXV][8], db[MAXV][8];
#pragma unroll
  for (int i = 0; i < MAXV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) dg[i][j] = db[i][j] = 0.f;
  uint4 gp[MAXV];  // gamma of this thread's vectors, loaded once per CTA
  load_params<MAXV>(gamma + col0, gp, nvh, kRowThreads);
  const int nk = pl.rows_of(rows);
  if (threadIdx.x == 0)
    for (int k = 0; k < min(stages, nk); ++k) ring.issue(k, src, pl.row(k));
  for (int k = 0; k < nk; ++k) {
    const int s = k % stages;
    const long long row = pl.row(k);
    mbar_wait(smem_u32(&ring.bar[s]), (k / stages) & 1);
    const uint4* dys = reinterpret_cast<const uint4*>(ring.slot(s, 0));
    const uint4* xs = reinterpret_cast<const uint4*>(ring.slot(s, 1));
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int v = threadIdx.x + i * kRowThreads;
      if (v < nvh) {
        float d[8], xv[8], g[8];
        unpack8f(dys[v], d);
        unpack8f(xs[v], xv);
        unpack8f(gp[i], g);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xv[j] - mu) * rs;
          const float dgj = d[j] * g[j];
          s1 += dgj;
          s2 += dgj * xh;
          dg[i][j] += d[j] * xh;
          db[i][j] += d[j];
        }
      }
    }
    float2 sums = row_sum2(s1, s2, red2);
    if constexpr (kSplit == 2) {
      float2 a, b;
      xchg_row(xg, k, pl.part, sums, a, b);
      sums = make_float2(a.x + b.x, a.y + b.y);
    }
    const float m1 = sums.x * inv_h, m2 = sums.y * inv_h;
    const size_t rbase = (size_t)row * nvec + col0;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int v = threadIdx.x + i * kRowThreads;
      if (v < nvh) {
        float d[8], xv[8], g[8], o[8];
        unpack8f(dys[v], d);
        unpack8f(xs[v], xv);
        unpack8f(gp[i], g);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (d[j] * g[j] - m1 - (xv[j] - mu) * rs * m2);
        if (resid != nullptr) {
          float r[8];
          unpack8f(nin == 3 ? reinterpret_cast<const uint4*>(ring.slot(s, 2))[v] : resid[rbase + v], r);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += r[j];
        }
        dx[rbase + v] = pack8f(o);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, pl.row(k + stages));
  }
  const size_t n = (size_t)nvec * 8;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int v = threadIdx.x + i * kRowThreads;
    if (v < nvh) {
      float* g0 = ws + (size_t)pl.unit * n + (size_t)(col0 + v) * 8;
      float* b0 = ws + ((size_t)pl.units + pl.unit) * n + (size_t)(col0 + v) * 8;
      *reinterpret_cast<float4*>(g0) = make_float4(dg[i][0], dg[i][1], dg[i][2], dg[i][3]);
      *reinterpret_cast<float4*>(g0 + 4) = make_float4(dg[i][4], dg[i][5], dg[i][6], dg[i][7]);
      *reinterpret_cast<float4*>(b0) = make_float4(db[i][0], db[i][1], db[i][2], db[i][3]);
      *reinterpret_cast<float4*>(b0 + 4) = make_float4(db[i][4], db[i][5], db[i][6], db[i][7]);
    }
  }
  if constexpr (kSplit == 2) cluster_sync();
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Ring depth for `nin` inputs of `row_bytes` each (0: the row does not fit -> caller falls back).
int ring_stages(int nin, size_t row_bytes) {
  const size_t per = (size_t)nin * row_bytes;
  const int st = (int)std::min<size_t>(3, (kRowSmemBudget - kRingTail) / per);
  return st >= 2 ? st : 0;
}

// Rows wider than 1536 vectors (h > 12288) are split over a cluster of two CTAs in the kernels that keep
// the most per-thread state (bias-dropout-residual + LayerNorm, LayerNorm backward): whole rows there
// need >= 4 vectors per thread and spill (h = 20480: 110 -> 86 us and 131 -> 84 us). The lighter kernels
// (LayerNorm forward, bias-dropout-residual) and rows up to 12288 are faster whole (the per-row
// exchange costs more than it saves: ln_bwd at h = 12288 49.6 vs 60 us split). MT_ROWS_SPLIT (read per
// call, for A/B measurements and tests): 1 = whole rows everywhere, 2 = split every even-width row.
int row_split(int nvec, bool heavy) {
  const char* e = getenv("MT_ROWS_SPLIT");
  if (e != nullptr && e[0] == '1') return 1;
  if (nvec % 2 != 0) return 1;
  if (e != nullptr && e[0] == '2') return 2;
  return heavy && nvec > 1536 ? 2 : 1;
}

// Launches a row kernel on exactly its resident CTAs (clusters of `split`): a second wave of CTAs would
// restart the ring and expose its fill latency again (ln_fwd at h = 12288: 24.3 -> 21.0 us, faster
// than a 50 MB + 50 MB device copy, 22.4 us — profiles/r02_ncu_summary.md). Returns the number of
// row units (CTAs / split, at most max_units), 0 on failure.
template <class... P, class... A>
int launch_rows(void (*kern)(P...), int split, int threads, size_t smem, int rows, int max_units, cudaStream_t s,
                A&&... args) {
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  int units = 0;
  if (split == 2) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2 * sm_count());
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc < 1) nc = sm_count() / 2;
    units = std::max(1, std::min(std::min(rows, max_units), nc));
    cfg.gridDim = dim3(2 * units);
  } else {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem) != cudaSuccess || per < 1) per = 1;
    units = std::max(1, std::min(std::min(rows, max_units), std::min(per, 4) * sm_count()));
    cfg.gridDim = dim3(units);
  }
  if (cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...) != cudaSuccess) return 0;
  return units;
}

}  // namespace

int row_kernel_ctas(int rows) { return std::max(1, std::min(rows, sm_count())); }

// Forward row kernels: T threads per CTA owning VPT <= 6 vectors (8 bf16) of every row (part) each.
struct RowLaunch {
  int split, threads, vpt, stages;
  size_t smem;
};
RowLaunch fwd_launch(int nvec, int nin, bool heavy) {
  RowLaunch l{};
  l.split = row_split(nvec, heavy);
  const int nvh = nvec / l.split;
  l.threads = nvh <= 3 * 256 ? 256 : 512;  // 512 threads = 16 warps for the wide rows
  l.vpt = (nvh + l.threads - 1) / l.threads;
  const size_t row_bytes = (size_t)nvh * 16;
  l.stages = 3;
  while (l.stages > 2 && (size_t)l.stages * nin * row_bytes + kRingTail > (size_t)kRowSmemBudget) --l.stages;
  l.smem = (size_t)l.stages * nin * row_bytes + kRingTail;
  return l;
}

bool ln_fwd_rows(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows, int h,
                 float eps, cudaStream_t s) {
  const int nvec = h / 8;
  const RowLaunch L = fwd_launch(nvec, 1, false);
  if (h % 8 || nvec > 6 * 512 * L.split) return false;
  if ((size_t)2 * nvec / L.split * 16 + kRingTail > (size_t)kRowSmemBudget || L.vpt > 6) return false;
  int units = 0;
#define LN(T, V)                                                                                                  \
  do {                                                                                                            \
    if (L.split == 2)                                                                                             \
      units = launch_rows(ln_fwd_rows_kernel<T, V, 2>, 2, T, L.smem, rows, 1 << 30, s, (const uint4*)x, (const uint4*)gamma, \
                          (const uint4*)beta, (uint4*)y, mean, rstd, rows, nvec, 1.f / h, eps, L.stages);         \
    else                                                                                                          \
      units = launch_rows(ln_fwd_rows_kernel<T, V, 1>, 1, T, L.smem, rows, 1 << 30, s, (const uint4*)x, (const uint4*)gamma, \
                          (const uint4*)beta, (uint4*)y, mean, rstd, rows, nvec, 1.f / h, eps, L.stages);         \
  } while (0)
  if (L.threads == 256) {
    switch (L.vpt) {
      case 1: LN(256, 1); break;
      case 2: LN(256, 2); break;
      default: LN(256, 3); break;
    }
  } else {
    switch (L.vpt) {
      case 2: LN(512, 2); break;
      case 3: LN(512, 3); break;
      case 4: LN(512, 4); break;
      case 5: LN(512, 5); break;
      default: LN(512, 6); break;
    }
  }
#undef LN
  return units > 0 && cudaGetLastError() == cudaSuccess;
}

bool bdr_ln_rows(const void* z, const void* bias, const void* resid, void* out, const void* gamma, const void* beta,
                 void* y, float* mean, float* rstd, int rows, int h, float eps, uint64_t seed, uint32_t thresh16,
                 float scale, uint64_t elem_offset, cudaStream_t s, uint8_t* keep_out) {
  const int nvec = h / 8;
  const RowLaunch L = fwd_launch(nvec, 2, gamma != nullptr);
  if (h % 8 || nvec > 6 * 512 * L.split) return false;
  if ((size_t)2 * 2 * nvec / L.split * 16 + kRingTail > (size_t)kRowSmemBudget || L.vpt > 6) return false;
  int units = 0;
#define BDR(T, V, LNF)                                                                                           \
  do {                                                                                                           \
    if (L.split == 2)                                                                                            \
      units = launch_rows(bdr_ln_rows_kernel<T, V, LNF, 2>, 2, T, L.smem, rows, 1 << 30, s, (const uint4*)z,              \
                          (const uint4*)bias, (const uint4*)resid, (uint4*)out, (const uint4*)gamma,             \
                          (const uint4*)beta, (uint4*)y, mean, rstd, rows, nvec, 1.f / h, eps, seed, thresh16,   \
                          scale, elem_offset, L.stages, keep_out);                                               \
    else                                                                                                         \
      units = launch_rows(bdr_ln_rows_kernel<T, V, LNF, 1>, 1, T, L.smem, rows, 1 << 30, s, (const uint4*)z,              \
                          (const uint4*)bias, (const uint4*)resid, (uint4*)out, (const uint4*)gamma,             \
                          (const uint4*)beta, (uint4*)y, mean, rstd, rows, nvec, 1.f / h, eps, seed, thresh16,   \
                          scale, elem_offset, L.stages, keep_out);                                               \
  } while (0)
#define BDR_V256(LNF)                \
  switch (L.vpt) {                   \
    case 1: BDR(256, 1, LNF); break; \
    case 2: BDR(256, 2, LNF); break; \
    default: BDR(256, 3, LNF); break; \
  }
#define BDR_V512(LNF)                \
  switch (L.vpt) {                   \
    case 2: BDR(512, 2, LNF); break; \
    case 3: BDR(512, 3, LNF); break; \
    case 4: BDR(512, 4, LNF); break; \
    case 5: BDR(512, 5, LNF); break; \
    default: BDR(512, 6, LNF); break; \
  }
  if (L.threads == 256) {
    if (gamma != nullptr) {
      BDR_V256(true)
    } else {
      BDR_V256(false)
    }
  } else {
    if (gamma != nullptr) {
      BDR_V512(true)
    } else {
      BDR_V512(false)
    }
  }
#undef BDR_V256
#undef BDR_V512
#undef BDR
  return units > 0 && cudaGetLastError() == cudaSuccess;
}

// Fused LayerNorm backward (dx and gamma/beta gradients in one pass). ws must hold
// 2 * row_kernel_ctas(rows) * h floats.
bool ln_bwd_rows(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                 const void* resid, void* dx, float* dgamma, float* dbeta, int rows, int h, float* ws, bool accumulate,
                 cudaStream_t s) {
  const int nvec = h / 8;
  if (h % 8) return false;
  const int split = row_split(nvec, true);
  const int nvh = nvec / split;
  const int nin = (resid != nullptr && ring_stages(3, (size_t)nvh * 16) != 0) ? 3 : 2;
  const int stages = ring_stages(nin, (size_t)nvh * 16);
  const int maxv = (nvh + kRowThreads - 1) / kRowThreads;
  if (stages == 0 || maxv > 6) return false;
  const size_t smem = (size_t)stages * nin * nvh * 16 + kRingTail;
  int units = 0;
#define L(V)                                                                                                         \
  do {                                                                                                               \
    if (split == 2)                                                                                                  \
      units = launch_rows(ln_bwd_rows_kernel<V, 2>, 2, kRowThreads, smem, rows, row_kernel_ctas(rows), s, (const uint4*)dy, (const uint4*)x, \
                          (const uint4*)gamma, mean, rstd, (const uint4*)resid, (uint4*)dx, ws, rows, nvec, 1.f / h,  \
                          stages, nin);                                                                              \
    else                                                                                                             \
      units = launch_rows(ln_bwd_rows_kernel<V, 1>, 1, kRowThreads, smem, rows, row_kernel_ctas(rows), s, (const uint4*)dy, (const uint4*)x, \
                          (const uint4*)gamma, mean, rstd, (const uint4*)resid, (uint4*)dx, ws, rows, nvec, 1.f / h,  \
                          stages, nin);                                                                              \
  } while (0)
  switch (maxv) {
    case 1: L(1); break;
    case 2: L(2); break;
    case 3: L(3); break;
    case 4: L(4); break;
    case 5: L(5); break;
    default: L(6); break;
  }
#undef L
  if (units == 0 || cudaGetLastError() != cudaSuccess) return false;
  colsum_partials(ws, dgamma, dbeta, h, units, accumulate, s);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace mt
