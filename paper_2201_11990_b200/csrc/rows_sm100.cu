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

// Ring of `stages` x `nin` row buffers + one mbarrier per stage. Thread 0 issues the loads.
struct Ring {
  uint8_t* buf;
  uint64_t* bar;
  int stages, nin;
  uint32_t row_bytes;
  __device__ uint8_t* slot(int s, int i) const { return buf + ((size_t)s * nin + i) * row_bytes; }
  __device__ void issue(int s, const void* const* src, long long row) const {
    const uint32_t b = smem_u32(&bar[s]);
    mbar_arrive_expect_tx(b, (uint32_t)nin * row_bytes);
    for (int i = 0; i < nin; ++i)
      bulk_load_1d(smem_u32(slot(s, i)), static_cast<const uint8_t*>(src[i]) + (size_t)row * row_bytes, row_bytes, b);
  }
};

__device__ __forceinline__ Ring make_ring(uint8_t* smem, int stages, int nin, uint32_t row_bytes) {
  Ring r;
  r.buf = smem;
  r.bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * nin * row_bytes);
  r.stages = stages;
  r.nin = nin;
  r.row_bytes = row_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&r.bar[s]), 1);
    fence_barrier_init();
  }
  __syncthreads();
  return r;
}

// LayerNorm of one row held in smem (bf16 [h]): y = (x - mean) * rstd * gamma + beta.
__device__ __forceinline__ void ln_row(const uint4* xs, const uint4* __restrict__ gamma, const uint4* __restrict__ beta,
                                       uint4* __restrict__ y, float* mean_out, float* rstd_out, int nvec, float inv_h,
                                       float eps, float* red) {
  float s = 0.f;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    float x[8];
    unpack8f(xs[v], x);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
  }
  const float mu = row_sum(s, red) * inv_h;
  float q = 0.f;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    float x[8];
    unpack8f(xs[v], x);
#pragma unroll
    for (int j = 0; j < 8; ++j) q += (x[j] - mu) * (x[j] - mu);
  }
  const float rs = rsqrtf(row_sum(q, red) * inv_h + eps);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    float x[8], g[8], b[8], o[8];
    unpack8f(xs[v], x);
    unpack8f(__ldg(gamma + v), g);
    unpack8f(__ldg(beta + v), b);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (x[j] - mu) * rs * g[j] + b[j];
    y[v] = pack8f(o);
  }
  if (threadIdx.x == 0) {
    *mean_out = mu;
    *rstd_out = rs;
  }
}

__global__ void __launch_bounds__(kRowThreads, 1)
    ln_fwd_rows_kernel(const uint4* __restrict__ x, const uint4* __restrict__ gamma, const uint4* __restrict__ beta,
                       uint4* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int rows, int nvec,
                       float inv_h, float eps, int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float red[32];
  const Ring ring = make_ring(smem, stages, 1, (uint32_t)nvec * 16);
  const void* src[1] = {x};
  const int nk = rows > (int)blockIdx.x ? (rows - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < min(stages, nk); ++k) ring.issue(k, src, blockIdx.x + (long long)k * gridDim.x);
  for (int k = 0; k < nk; ++k) {
    const int s = k % stages;
    const long long row = blockIdx.x + (long long)k * gridDim.x;
    mbar_wait(smem_u32(&ring.bar[s]), (k / stages) & 1);
    ln_row(reinterpret_cast<const uint4*>(ring.slot(s, 0)), gamma, beta, y + row * nvec, mean + row, rstd + row, nvec,
           inv_h, eps, red);
    __syncthreads();  // slot s fully consumed
    if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, blockIdx.x + (long long)(k + stages) * gridDim.x);
  }
}

// out = resid + dropout(z + bias) (written), then optionally y = LayerNorm(out).
__global__ void __launch_bounds__(kRowThreads, 1)
    bdr_ln_rows_kernel(const uint4* __restrict__ z, const uint4* __restrict__ bias, const uint4* __restrict__ resid,
                       uint4* __restrict__ out, const uint4* __restrict__ gamma, const uint4* __restrict__ beta,
                       uint4* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int rows, int nvec,
                       float inv_h, float eps, uint64_t seed, uint32_t thresh16, float scale, uint64_t elem_offset,
                       int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float red[32];
  const Ring ring = make_ring(smem, stages, 2, (uint32_t)nvec * 16);
  const void* src[2] = {z, resid};
  const int nk = rows > (int)blockIdx.x ? (rows - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < min(stages, nk); ++k) ring.issue(k, src, blockIdx.x + (long long)k * gridDim.x);
  for (int k = 0; k < nk; ++k) {
    const int s = k % stages;
    const long long row = blockIdx.x + (long long)k * gridDim.x;
    mbar_wait(smem_u32(&ring.bar[s]), (k / stages) & 1);
    uint4* zs = reinterpret_cast<uint4*>(ring.slot(s, 0));
    const uint4* rs_ = reinterpret_cast<const uint4*>(ring.slot(s, 1));
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      float a[8], b[8], r[8], o[8];
      unpack8f(zs[v], a);
      unpack8f(__ldg(bias + v), b);
      unpack8f(rs_[v], r);
      const uint32_t keep = keep_mask8_rows(seed, elem_offset + ((uint64_t)row * nvec + v) * 8, thresh16);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = r[j] + (((keep >> j) & 1u) ? (a[j] + b[j]) * scale : 0.f);
      const uint4 packed = pack8f(o);
      out[row * nvec + v] = packed;
      zs[v] = packed;  // LN input (each thread rewrites only its own vectors)
    }
    if (gamma != nullptr) {
      __syncthreads();
      ln_row(zs, gamma, beta, y + row * nvec, mean + row, rstd + row, nvec, inv_h, eps, red);
    }
    __syncthreads();
    if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, blockIdx.x + (long long)(k + stages) * gridDim.x);
  }
}

// LayerNorm backward: dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)) [+ resid], and the
// per-CTA partial sums of dgamma = sum(dy * xhat), dbeta = sum(dy) over this CTA's rows
// (ws[0][cta][col], ws[1][cta][col]). MAXV = vectors per thread (ceil(nvec / 512)).
template <int MAXV>
__global__ void __launch_bounds__(kRowThreads, 1)
    ln_bwd_rows_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ x, const uint4* __restrict__ gamma,
                       const float* __restrict__ mean, const float* __restrict__ rstd, const uint4* __restrict__ resid,
                       uint4* __restrict__ dx, float* __restrict__ ws, int rows, int nvec, float inv_h, int stages,
                       int nin) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red2[32];
  // nin == 3: the residual-gradient rows are streamed through the ring too (when they fit in smem)
  const Ring ring = make_ring(smem, stages, nin, (uint32_t)nvec * 16);
  const void* src[3] = {dy, x, resid};
  float dg[MAXV][8], db[MAXV][8];
#pragma unroll
  for (int i = 0; i < MAXV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) dg[i][j] = db[i][j] = 0.f;
  const int nk = rows > (int)blockIdx.x ? (rows - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < min(stages, nk); ++k) ring.issue(k, src, blockIdx.x + (long long)k * gridDim.x);
  for (int k = 0; k < nk; ++k) {
    const int s = k % stages;
    const long long row = blockIdx.x + (long long)k * gridDim.x;
    mbar_wait(smem_u32(&ring.bar[s]), (k / stages) & 1);
    const uint4* dys = reinterpret_cast<const uint4*>(ring.slot(s, 0));
    const uint4* xs = reinterpret_cast<const uint4*>(ring.slot(s, 1));
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int v = threadIdx.x + i * kRowThreads;
      if (v < nvec) {
        float d[8], xv[8], g[8];
        unpack8f(dys[v], d);
        unpack8f(xs[v], xv);
        unpack8f(__ldg(gamma + v), g);
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
    const float2 sums = row_sum2(s1, s2, red2);
    const float m1 = sums.x * inv_h, m2 = sums.y * inv_h;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int v = threadIdx.x + i * kRowThreads;
      if (v < nvec) {
        float d[8], xv[8], g[8], o[8];
        unpack8f(dys[v], d);
        unpack8f(xs[v], xv);
        unpack8f(__ldg(gamma + v), g);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (d[j] * g[j] - m1 - (xv[j] - mu) * rs * m2);
        if (resid != nullptr) {
          float r[8];
          unpack8f(nin == 3 ? reinterpret_cast<const uint4*>(ring.slot(s, 2))[v] : resid[row * nvec + v], r);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += r[j];
        }
        dx[row * nvec + v] = pack8f(o);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && k + stages < nk) ring.issue(s, src, blockIdx.x + (long long)(k + stages) * gridDim.x);
  }
  const size_t n = (size_t)nvec * 8;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int v = threadIdx.x + i * kRowThreads;
    if (v < nvec) {
      float* g0 = ws + (size_t)blockIdx.x * n + (size_t)v * 8;
      float* b0 = ws + ((size_t)gridDim.x + blockIdx.x) * n + (size_t)v * 8;
      *reinterpret_cast<float4*>(g0) = make_float4(dg[i][0], dg[i][1], dg[i][2], dg[i][3]);
      *reinterpret_cast<float4*>(g0 + 4) = make_float4(dg[i][4], dg[i][5], dg[i][6], dg[i][7]);
      *reinterpret_cast<float4*>(b0) = make_float4(db[i][0], db[i][1], db[i][2], db[i][3]);
      *reinterpret_cast<float4*>(b0 + 4) = make_float4(db[i][4], db[i][5], db[i][6], db[i][7]);
    }
  }
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
  const int st = (int)std::min<size_t>(3, (kRowSmemBudget - 64) / per);
  return st >= 2 ? st : 0;
}

template <class K>
bool set_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
}

}  // namespace

int row_kernel_ctas(int rows) { return std::max(1, std::min(rows, sm_count())); }

// Element-wise row kernels (no per-thread column state): 256-thread CTAs, as many per SM as the
// shared-memory ring allows (2-deep rings; more resident warps hide the per-row dependency chains).
struct RowLaunch {
  int ctas, threads, stages;
  size_t smem;
};
RowLaunch small_cta_launch(int rows, int nin, size_t row_bytes) {
  RowLaunch l{};
  l.threads = 256;
  l.stages = 2;
  l.smem = (size_t)l.stages * nin * row_bytes + 64;
  const int per_sm = std::max(1, std::min(4, (int)((227 * 1024) / (l.smem + 1024))));
  l.ctas = std::max(1, std::min(rows, per_sm * sm_count()));
  return l;
}

bool ln_fwd_rows(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows, int h,
                 float eps, cudaStream_t s) {
  const int nvec = h / 8;
  if (h % 8 || ring_stages(1, (size_t)nvec * 16) == 0) return false;
  const RowLaunch L = small_cta_launch(rows, 1, (size_t)nvec * 16);
  if (!set_smem(ln_fwd_rows_kernel, L.smem)) return false;
  ln_fwd_rows_kernel<<<L.ctas, L.threads, L.smem, s>>>((const uint4*)x, (const uint4*)gamma, (const uint4*)beta,
                                                      (uint4*)y, mean, rstd, rows, nvec, 1.f / h, eps, L.stages);
  return cudaGetLastError() == cudaSuccess;
}

bool bdr_ln_rows(const void* z, const void* bias, const void* resid, void* out, const void* gamma, const void* beta,
                 void* y, float* mean, float* rstd, int rows, int h, float eps, uint64_t seed, uint32_t thresh16,
                 float scale, uint64_t elem_offset, cudaStream_t s) {
  const int nvec = h / 8;
  if (h % 8 || ring_stages(2, (size_t)nvec * 16) == 0) return false;
  const RowLaunch L = small_cta_launch(rows, 2, (size_t)nvec * 16);
  if (!set_smem(bdr_ln_rows_kernel, L.smem)) return false;
  bdr_ln_rows_kernel<<<L.ctas, L.threads, L.smem, s>>>(
      (const uint4*)z, (const uint4*)bias, (const uint4*)resid, (uint4*)out, (const uint4*)gamma, (const uint4*)beta,
      (uint4*)y, mean, rstd, rows, nvec, 1.f / h, eps, seed, thresh16, scale, elem_offset, L.stages);
  return cudaGetLastError() == cudaSuccess;
}

// Fused LayerNorm backward (dx and gamma/beta gradients in one pass). ws must hold
// 2 * row_kernel_ctas(rows) * h floats.
bool ln_bwd_rows(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                 const void* resid, void* dx, float* dgamma, float* dbeta, int rows, int h, float* ws, bool accumulate,
                 cudaStream_t s) {
  const int nvec = h / 8;
  const int nin = (resid != nullptr && ring_stages(3, (size_t)nvec * 16) != 0) ? 3 : 2;
  const int stages = ring_stages(nin, (size_t)nvec * 16);
  const int maxv = (nvec + kRowThreads - 1) / kRowThreads;
  if (h % 8 || stages == 0 || maxv > 6) return false;
  const size_t smem = (size_t)stages * nin * nvec * 16 + 64;
  const int ctas = row_kernel_ctas(rows);
  bool ok = true;
#define L(V)                                                                                                       \
  do {                                                                                                             \
    ok = set_smem(ln_bwd_rows_kernel<V>, smem);                                                                    \
    if (ok)                                                                                                        \
      ln_bwd_rows_kernel<V><<<ctas, kRowThreads, smem, s>>>((const uint4*)dy, (const uint4*)x, (const uint4*)gamma, \
                                                            mean, rstd, (const uint4*)resid, (uint4*)dx, ws, rows,  \
                                                            nvec, 1.f / h, stages, nin);                            \
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
  if (!ok || cudaGetLastError() != cudaSuccess) return false;
  colsum_partials(ws, dgamma, dbeta, h, ctas, accumulate, s);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace mt
