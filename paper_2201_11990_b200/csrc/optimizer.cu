// Optimizer step after the DP gradient all-reduce: global gradient-norm
// clipping + AdamW with the MT-NLG recipe (reference TrainingRecipe, proj/include/curator/
// planner.hpp:39-53: beta = (0.9, 0.95), eps = 1e-8, clip 1.0, weight decay 0.1) and the
// reference's learning-rate schedule curator::lr_at (proj/src/planner.cpp:59-70).
//
// Mixed-precision state per parameter (reference model_state_bytes = 20 B/param):
// bf16 weight (2) + fp32 master weight (4) + fp32 gradient (4) + Adam m, v (4 + 4), i.e. 18 B here
// (the reference's extra 2 B bf16 gradient copy does not exist: wgrad GEMMs write fp32 directly).
//
// One fused HBM-bound kernel per layer: reads grad, m, v, master (16 B/param), writes m, v,
// master and the bf16 weight (14 B/param); the squared-norm reduction reads the grads once more.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "curator/planner.hpp"
#include "kernels.cuh"
#include "runtime.hpp"

namespace mt {
void set_error(const std::string& e);
namespace {

struct Segments {
  long long begin[MT_P_COUNT + 1];  // element offsets (param_off) and the end of the last slice
  long long count[MT_P_COUNT];
  int decay[MT_P_COUNT];
  int replicated[MT_P_COUNT];
};

// Sum of squares of one parameter slice (float4 loads) into *out (TP-sharded or replicated slot).
__global__ void grad_sq_kernel(const float4* __restrict__ g, long long n4, float* __restrict__ out) {
  float acc = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = g[i];
    acc += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    float a = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) atomicAdd(out, a);
  }
}

struct AdamScalars {
  float lr, beta1, beta2, eps, weight_decay;
  float bc1, bc2;  // 1 - beta^t
};

// One launch per parameter slice (slices are 128-byte aligned, lengths multiples of 4): float4 /
// 8-byte bf16x4 vector accesses, no per-element segment lookup. clip_coef is read from device
// memory (computed from the all-reduced norm), so the step never synchronises with the host.
__global__ void adamw_kernel(const float4* __restrict__ g, float4* __restrict__ m, float4* __restrict__ v,
                             float4* __restrict__ master, uint2* __restrict__ w, long long n4, AdamScalars a, int decay,
                             const float* __restrict__ clip_coef) {
  const float cc = *clip_coef;
  const float wd = decay ? a.lr * a.weight_decay : 0.f;
  const float inv_bc1 = 1.f / a.bc1, inv_bc2 = 1.f / a.bc2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 g4 = g[i];
    float4 m4 = m[i], v4 = v[i], p4 = master[i];
    float* gp = (float*)&g4;
    float* mp = (float*)&m4;
    float* vp = (float*)&v4;
    float* pp = (float*)&p4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gi = gp[j] * cc;
      mp[j] = a.beta1 * mp[j] + (1.f - a.beta1) * gi;
      vp[j] = a.beta2 * vp[j] + (1.f - a.beta2) * gi * gi;
      const float upd = (mp[j] * inv_bc1) / (sqrtf(vp[j] * inv_bc2) + a.eps);
      pp[j] = pp[j] - wd * pp[j] - a.lr * upd;
    }
    m[i] = m4;
    v[i] = v4;
    master[i] = p4;
    __nv_bfloat162 lo = __floats2bfloat162_rn(p4.x, p4.y), hi = __floats2bfloat162_rn(p4.z, p4.w);
    w[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ w, float* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __bfloat162float(w[i]);
}

// norm = sqrt(sum); coef = min(1, max_norm / (norm + 1e-6)); out = {norm, coef}
__global__ void clip_coef_kernel(const float* __restrict__ sq, float max_norm, float* __restrict__ out) {
  const float norm = sqrtf(sq[0] + sq[1]);
  out[0] = norm;
  out[1] = (max_norm > 0.f) ? fminf(1.f, max_norm / (norm + 1e-6f)) : 1.f;
}

Segments segments_of(const mt_layer* l) {
  Segments sg{};
  for (int p = 0; p < MT_P_COUNT; ++p) {
    sg.begin[p] = l->param_off[p];
    sg.count[p] = l->param_rows[p] * l->param_cols[p];
    // decoupled weight decay on the four weight matrices only (not biases / LayerNorm)
    sg.decay[p] = (p == MT_P_QKV_W || p == MT_P_PROJ_W || p == MT_P_FC1_W || p == MT_P_FC2_W) ? 1 : 0;
    sg.replicated[p] = (p == MT_P_LN1_GAMMA || p == MT_P_LN1_BETA || p == MT_P_LN2_GAMMA || p == MT_P_LN2_BETA ||
                        p == MT_P_PROJ_B || p == MT_P_FC2_B)
                           ? 1
                           : 0;
  }
  sg.begin[MT_P_COUNT] = l->param_total;
  return sg;
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g > 148 * 8 ? 148 * 8 : (g < 1 ? 1 : g));
}

}  // namespace

// Lazily creates the fp32 master copy (from the current bf16 weights) and zeroed Adam moments.
void ensure_optimizer_state(mt_layer* l, cudaStream_t s) {
  if (l->opt_master.ptr) return;
  const size_t n = static_cast<size_t>(l->param_total);
  l->opt_master.ensure(n * 4);
  l->opt_m.ensure(n * 4);
  l->opt_v.ensure(n * 4);
  check_cuda(cudaMemsetAsync(l->opt_m.ptr, 0, n * 4, s), "memset m");
  check_cuda(cudaMemsetAsync(l->opt_v.ptr, 0, n * 4, s), "memset v");
  bf16_to_f32_kernel<<<grid_for((long long)n), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(l->params.ptr),
                                                            l->opt_master.as<float>(), (long long)n);
  check_cuda(cudaGetLastError(), "bf16_to_f32");
}

// Adds this layer's squared gradient norm into sq[0] (TP-sharded params) and sq[1] (replicated).
void layer_grad_sq(mt_layer* l, float* sq, cudaStream_t s) {
  const Segments sg = segments_of(l);
  for (int p = 0; p < MT_P_COUNT; ++p) {
    const long long n4 = sg.count[p] / 4;
    grad_sq_kernel<<<grid_for(n4), 256, 0, s>>>(reinterpret_cast<const float4*>(l->grads.as<float>() + sg.begin[p]),
                                                n4, sq + (sg.replicated[p] ? 1 : 0));
  }
  check_cuda(cudaGetLastError(), "grad_sq");
}

void layer_adamw(mt_layer* l, const mt_adam_desc& d, float lr, const float* clip, cudaStream_t s) {
  ensure_optimizer_state(l, s);
  AdamScalars a;
  a.lr = lr;
  a.beta1 = d.beta1;
  a.beta2 = d.beta2;
  a.eps = d.eps;
  a.weight_decay = d.weight_decay;
  a.bc1 = 1.f - std::pow(d.beta1, (float)d.step);
  a.bc2 = 1.f - std::pow(d.beta2, (float)d.step);
  const Segments sg = segments_of(l);
  for (int p = 0; p < MT_P_COUNT; ++p) {
    const long long off = sg.begin[p], n4 = sg.count[p] / 4;
    adamw_kernel<<<grid_for(n4), 256, 0, s>>>(
        reinterpret_cast<const float4*>(l->grads.as<float>() + off), reinterpret_cast<float4*>(l->opt_m.as<float>() + off),
        reinterpret_cast<float4*>(l->opt_v.as<float>() + off), reinterpret_cast<float4*>(l->opt_master.as<float>() + off),
        reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(l->params.ptr) + off), n4, a, sg.decay[p], clip);
  }
  check_cuda(cudaGetLastError(), "adamw");
}

// Generic parameter slices (used by the vocab module): n must be a multiple of 4.
void grad_sq_segment(const float* g, int64_t n, float* out, cudaStream_t s) {
  grad_sq_kernel<<<grid_for(n / 4), 256, 0, s>>>(reinterpret_cast<const float4*>(g), n / 4, out);
  check_cuda(cudaGetLastError(), "grad_sq");
}

void adamw_segment(const float* g, float* m, float* v, float* master, void* w_bf16, int64_t n, const mt_adam_desc& d,
                   float lr, int decay, const float* clip, cudaStream_t s) {
  AdamScalars a;
  a.lr = lr;
  a.beta1 = d.beta1;
  a.beta2 = d.beta2;
  a.eps = d.eps;
  a.weight_decay = d.weight_decay;
  a.bc1 = 1.f - std::pow(d.beta1, (float)d.step);
  a.bc2 = 1.f - std::pow(d.beta2, (float)d.step);
  adamw_kernel<<<grid_for(n / 4), 256, 0, s>>>(reinterpret_cast<const float4*>(g), reinterpret_cast<float4*>(m),
                                               reinterpret_cast<float4*>(v), reinterpret_cast<float4*>(master),
                                               reinterpret_cast<uint2*>(w_bf16), n / 4, a, decay, clip);
  check_cuda(cudaGetLastError(), "adamw");
}

void bf16_to_f32(const void* w, float* out, int64_t n, cudaStream_t s) {
  bf16_to_f32_kernel<<<grid_for(n), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(w), out, n);
  check_cuda(cudaGetLastError(), "bf16_to_f32");
}

void clip_coefficient(const float* sq, float max_norm, float* out, cudaStream_t s) {
  clip_coef_kernel<<<1, 1, 0, s>>>(sq, max_norm, out);
  check_cuda(cudaGetLastError(), "clip_coef");
}

}  // namespace mt
