// Vocab-parallel embedding, tied LM head and vocab-parallel cross-entropy —
// the first- and last-stage work of the MT-NLG model around the transformer layers (GPT-2 decoder,
// PAPER.md:346-347; vocab V = 50257, reference ModelShape::vocab, planner.hpp:15).
//
// Layout (Megatron vocab parallelism): the word-embedding table is padded to a multiple of 128 * TP
// rows and rank r owns rows [r*Vp, (r+1)*Vp). Position embeddings and the final LayerNorm are
// replicated. The LM head is tied to the word embeddings: logits_r = LN_f(y) E_r^T (fp32, this
// rank's vocab slice), and the cross-entropy is computed without gathering the logits:
// row max (all-reduce MAX) -> sum of exp and the target logit (all-reduce SUM) -> loss and the
// logit gradient (softmax - onehot) / tokens, entirely on the vocab slice.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <string>

#include "curator/dropout.hpp"
#include "kernels.cuh"
#include "runtime.hpp"

namespace mt {
void set_error(const std::string& e);
}  // namespace mt

struct mt_vocab {
  mt_ctx* ctx = nullptr;
  mt_vocab_desc d{};
  uint64_t step = 0;  // training step keying the embedding-dropout masks (curator::step_seed)
  float loss_scale = 1.f;  // multiplies the head's loss and dlogits (the stage sets 1 / microbatches)
  int64_t vpad = 0, vp = 0, v0 = 0, M = 0, h = 0;
  mt::DeviceBuffer word, pos, lnf_g, lnf_b;        // bf16 params (word: [vp, h])
  mt::DeviceBuffer g_word, g_pos, g_lnf_g, g_lnf_b; // fp32 grads
  mt::DeviceBuffer logits;                          // fp32 [M, vp]
  mt::DeviceBuffer dlogits;                         // bf16 [M, vp]
  mt::DeviceBuffer yn, stats, rowbuf, dyn, ws;      // LN_f out, mean/rstd, per-row CE scalars, dLN_f out
  // optimizer state (fp32 master, Adam m, v) per parameter, created on the first optimizer step
  mt::DeviceBuffer opt_master[4], opt_m[4], opt_v[4];
  mt::DeviceBuffer* param(int i) { return i == 0 ? &word : i == 1 ? &pos : i == 2 ? &lnf_g : &lnf_b; }
  mt::DeviceBuffer* grad(int i) { return i == 0 ? &g_word : i == 1 ? &g_pos : i == 2 ? &g_lnf_g : &g_lnf_b; }
  int64_t count(int i) const { return i == 0 ? vp * h : i == 1 ? int64_t{d.seq} * h : h; }
};

namespace {

using mt::check_cuda;
using mt::check_nccl;

template <class F>
int call(F&& f) {
  try {
    f();
    return MT_OK;
  } catch (const std::invalid_argument& e) {
    mt::set_error(e.what());
    return MT_ERR_CONFIG;
  } catch (const std::exception& e) {
    mt::set_error(e.what());
    return MT_ERR_DATA;
  }
}

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// x[row] = E[tok - v0] if the token is in this rank's slice, else 0   (8 bf16 per thread)
__global__ void embed_gather_kernel(const int32_t* __restrict__ tokens, const uint4* __restrict__ word,
                                    uint4* __restrict__ out, int nvec_row, long long v0, long long vp) {
  const int row = blockIdx.y;
  const int cv = blockIdx.x * blockDim.x + threadIdx.x;
  if (cv >= nvec_row) return;
  const long long t = (long long)tokens[row] - v0;
  out[(size_t)row * nvec_row + cv] = (t >= 0 && t < vp) ? word[t * nvec_row + cv] : make_uint4(0, 0, 0, 0);
}

// x = dropout(x + P[pos]) in place (pos = row % seq)
__global__ void embed_pos_dropout_kernel(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ pos, int h,
                                         int seq, uint64_t seed, uint32_t th, float scale) {
  const int row = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  const size_t i = (size_t)row * h + c;
  const float v = bf(x[i]) + bf(pos[(size_t)(row % seq) * h + c]);
  x[i] = __float2bfloat16_rn(curator::dropout_keep(seed, i, th) ? v * scale : 0.f);
}

// embedding backward: g = dropout'(dx); dP[pos] += g; dE[tok - v0] += g for in-slice tokens
__global__ void embed_backward_kernel(const int32_t* __restrict__ tokens, const __nv_bfloat16* __restrict__ dx,
                                      float* __restrict__ g_word, float* __restrict__ g_pos, int h, int seq,
                                      long long v0, long long vp, uint64_t seed, uint32_t th, float scale) {
  const int row = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  const size_t i = (size_t)row * h + c;
  const float g = curator::dropout_keep(seed, i, th) ? bf(dx[i]) * scale : 0.f;
  atomicAdd(&g_pos[(size_t)(row % seq) * h + c], g);
  const long long t = (long long)tokens[row] - v0;
  if (t >= 0 && t < vp) atomicAdd(&g_word[t * h + c], g);
}

__device__ __forceinline__ float block_reduce(float v, float* red, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : (is_max ? -INFINITY : 0.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, t, o);
    t = is_max ? fmaxf(t, u) : t + u;
  }
  return t;
}

// pass A: rowbuf[row].x = local max over the valid vocab columns of this slice
__global__ void ce_max_kernel(const float* __restrict__ logits, long long vp, long long v0, long long vocab,
                              float* __restrict__ rowmax) {
  __shared__ float red[32];
  const int row = blockIdx.x;
  const float* l = logits + (size_t)row * vp;
  float m = -INFINITY;
  for (long long c = threadIdx.x; c < vp; c += blockDim.x)
    if (v0 + c < vocab) m = fmaxf(m, l[c]);
  m = block_reduce(m, red, true);
  if (threadIdx.x == 0) rowmax[row] = m;
}

// pass B: sums[2*row] = sum exp(l - gmax), sums[2*row+1] = target logit (0 if not in this slice)
__global__ void ce_sum_kernel(const float* __restrict__ logits, long long vp, long long v0, long long vocab,
                              const float* __restrict__ gmax, const int32_t* __restrict__ targets,
                              float* __restrict__ sums) {
  __shared__ float red[32];
  const int row = blockIdx.x;
  const float* l = logits + (size_t)row * vp;
  const float m = gmax[row];
  float s = 0.f;
  for (long long c = threadIdx.x; c < vp; c += blockDim.x)
    if (v0 + c < vocab) s += __expf(l[c] - m);
  s = block_reduce(s, red, false);
  if (threadIdx.x == 0) {
    sums[2 * row] = s;
    const long long t = (long long)targets[row] - v0;
    sums[2 * row + 1] = (t >= 0 && t < vp) ? l[t] : 0.f;
  }
}

// pass C: loss += (log(S) + gmax - target_logit) / M ; dlogits = (softmax - onehot) / M (bf16)
__global__ void ce_grad_kernel(const float* __restrict__ logits, long long vp, long long v0, long long vocab,
                               const float* __restrict__ gmax, const float* __restrict__ sums,
                               const int32_t* __restrict__ targets, __nv_bfloat16* __restrict__ dlogits,
                               float* __restrict__ loss, float inv_m) {
  const int row = blockIdx.x;
  const float m = gmax[row], S = sums[2 * row];
  const float inv_s = 1.f / S;
  const long long t = (long long)targets[row] - v0;
  const float* l = logits + (size_t)row * vp;
  __nv_bfloat16* g = dlogits + (size_t)row * vp;
  for (long long c = threadIdx.x; c < vp; c += blockDim.x) {
    float p = (v0 + c < vocab) ? __expf(l[c] - m) * inv_s : 0.f;
    if (c == t) p -= 1.f;
    g[c] = __float2bfloat16_rn(p * inv_m);
  }
  if (threadIdx.x == 0) atomicAdd(loss, (logf(S) + m - sums[2 * row + 1]) * inv_m);
}

__global__ void fill_f32(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

int64_t padded_vocab(int64_t vocab, int tp) {
  const int64_t q = 128 * int64_t{tp};
  return (vocab + q - 1) / q * q;
}

void gemm(const mt_gemm_args& a, cudaStream_t s) {
  const int rc = mt_gemm(&a, s);
  if (rc == 1) throw std::invalid_argument("mt_gemm: invalid arguments");
  if (rc != 0) throw mt::RuntimeFailure("mt_gemm failed");
}

mt_gemm_args gemm_args(const void* A, int64_t lda, bool amn, const void* B, int64_t ldb, bool bmn, void* D, int64_t ldd,
                       int64_t m, int64_t n, int64_t k, int epi) {
  mt_gemm_args a{};
  a.a = A;
  a.lda = lda;
  a.a_mn_major = amn;
  a.b = B;
  a.ldb = ldb;
  a.b_mn_major = bmn;
  a.d = D;
  a.ldd = ldd;
  a.m = m;
  a.n = n;
  a.k = k;
  a.batch = 1;
  a.alpha = 1.f;
  a.epilogue = epi;
  return a;
}

}  // namespace

extern "C" int mt_vocab_create(mt_ctx* c, const mt_vocab_desc* d, mt_vocab** out) {
  return call([&] {
    if (!c || !d || !out) throw std::invalid_argument("null argument");
    if (d->vocab <= 0 || d->hidden <= 0 || d->hidden % 64 || d->seq <= 0 || d->micro_batch <= 0)
      throw std::invalid_argument("bad vocab descriptor");
    if (d->tp_size < 1 || d->tp_rank < 0 || d->tp_rank >= d->tp_size) throw std::invalid_argument("bad TP rank");
    check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
    auto v = new mt_vocab();
    v->ctx = c;
    v->d = *d;
    v->vpad = padded_vocab(d->vocab, d->tp_size);
    v->vp = v->vpad / d->tp_size;
    v->v0 = v->vp * d->tp_rank;
    v->M = int64_t{d->micro_batch} * d->seq;
    v->h = d->hidden;
    const int64_t h = v->h, vp = v->vp, M = v->M;
    v->word.ensure(vp * h * 2);
    v->pos.ensure(int64_t{d->seq} * h * 2);
    v->lnf_g.ensure(h * 2);
    v->lnf_b.ensure(h * 2);
    v->g_word.ensure(vp * h * 4);
    v->g_pos.ensure(int64_t{d->seq} * h * 4);
    v->g_lnf_g.ensure(h * 4);
    v->g_lnf_b.ensure(h * 4);
    v->logits.ensure(M * vp * 4);
    v->dlogits.ensure(M * vp * 2);
    v->yn.ensure(M * h * 2);
    v->dyn.ensure(M * h * 2);
    v->stats.ensure(2 * M * 4);
    v->rowbuf.ensure(3 * M * 4);
    v->ws.ensure(mt::colsum_workspace_floats((int)M, (int)h) * 4);
    *out = v;
    check_cuda(cudaMemset(v->g_word.ptr, 0, vp * h * 4), "memset");
    check_cuda(cudaMemset(v->g_pos.ptr, 0, int64_t{d->seq} * h * 4), "memset");
    check_cuda(cudaMemset(v->g_lnf_g.ptr, 0, h * 4), "memset");
    check_cuda(cudaMemset(v->g_lnf_b.ptr, 0, h * 4), "memset");
  });
}

extern "C" int mt_vocab_destroy(mt_vocab* v) {
  return call([&] { delete v; });
}

extern "C" int mt_vocab_padded(const mt_vocab* v, int64_t* vocab_padded, int64_t* slice_begin, int64_t* slice_rows) {
  return call([&] {
    *vocab_padded = v->vpad;
    *slice_begin = v->v0;
    *slice_rows = v->vp;
  });
}

// param: 0 word [vpad, h] (global, this rank's rows copied), 1 pos [seq, h], 2 lnf gamma [h], 3 lnf beta [h]
extern "C" int mt_vocab_set_param(mt_vocab* v, int32_t param, const void* host_global_bf16) {
  return call([&] {
    const uint16_t* src = static_cast<const uint16_t*>(host_global_bf16);
    switch (param) {
      case 0:
        check_cuda(cudaMemcpy(v->word.ptr, src + v->v0 * v->h, v->vp * v->h * 2, cudaMemcpyHostToDevice), "H2D");
        break;
      case 1:
        check_cuda(cudaMemcpy(v->pos.ptr, src, int64_t{v->d.seq} * v->h * 2, cudaMemcpyHostToDevice), "H2D");
        break;
      case 2:
        check_cuda(cudaMemcpy(v->lnf_g.ptr, src, v->h * 2, cudaMemcpyHostToDevice), "H2D");
        break;
      case 3:
        check_cuda(cudaMemcpy(v->lnf_b.ptr, src, v->h * 2, cudaMemcpyHostToDevice), "H2D");
        break;
      default:
        throw std::invalid_argument("unknown vocab parameter");
    }
  });
}

extern "C" int mt_vocab_get_param(mt_vocab* v, int32_t param, void* host) {
  return call([&] {
    if (param < 0 || param > 3) throw std::invalid_argument("unknown vocab parameter");
    check_cuda(cudaDeviceSynchronize(), "sync");
    check_cuda(cudaMemcpy(host, v->param(param)->ptr, v->count(param) * 2, cudaMemcpyDeviceToHost), "D2H");
  });
}

extern "C" int mt_vocab_get_grad(mt_vocab* v, int32_t param, float* host) {
  return call([&] {
    check_cuda(cudaDeviceSynchronize(), "sync");
    const mt::DeviceBuffer* b = param == 0 ? &v->g_word : param == 1 ? &v->g_pos : param == 2 ? &v->g_lnf_g
                                : param == 3                         ? &v->g_lnf_b
                                                                     : nullptr;
    if (!b) throw std::invalid_argument("unknown vocab parameter");
    const int64_t n = param == 0 ? v->vp * v->h : param == 1 ? int64_t{v->d.seq} * v->h : v->h;
    check_cuda(cudaMemcpy(host, b->ptr, n * 4, cudaMemcpyDeviceToHost), "D2H");
  });
}

namespace mt {
int64_t vocab_tokens(const mt_vocab* v) { return v->M; }
int64_t vocab_hidden(const mt_vocab* v) { return v->h; }
int vocab_tp(const mt_vocab* v) { return v->d.tp_size; }

void vocab_zero_grads(mt_vocab* v, cudaStream_t s) {
  for (int i = 0; i < 4; ++i) check_cuda(cudaMemsetAsync(v->grad(i)->ptr, 0, v->count(i) * 4, s), "memset");
}

void vocab_grad_sq(mt_vocab* v, bool count_word, float* sq, cudaStream_t s) {
  if (count_word) grad_sq_segment(v->g_word.as<float>(), v->count(0), sq, s);  // vocab-sharded
  for (int i = 1; i < 4; ++i) grad_sq_segment(v->grad(i)->as<float>(), v->count(i), sq + 1, s);  // replicated
}

// AdamW on the four vocab parameters; weight decay on the embeddings, not on LN_f (Megatron).
void vocab_adamw(mt_vocab* v, const mt_adam_desc& d, float lr, const float* clip, cudaStream_t s) {
  for (int i = 0; i < 4; ++i) {
    const int64_t n = v->count(i);
    if (!v->opt_master[i].ptr) {
      v->opt_master[i].ensure(n * 4);
      v->opt_m[i].ensure(n * 4);
      v->opt_v[i].ensure(n * 4);
      check_cuda(cudaMemsetAsync(v->opt_m[i].ptr, 0, n * 4, s), "memset m");
      check_cuda(cudaMemsetAsync(v->opt_v[i].ptr, 0, n * 4, s), "memset v");
      bf16_to_f32(v->param(i)->ptr, v->opt_master[i].as<float>(), n, s);
    }
    adamw_segment(v->grad(i)->as<float>(), v->opt_m[i].as<float>(), v->opt_v[i].as<float>(),
                  v->opt_master[i].as<float>(), v->param(i)->ptr, n, d, lr, i < 2 ? 1 : 0, clip, s);
  }
}

void vocab_allreduce_grads(mt_vocab* v, ncclComm_t comm, bool word_only, bool average, cudaStream_t s) {
  check_nccl(ncclGroupStart(), "group");
  for (int i = 0; i < (word_only ? 1 : 4); ++i)
    check_nccl(ncclAllReduce(v->grad(i)->ptr, v->grad(i)->ptr, v->count(i), ncclFloat32, average ? ncclAvg : ncclSum,
                             comm, s),
               "ncclAllReduce(vocab grads)");
  check_nccl(ncclGroupEnd(), "group");
}
}  // namespace mt

extern "C" int mt_vocab_set_step(mt_vocab* v, uint64_t step) {
  return call([&] {
    if (!v) throw std::invalid_argument("null vocab");
    v->step = step;
  });
}

extern "C" int mt_vocab_set_loss_scale(mt_vocab* v, float scale) {
  return call([&] {
    if (!v || !(scale > 0.f)) throw std::invalid_argument("bad loss scale");
    v->loss_scale = scale;
  });
}

extern "C" int mt_vocab_zero_grads(mt_vocab* v, void* stream) {
  return call([&] { mt::vocab_zero_grads(v, (cudaStream_t)stream); });
}

static bool tp_active(const mt_vocab* v) { return v->d.tp_size > 1 && v->ctx->tp; }

extern "C" int mt_vocab_embed_forward(mt_vocab* v, const int32_t* tokens, void* x, uint32_t mb, void* stream) {
  return call([&] {
    cudaStream_t s = (cudaStream_t)stream;
    const int h = (int)v->h, M = (int)v->M;
    embed_gather_kernel<<<dim3((h / 8 + 127) / 128, M), 128, 0, s>>>(tokens, (const uint4*)v->word.ptr, (uint4*)x, h / 8,
                                                                     v->v0, v->vp);
    if (tp_active(v))
      check_nccl(ncclAllReduce(x, x, int64_t{M} * h, ncclBfloat16, ncclSum, v->ctx->tp, s), "ncclAllReduce(embed)");
    const uint64_t site = curator::site_seed(curator::step_seed(v->d.seed, v->step), "embed.dropout", 0, mb);
    embed_pos_dropout_kernel<<<dim3((h + 255) / 256, M), 256, 0, s>>>(
        (__nv_bfloat16*)x, (const __nv_bfloat16*)v->pos.ptr, h, v->d.seq, site,
        curator::dropout_threshold16(v->d.dropout), 1.f / (1.f - v->d.dropout));
    check_cuda(cudaGetLastError(), "embed forward");
  });
}

extern "C" int mt_vocab_embed_backward(mt_vocab* v, const int32_t* tokens, const void* dx, uint32_t mb,
                                       void* stream) {
  return call([&] {
    cudaStream_t s = (cudaStream_t)stream;
    const int h = (int)v->h, M = (int)v->M;
    const uint64_t site = curator::site_seed(curator::step_seed(v->d.seed, v->step), "embed.dropout", 0, mb);
    embed_backward_kernel<<<dim3((h + 255) / 256, M), 256, 0, s>>>(
        tokens, (const __nv_bfloat16*)dx, v->g_word.as<float>(), v->g_pos.as<float>(), h, v->d.seq, v->v0, v->vp, site,
        curator::dropout_threshold16(v->d.dropout), 1.f / (1.f - v->d.dropout));
    check_cuda(cudaGetLastError(), "embed backward");
  });
}

// Final LayerNorm + tied LM head + vocab-parallel cross-entropy, forward and backward fused:
// loss_dev += mean token loss of the microbatch; dy (device bf16 [M, h]) = d loss / d y.
extern "C" int mt_vocab_head_loss(mt_vocab* v, const void* y, const int32_t* targets, void* dy, float* loss_dev,
                                  void* stream) {
  return call([&] {
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t h = v->h, M = v->M, vp = v->vp;
    float* mean = v->stats.as<float>();
    float* rstd = mean + M;
    mt::ln_fwd(y, v->lnf_g.ptr, v->lnf_b.ptr, v->yn.ptr, mean, rstd, (int)M, (int)h, v->d.ln_eps, s);
    // logits (fp32) = LN_f(y) E_slice^T
    gemm(gemm_args(v->yn.ptr, h, false, v->word.ptr, h, false, v->logits.ptr, vp, M, vp, h, MT_EPI_STORE_F32), s);
    float* rmax = v->rowbuf.as<float>();
    float* sums = rmax + M;
    ce_max_kernel<<<(int)M, 256, 0, s>>>(v->logits.as<float>(), vp, v->v0, v->d.vocab, rmax);
    if (tp_active(v)) check_nccl(ncclAllReduce(rmax, rmax, M, ncclFloat32, ncclMax, v->ctx->tp, s), "AR max");
    ce_sum_kernel<<<(int)M, 256, 0, s>>>(v->logits.as<float>(), vp, v->v0, v->d.vocab, rmax, targets, sums);
    if (tp_active(v)) check_nccl(ncclAllReduce(sums, sums, 2 * M, ncclFloat32, ncclSum, v->ctx->tp, s), "AR sum");
    ce_grad_kernel<<<(int)M, 256, 0, s>>>(v->logits.as<float>(), vp, v->v0, v->d.vocab, rmax, sums, targets,
                                          (__nv_bfloat16*)v->dlogits.ptr, loss_dev, v->loss_scale / (float)M);
    // d LN_f(y) = dlogits E_slice (partial over the vocab slices) -> all-reduce
    gemm(gemm_args(v->dlogits.ptr, vp, false, v->word.ptr, h, true, v->dyn.ptr, h, M, h, vp, MT_EPI_STORE_BF16), s);
    if (tp_active(v))
      check_nccl(ncclAllReduce(v->dyn.ptr, v->dyn.ptr, M * h, ncclBfloat16, ncclSum, v->ctx->tp, s), "AR dLNf");
    // tied-embedding gradient: dE_slice += dlogits^T LN_f(y)
    gemm(gemm_args(v->dlogits.ptr, vp, true, v->yn.ptr, h, true, v->g_word.ptr, h, vp, h, M, MT_EPI_ACCUM_F32), s);
    // one pass over dLN_f and y (dy may overwrite y in place: the stage driver does that)
    mt::ln_bwd(v->dyn.ptr, y, v->lnf_g.ptr, mean, rstd, nullptr, dy, v->g_lnf_g.as<float>(), v->g_lnf_b.as<float>(),
               (int)M, (int)h, v->ws.as<float>(), true, s);
    check_cuda(cudaGetLastError(), "head loss");
  });
}
