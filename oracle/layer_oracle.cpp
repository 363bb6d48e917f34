// ORACLE — test infrastructure only. Never linked into or called by the product path
// (paper_2201_11990_b200/); only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load it, as the checker and the CPU baseline.
//
// CPU restatement (fp32, OpenMP) of one tensor-sliced GPT transformer layer, forward and backward,
// exactly as the GPU runtime executes it. The reference (arxiv/paper_2201_11990) has NO
// implementation of this path ("OUT OF SCOPE — actual neural-network training"), so this
// follows the paper text:
//   * Megatron tensor slicing, column-parallel QKV / fc1, row-parallel attn-out / fc2, all-reduce
//     after the row-parallel GEMMs ("g") and on the LN-input gradients ("f"): PAPER.md:133-150;
//   * GPT-2 pre-LN decoder block, causal self-attention, GeLU MLP (4h): PAPER.md:346-347;
//   * init std sqrt(1/(3h)): PAPER.md:348,351 = reference proj/src/planner.cpp:34-37;
//   * mixed precision (bf16 storage, fp32 accumulation): PAPER.md:55-70, 257;
//   * seeded streams from the reference's hashing primitives (proj/include/curator/hashing.hpp:45-63)
//     via include/curator/dropout.hpp.
// PARITY UNPINNED by the reference: no golden vectors for the layer exist upstream.
// It is self-pinned instead: TP=t == TP=1 (tests/test_oracle.py), a torch autograd cross-check of
// forward and backward (tests/test_oracle.py), and the GPU kernels against it (tests/test_layer_gpu.py).
//
// Modes: bf16_emulate = 1 rounds to bf16 at every point the GPU stores a bf16 tensor (GEMM
// epilogues, softmax output, LayerNorm output, residual stream, TP all-reduce result), so GPU vs
// oracle differences reduce to fp32 summation order; bf16_emulate = 0 keeps everything fp32.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "curator/dropout.hpp"

namespace {

using Vec = std::vector<float>;

inline float bf16_round(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f;  // inf / nan unchanged
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

struct Ctx {
  bool emu = false;
  void round(float* p, size_t n) const {
    if (!emu) return;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) p[i] = bf16_round(p[i]);
  }
  void round(Vec& v) const { round(v.data(), v.size()); }
};

// Packed, register-blocked fp32 GEMM (Goto-style): C[m][n] (+)= sum_q A(m,q) B(q,n) with
//   A(m,q) = a_t ? A[q*lda + m] : A[m*lda + q],   B(q,n) = b_t ? B[n*ldb + q] : B[q*ldb + n].
// A is packed once into 6-row slivers, B per 16-column panel and 256-deep k-block; the 6x16
// micro-kernel keeps its accumulators in vector registers. OpenMP over column panels.
constexpr int kMR = 6, kNR = 16, kKC = 256;

void micro_kernel_scalar(const float* __restrict__ ap, const float* __restrict__ bp, int kc, float* __restrict__ out) {
  float acc[kMR][kNR] = {};
  for (int q = 0; q < kc; ++q)
    for (int r = 0; r < kMR; ++r)
      for (int j = 0; j < kNR; ++j) acc[r][j] += ap[q * kMR + r] * bp[q * kNR + j];
  for (int r = 0; r < kMR; ++r)
    for (int j = 0; j < kNR; ++j) out[r * kNR + j] = acc[r][j];
}

typedef float v8 __attribute__((vector_size(32), aligned(4)));

// 6x16 block, 12 ymm accumulators, one broadcast + two FMAs per (row, k).
__attribute__((target("avx2,fma"))) void micro_kernel_avx2(const float* __restrict__ ap, const float* __restrict__ bp,
                                                           int kc, float* __restrict__ out) {
  v8 c0a = {}, c0b = {}, c1a = {}, c1b = {}, c2a = {}, c2b = {}, c3a = {}, c3b = {}, c4a = {}, c4b = {}, c5a = {},
     c5b = {};
  for (int q = 0; q < kc; ++q) {
    const v8 b0 = *reinterpret_cast<const v8*>(bp + q * kNR);
    const v8 b1 = *reinterpret_cast<const v8*>(bp + q * kNR + 8);
    const float* a = ap + q * kMR;
#define MT_ROW(R, CA, CB)      \
  {                            \
    const float av = a[R];     \
    const v8 vv = {av, av, av, av, av, av, av, av}; \
    CA += vv * b0;             \
    CB += vv * b1;             \
  }
    MT_ROW(0, c0a, c0b) MT_ROW(1, c1a, c1b) MT_ROW(2, c2a, c2b) MT_ROW(3, c3a, c3b) MT_ROW(4, c4a, c4b)
    MT_ROW(5, c5a, c5b)
#undef MT_ROW
  }
  const v8* rows[kMR][2] = {{&c0a, &c0b}, {&c1a, &c1b}, {&c2a, &c2b}, {&c3a, &c3b}, {&c4a, &c4b}, {&c5a, &c5b}};
  for (int r = 0; r < kMR; ++r) {
    *reinterpret_cast<v8*>(out + r * kNR) = *rows[r][0];
    *reinterpret_cast<v8*>(out + r * kNR + 8) = *rows[r][1];
  }
}

void micro_kernel(const float* __restrict__ ap, const float* __restrict__ bp, int kc, float* __restrict__ out) {
  static const bool avx2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
  if (avx2)
    micro_kernel_avx2(ap, bp, kc, out);
  else
    micro_kernel_scalar(ap, bp, kc, out);
}

void gemm(bool a_t, bool b_t, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
          int64_t ldb, float* C, int64_t ldc, bool accumulate) {
  const int64_t mb = (m + kMR - 1) / kMR, nb = (n + kNR - 1) / kNR;
  // pack A: Ap[ib][q][r]
  std::vector<float> Ap(static_cast<size_t>(mb * k * kMR));
#pragma omp parallel for schedule(static)
  for (int64_t ib = 0; ib < mb; ++ib)
    for (int64_t q = 0; q < k; ++q)
      for (int r = 0; r < kMR; ++r) {
        const int64_t i = ib * kMR + r;
        Ap[(ib * k + q) * kMR + r] = i < m ? (a_t ? A[q * lda + i] : A[i * lda + q]) : 0.f;
      }
#pragma omp parallel
  {
    std::vector<float> Bp(static_cast<size_t>(kKC) * kNR);
    float blk[kMR * kNR];
#pragma omp for schedule(dynamic)
    for (int64_t jb = 0; jb < nb; ++jb) {
      const int64_t j0 = jb * kNR, nj = std::min<int64_t>(kNR, n - j0);
      for (int64_t q0 = 0; q0 < k; q0 += kKC) {
        const int kc = static_cast<int>(std::min<int64_t>(kKC, k - q0));
        for (int q = 0; q < kc; ++q)
          for (int j = 0; j < kNR; ++j)
            Bp[q * kNR + j] = j < nj ? (b_t ? B[(j0 + j) * ldb + q0 + q] : B[(q0 + q) * ldb + j0 + j]) : 0.f;
        const bool first = q0 == 0 && !accumulate;
        for (int64_t ib = 0; ib < mb; ++ib) {
          micro_kernel(&Ap[(ib * k + q0) * kMR], Bp.data(), kc, blk);
          const int64_t i0 = ib * kMR, ni = std::min<int64_t>(kMR, m - i0);
          for (int64_t r = 0; r < ni; ++r)
            for (int64_t j = 0; j < nj; ++j) {
              float& c = C[(i0 + r) * ldc + j0 + j];
              c = first ? blk[r * kNR + j] : c + blk[r * kNR + j];
            }
        }
      }
    }
  }
}

// C[m][n] = sum_k A[m*lda + k] * B[n*ldb + k]
void gemm_nt(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int64_t m, int64_t n,
             int64_t k) {
  gemm(false, true, m, n, k, A, lda, B, ldb, C, ldc, false);
}

float gelu(float x) { return 0.5f * x * (1.f + std::tanh(0.7978845608028654f * x * (1.f + 0.044715f * x * x))); }
float gelu_grad(float x) {
  const float t = std::tanh(0.7978845608028654f * x * (1.f + 0.044715f * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * 0.7978845608028654f * (1.f + 3.f * 0.044715f * x * x);
}

}  // namespace

extern "C" {

typedef struct or_layer_desc {
  int32_t hidden, heads, seq, micro_batch, tp_size, ffn_mult;
  float dropout_hidden, dropout_attn, ln_eps;
  uint64_t seed;
  uint32_t layer_index;
  int32_t bf16_emulate;
  // -1: the whole layer (all TP shards, the row-parallel partials summed = the TP all-reduce);
  // r >= 0: only TP shard r with no all-reduce, which is what one GPU computes in the runtime's
  // shard-only measurement mode (mt_ctx_shard_only; bench.py --shard-of t)
  int32_t shard_rank;
} or_layer_desc;

// Parameter order and global shapes as in include/mtnlg.h (enum mt_param).
struct or_layer {
  or_layer_desc d;
  Ctx cx;
  std::vector<const float*> p;  // 12 global parameters (caller-owned, non-owning views)
  struct Saved {
    Vec x, ln1, mean1, rstd1, qkv, S, P, lse, ctx, x1, ln2, mean2, rstd2, pre, act;
  };
  std::map<uint32_t, Saved> saved;
};

enum { P_LN1G, P_LN1B, P_QKVW, P_QKVB, P_PROJW, P_PROJB, P_LN2G, P_LN2B, P_FC1W, P_FC1B, P_FC2W, P_FC2B, P_N };

void or_param_shape(const or_layer_desc* d, int p, int64_t* rows, int64_t* cols) {
  const int64_t h = d->hidden, ff = int64_t{d->ffn_mult} * h;
  const int64_t shapes[P_N][2] = {{1, h},  {1, h}, {3 * h, h}, {1, 3 * h}, {h, h},  {1, h},
                                  {1, h},  {1, h}, {ff, h},    {1, ff},    {h, ff}, {1, h}};
  *rows = shapes[p][0];
  *cols = shapes[p][1];
}

or_layer* or_layer_create(const or_layer_desc* d, const float* const* params) {
  auto* l = new or_layer();
  l->d = *d;
  l->cx.emu = d->bf16_emulate != 0;
  for (int i = 0; i < P_N; ++i) {
    l->p.push_back(params[i]);
  }
  return l;
}

void or_layer_destroy(or_layer* l) { delete l; }

int or_num_threads(void) { return omp_get_max_threads(); }

}  // extern "C"

namespace {

// s0 / ns: the TP shards computed ([s0, s0 + ns)); the column-parallel widths of that range are
// Hc heads (global head index head0 + local head), cw = ns * h/t context columns, fw = ns * ff/t.
struct Dims {
  int64_t b, s, h, H, hd, M, ff, t, Hl, hl, ffl;
  int64_t s0, ns, Hc, head0, cw, fw;
};
Dims dims(const or_layer_desc& d) {
  Dims x;
  x.b = d.micro_batch;
  x.s = d.seq;
  x.h = d.hidden;
  x.H = d.heads;
  x.hd = x.h / x.H;
  x.M = x.b * x.s;
  x.ff = int64_t{d.ffn_mult} * x.h;
  x.t = d.tp_size;
  x.Hl = x.H / x.t;
  x.hl = x.h / x.t;
  x.ffl = x.ff / x.t;
  x.s0 = d.shard_rank >= 0 ? d.shard_rank : 0;
  x.ns = d.shard_rank >= 0 ? 1 : x.t;
  x.Hc = x.ns * x.Hl;
  x.head0 = x.s0 * x.Hl;
  x.cw = x.ns * x.hl;
  x.fw = x.ns * x.ffl;
  return x;
}

void layer_norm(const Ctx& cx, const Vec& x, const float* g, const float* be, Vec& y, Vec& mean, Vec& rstd, int64_t M,
                int64_t h, float eps) {
  y.assign(M * h, 0.f);
  mean.assign(M, 0.f);
  rstd.assign(M, 0.f);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < M; ++r) {
    const float* xr = &x[r * h];
    double s = 0;
    for (int64_t c = 0; c < h; ++c) s += xr[c];
    const float mu = static_cast<float>(s / h);
    double v = 0;
    for (int64_t c = 0; c < h; ++c) v += double(xr[c] - mu) * (xr[c] - mu);
    const float rs = 1.f / std::sqrt(static_cast<float>(v / h) + eps);
    for (int64_t c = 0; c < h; ++c) y[r * h + c] = (xr[c] - mu) * rs * g[c] + be[c];
    mean[r] = mu;
    rstd[r] = rs;
  }
  cx.round(y);
}

// y = resid + dropout(z + bias)
void bias_dropout_residual(const Ctx& cx, const Vec& z, const float* bias, const Vec& resid, Vec& y, int64_t M, int64_t h,
                           uint64_t site, uint32_t th, float scale) {
  y.assign(M * h, 0.f);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M * h; ++i) {
    const bool keep = curator::dropout_keep(site, static_cast<uint64_t>(i), th);
    y[i] = resid[i] + (keep ? (z[i] + bias[i % h]) * scale : 0.f);
  }
  cx.round(y);
}

uint64_t site(const or_layer_desc& d, const char* name, uint32_t mb) {
  return curator::site_seed(d.seed, name, d.layer_index, mb);
}

}  // namespace

extern "C" void or_layer_forward(or_layer* l, const float* x_in, float* y_out, uint32_t mb) {
  const or_layer_desc& d = l->d;
  const Ctx& cx = l->cx;
  const Dims D = dims(d);
  auto& sv = l->saved[mb];
  sv.x.assign(x_in, x_in + D.M * D.h);
  const auto& P = l->p;
  const float scale_h = 1.f / (1.f - d.dropout_hidden), scale_a = 1.f / (1.f - d.dropout_attn);
  const uint32_t th_h = curator::dropout_threshold16(d.dropout_hidden), th_a = curator::dropout_threshold16(d.dropout_attn);
  const float alpha = 1.f / std::sqrt(static_cast<float>(D.hd));
  const int64_t ld3 = 3 * D.cw;  // QKV columns of the computed shards, (local head, {q,k,v}, hd) order

  layer_norm(cx, sv.x, P[P_LN1G], P[P_LN1B], sv.ln1, sv.mean1, sv.rstd1, D.M, D.h, d.ln_eps);
  // column-parallel QKV: the shards' outputs are contiguous row blocks of the global weight
  // (rows in (head, {q,k,v}, hd) order), so the computed shards are one GEMM.
  sv.qkv.assign(D.M * ld3, 0.f);
  gemm_nt(sv.ln1.data(), D.h, P[P_QKVW] + D.s0 * 3 * D.hl * D.h, D.h, sv.qkv.data(), ld3, D.M, ld3, D.h);
  const float* qkv_b = P[P_QKVB] + D.s0 * 3 * D.hl;
  for (int64_t r = 0; r < D.M; ++r)
    for (int64_t c = 0; c < ld3; ++c) sv.qkv[r * ld3 + c] += qkv_b[c];
  cx.round(sv.qkv);

  // causal attention per (microbatch row bb, head): S = alpha Q K^T and ctx = P V as packed GEMMs
  // (one head per thread), the softmax + dropout per row in between. Entries above the diagonal
  // are never read (S) or zero (P).
  const int64_t s = D.s, hd = D.hd;
  sv.S.assign(D.b * D.Hc * s * s, 0.f);
  sv.P.assign(D.b * D.Hc * s * s, 0.f);
  sv.lse.assign(D.b * D.Hc * s, 0.f);
  sv.ctx.assign(D.M * D.cw, 0.f);
  const uint64_t site_a = site(d, "attn.probs", mb);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t bb = 0; bb < D.b; ++bb) {
    for (int64_t hh = 0; hh < D.Hc; ++hh) {
      const float* q = &sv.qkv[bb * s * ld3 + hh * 3 * hd];
      const float* k = q + hd;
      const float* v = q + 2 * hd;
      float* S = &sv.S[(bb * D.Hc + hh) * s * s];
      float* Pm = &sv.P[(bb * D.Hc + hh) * s * s];
      gemm(false, true, s, s, hd, q, ld3, k, ld3, S, s, false);  // nested: runs on this thread
      const int64_t hg = D.head0 + hh;  // global head index (keys the attention-dropout stream)
      for (int64_t i = 0; i < s; ++i) {
        float mx = -INFINITY;
        for (int64_t j = 0; j <= i; ++j) {
          float acc = S[i * s + j] * alpha;
          if (cx.emu) acc = bf16_round(acc);
          S[i * s + j] = acc;
          mx = std::max(mx, acc);
        }
        for (int64_t j = i + 1; j < s; ++j) S[i * s + j] = 0.f;
        float sum = 0.f;
        for (int64_t j = 0; j <= i; ++j) sum += std::exp(S[i * s + j] - mx);
        const float lse = mx + std::log(sum);
        sv.lse[(bb * D.Hc + hh) * s + i] = lse;
        const uint64_t base = ((static_cast<uint64_t>(bb) * D.H + hg) * s + i) * static_cast<uint64_t>(s);
        for (int64_t j = 0; j <= i; ++j) {
          float pv = std::exp(S[i * s + j] - mx) / sum;
          pv = curator::dropout_keep(site_a, base + j, th_a) ? pv * scale_a : 0.f;
          Pm[i * s + j] = cx.emu ? bf16_round(pv) : pv;
        }
      }
      gemm(false, false, s, hd, s, Pm, s, v, ld3, &sv.ctx[bb * s * D.cw + hh * hd], D.cw, false);
    }
  }
  cx.round(sv.ctx);

  // row-parallel GEMM: per TP shard partial (rounded like the GPU epilogue), summed over the computed
  // shards (the all-reduce; a single shard in shard mode) and rounded
  auto row_parallel = [&](const Vec& in, int64_t in_cols, const float* W, int64_t w_cols, int64_t shard_cols, Vec& out) {
    out.assign(D.M * D.h, 0.f);
    Vec part(D.M * D.h);
    for (int64_t r = 0; r < D.ns; ++r) {
      // shard s0 + r: input columns [r*shard_cols, ...) of `in`, weight columns [(s0+r)*shard_cols, ...)
      gemm_nt(in.data() + r * shard_cols, in_cols, W + (D.s0 + r) * shard_cols, w_cols, part.data(), D.h, D.M, D.h,
              shard_cols);
      cx.round(part);
      for (int64_t i = 0; i < D.M * D.h; ++i) out[i] += part[i];
    }
    cx.round(out);
  };
  Vec z;
  row_parallel(sv.ctx, D.cw, P[P_PROJW], D.h, D.hl, z);
  bias_dropout_residual(cx, z, P[P_PROJB], sv.x, sv.x1, D.M, D.h, site(d, "attn.out", mb), th_h, scale_h);
  layer_norm(cx, sv.x1, P[P_LN2G], P[P_LN2B], sv.ln2, sv.mean2, sv.rstd2, D.M, D.h, d.ln_eps);
  sv.pre.assign(D.M * D.fw, 0.f);
  gemm_nt(sv.ln2.data(), D.h, P[P_FC1W] + D.s0 * D.ffl * D.h, D.h, sv.pre.data(), D.fw, D.M, D.fw, D.h);
  sv.act.assign(D.M * D.fw, 0.f);
  const float* fc1_b = P[P_FC1B] + D.s0 * D.ffl;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < D.M * D.fw; ++i) {
    float pr = sv.pre[i] + fc1_b[i % D.fw];
    if (cx.emu) pr = bf16_round(pr);
    sv.pre[i] = pr;
    const float a = gelu(pr);
    sv.act[i] = cx.emu ? bf16_round(a) : a;
  }
  Vec m;
  row_parallel(sv.act, D.fw, P[P_FC2W], D.ff, D.ffl, m);
  Vec y;
  bias_dropout_residual(cx, m, P[P_FC2B], sv.x1, y, D.M, D.h, site(d, "mlp.out", mb), th_h, scale_h);
  std::copy(y.begin(), y.end(), y_out);
}

namespace {

void colsum_acc(const Vec& x, int64_t M, int64_t n, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double s = 0;
    for (int64_t r = 0; r < M; ++r) s += x[r * n + c];
    out[c] += static_cast<float>(s);
  }
}

// LayerNorm backward: returns dx (+resid), accumulates dgamma, dbeta.
void ln_backward(const Ctx& cx, const Vec& dy, const Vec& x, const float* g, const Vec& mean, const Vec& rstd,
                 const Vec* resid, Vec& dx, float* dg, float* db, int64_t M, int64_t h) {
  dx.assign(M * h, 0.f);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < M; ++r) {
    double s1 = 0, s2 = 0;
    for (int64_t c = 0; c < h; ++c) {
      const float xh = (x[r * h + c] - mean[r]) * rstd[r];
      const float gg = dy[r * h + c] * g[c];
      s1 += gg;
      s2 += double(gg) * xh;
    }
    const float m1 = static_cast<float>(s1 / h), m2 = static_cast<float>(s2 / h);
    for (int64_t c = 0; c < h; ++c) {
      const float xh = (x[r * h + c] - mean[r]) * rstd[r];
      const float gg = dy[r * h + c] * g[c];
      dx[r * h + c] = rstd[r] * (gg - m1 - xh * m2) + (resid ? (*resid)[r * h + c] : 0.f);
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < h; ++c) {
    double sg = 0, sb = 0;
    for (int64_t r = 0; r < M; ++r) {
      const float xh = (x[r * h + c] - mean[r]) * rstd[r];
      sg += double(dy[r * h + c]) * xh;
      sb += dy[r * h + c];
    }
    dg[c] += static_cast<float>(sg);
    db[c] += static_cast<float>(sb);
  }
  cx.round(dx);
}

void dropout_bwd(const Ctx& cx, const Vec& dy, Vec& dz, int64_t n, uint64_t site_seed, uint32_t th, float scale) {
  dz.assign(n, 0.f);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) dz[i] = curator::dropout_keep(site_seed, static_cast<uint64_t>(i), th) ? dy[i] * scale : 0.f;
  cx.round(dz);
}

}  // namespace

extern "C" void or_layer_backward(or_layer* l, const float* dy_in, float* dx_out, uint32_t mb, float* const* grads) {
  const or_layer_desc& d = l->d;
  const Ctx& cx = l->cx;
  const Dims D = dims(d);
  auto it = l->saved.find(mb);
  if (it == l->saved.end()) return;
  auto& sv = it->second;
  const auto& P = l->p;
  const float scale_h = 1.f / (1.f - d.dropout_hidden), scale_a = 1.f / (1.f - d.dropout_attn);
  const uint32_t th_h = curator::dropout_threshold16(d.dropout_hidden), th_a = curator::dropout_threshold16(d.dropout_attn);
  const float alpha = 1.f / std::sqrt(static_cast<float>(D.hd));
  const int64_t M = D.M, h = D.h, ff = D.ff, s = D.s, hd = D.hd, cw = D.cw, fw = D.fw, ld3 = 3 * cw;
  Vec dy(dy_in, dy_in + M * h);

  // column-parallel "f" backward: per-shard dgrad partials rounded, summed over the computed shards
  // (the TP all-reduce), rounded. dout holds the computed shards' columns ([M, ns * shard_rows]);
  // W is the global [.., h] weight, shard r owns its rows [(s0+r)*shard_rows, ...).
  auto col_parallel_dgrad = [&](const Vec& dout, int64_t out_cols, const float* W, int64_t shard_rows, Vec& din) {
    din.assign(M * h, 0.f);
    Vec part(M * h);
    for (int64_t r = 0; r < D.ns; ++r) {
      gemm(false, false, M, h, shard_rows, dout.data() + r * shard_rows, out_cols, W + (D.s0 + r) * shard_rows * h, h,
           part.data(), h, false);
      cx.round(part);
      for (int64_t i = 0; i < M * h; ++i) din[i] += part[i];
    }
    cx.round(din);
  };

  // ---- MLP
  Vec dm;
  dropout_bwd(cx, dy, dm, M * h, site(d, "mlp.out", mb), th_h, scale_h);
  colsum_acc(dm, M, h, grads[P_FC2B]);
  Vec dpre(M * fw);
  // dpre = dm W2[:, shards] (W2 is [h, ff]), times GeLU'(pre)
  gemm(false, false, M, fw, h, dm.data(), h, P[P_FC2W] + D.s0 * D.ffl, ff, dpre.data(), fw, false);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M * fw; ++i) dpre[i] *= gelu_grad(sv.pre[i]);
  cx.round(dpre);
  // dW2[:, shards] += dm^T act ; db1[shards] += colsum dpre ; dW1[shards, :] += dpre^T ln2
  gemm(true, false, h, fw, M, dm.data(), h, sv.act.data(), fw, grads[P_FC2W] + D.s0 * D.ffl, ff, true);
  colsum_acc(dpre, M, fw, grads[P_FC1B] + D.s0 * D.ffl);
  gemm(true, false, fw, h, M, dpre.data(), fw, sv.ln2.data(), h, grads[P_FC1W] + D.s0 * D.ffl * h, h, true);
  Vec dln2;
  col_parallel_dgrad(dpre, fw, P[P_FC1W], D.ffl, dln2);
  Vec dx1;
  ln_backward(cx, dln2, sv.x1, P[P_LN2G], sv.mean2, sv.rstd2, &dy, dx1, grads[P_LN2G], grads[P_LN2B], M, h);

  // ---- attention
  Vec dz;
  dropout_bwd(cx, dx1, dz, M * h, site(d, "attn.out", mb), th_h, scale_h);
  colsum_acc(dz, M, h, grads[P_PROJB]);
  Vec dctx(M * cw);
  gemm(false, false, M, cw, h, dz.data(), h, P[P_PROJW] + D.s0 * D.hl, h, dctx.data(), cw, false);
  cx.round(dctx);
  gemm(true, false, h, cw, M, dz.data(), h, sv.ctx.data(), cw, grads[P_PROJW] + D.s0 * D.hl, h, true);

  // attention backward per (bb, head) as packed GEMMs, one head per thread:
  //   dP = dctx V^T ; dS = alpha P~ (dP_kept - D_i) (softmax + dropout backward, row by row) ;
  //   dV = P^T dctx ; dK = dS^T Q ; dQ = dS K
  Vec dqkv(M * ld3, 0.f);
  const uint64_t site_a = site(d, "attn.probs", mb);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t bb = 0; bb < D.b; ++bb) {
    for (int64_t hh = 0; hh < D.Hc; ++hh) {
      const float* q = &sv.qkv[bb * s * ld3 + hh * 3 * hd];
      const float* k = q + hd;
      const float* v = q + 2 * hd;
      float* dq = &dqkv[bb * s * ld3 + hh * 3 * hd];
      float* dk = dq + hd;
      float* dv = dq + 2 * hd;
      const float* S = &sv.S[(bb * D.Hc + hh) * s * s];
      const float* Pm = &sv.P[(bb * D.Hc + hh) * s * s];
      const float* dc = &dctx[bb * s * cw + hh * hd];
      Vec dP(s * s), dS(s * s, 0.f);
      gemm(false, true, s, s, hd, dc, cw, v, ld3, dP.data(), s, false);
      const uint64_t base0 = (static_cast<uint64_t>(bb) * D.H + D.head0 + hh) * s;
      Vec y(s), g(s);
      for (int64_t i = 0; i < s; ++i) {
        const float lse = sv.lse[(bb * D.Hc + hh) * s + i];
        float dot = 0.f;
        for (int64_t j = 0; j <= i; ++j) {
          float acc = dP[i * s + j];
          if (cx.emu) acc = bf16_round(acc);
          const bool keep = curator::dropout_keep(site_a, (base0 + i) * static_cast<uint64_t>(s) + j, th_a);
          y[j] = std::exp(S[i * s + j] - lse);
          g[j] = keep ? acc * scale_a : 0.f;
          dot += y[j] * g[j];
        }
        for (int64_t j = 0; j <= i; ++j) {
          const float ds = alpha * y[j] * (g[j] - dot);
          dS[i * s + j] = cx.emu ? bf16_round(ds) : ds;
        }
      }
      gemm(true, false, s, hd, s, Pm, s, dc, cw, dv, ld3, false);
      gemm(true, false, s, hd, s, dS.data(), s, q, ld3, dk, ld3, false);
      gemm(false, false, s, hd, s, dS.data(), s, k, ld3, dq, ld3, false);
    }
  }
  cx.round(dqkv);
  colsum_acc(dqkv, M, ld3, grads[P_QKVB] + D.s0 * 3 * D.hl);
  gemm(true, false, ld3, h, M, dqkv.data(), ld3, sv.ln1.data(), h, grads[P_QKVW] + D.s0 * 3 * D.hl * h, h, true);
  Vec dln1;
  col_parallel_dgrad(dqkv, ld3, P[P_QKVW], 3 * D.hl, dln1);
  Vec dx;
  ln_backward(cx, dln1, sv.x, P[P_LN1G], sv.mean1, sv.rstd1, &dx1, dx, grads[P_LN1G], grads[P_LN1B], M, h);
  std::copy(dx.begin(), dx.end(), dx_out);
  l->saved.erase(it);
}

// ---------------------------------------------------------------------------- seeded streams
extern "C" void or_fill_normal(float* out, int64_t rows, int64_t cols, int64_t global_cols, int64_t row0, int64_t col0,
                               uint64_t key, float mean, float std, int32_t round_bf16) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < rows * cols; ++e) {
    const int64_t r = e / cols, c = e % cols;
    const uint64_t g = static_cast<uint64_t>(row0 + r) * static_cast<uint64_t>(global_cols) + static_cast<uint64_t>(col0 + c);
    const float v = mean + std * static_cast<float>(curator::normal_at(key, g));
    out[e] = round_bf16 ? bf16_round(v) : v;
  }
}

extern "C" uint64_t or_site_seed(uint64_t seed, const char* name, uint32_t layer, uint32_t mb) {
  return curator::site_seed(seed, name, layer, mb);
}

extern "C" uint64_t or_step_seed(uint64_t seed, uint64_t step) { return curator::step_seed(seed, step); }

extern "C" int32_t or_dropout_keep(uint64_t site_seed, uint64_t idx, uint32_t th16) {
  return curator::dropout_keep(site_seed, idx, th16) ? 1 : 0;
}

extern "C" void or_mse_loss(const float* y, const float* t, float* dy, float* loss, int64_t n) {
  double acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float dd = y[i] - t[i];
    acc += 0.5 * double(dd) * dd;
    dy[i] = dd / static_cast<float>(n);
  }
  *loss = static_cast<float>(acc / n);
}
