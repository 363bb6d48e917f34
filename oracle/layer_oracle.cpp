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

// C[m][n] = sum_k A[m*lda + k] * B[n*ldb + k]  (both operands contiguous in k)
void gemm_nt(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int64_t m, int64_t n,
             int64_t k) {
  constexpr int RB = 4, CB = 4;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t i0 = 0; i0 < m; i0 += RB) {
    for (int64_t j0 = 0; j0 < n; j0 += CB) {
      float acc[RB][CB] = {};
      const int64_t ri = std::min<int64_t>(RB, m - i0), cj = std::min<int64_t>(CB, n - j0);
      if (ri == RB && cj == CB) {
        const float* a[RB];
        const float* b[CB];
        for (int r = 0; r < RB; ++r) a[r] = A + (i0 + r) * lda;
        for (int c = 0; c < CB; ++c) b[c] = B + (j0 + c) * ldb;
        for (int r = 0; r < RB; ++r)
          for (int c = 0; c < CB; ++c) {
            float s = 0.f;
#pragma omp simd reduction(+ : s)
            for (int64_t q = 0; q < k; ++q) s += a[r][q] * b[c][q];
            acc[r][c] = s;
          }
      } else {
        for (int r = 0; r < ri; ++r)
          for (int c = 0; c < cj; ++c) {
            float s = 0.f;
            for (int64_t q = 0; q < k; ++q) s += A[(i0 + r) * lda + q] * B[(j0 + c) * ldb + q];
            acc[r][c] = s;
          }
      }
      for (int r = 0; r < ri; ++r)
        for (int c = 0; c < cj; ++c) C[(i0 + r) * ldc + j0 + c] = acc[r][c];
    }
  }
}

// out[c][r] = in[r][c]   (in: rows x cols, leading dimension ld)
Vec transpose(const float* in, int64_t rows, int64_t cols, int64_t ld) {
  Vec out(static_cast<size_t>(rows * cols));
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) out[c * rows + r] = in[r * ld + c];
  return out;
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
} or_layer_desc;

// Parameter order and global shapes as in include/mtnlg.h (enum mt_param).
struct or_layer {
  or_layer_desc d;
  Ctx cx;
  std::vector<Vec> p;  // 12 global parameters
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
    int64_t r, c;
    or_param_shape(d, i, &r, &c);
    l->p.emplace_back(params[i], params[i] + r * c);
  }
  return l;
}

void or_layer_destroy(or_layer* l) { delete l; }

int or_num_threads(void) { return omp_get_max_threads(); }

}  // extern "C"

namespace {

struct Dims {
  int64_t b, s, h, H, hd, M, ff, t, Hl, hl, ffl;
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
  return x;
}

void layer_norm(const Ctx& cx, const Vec& x, const Vec& g, const Vec& be, Vec& y, Vec& mean, Vec& rstd, int64_t M,
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
void bias_dropout_residual(const Ctx& cx, const Vec& z, const Vec& bias, const Vec& resid, Vec& y, int64_t M, int64_t h,
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

// Slice rows [r0, r0+nr) x cols [c0, c0+nc) of a row-major matrix with `cols` columns.
Vec slice(const Vec& m, int64_t cols, int64_t r0, int64_t nr, int64_t c0, int64_t nc) {
  Vec o(nr * nc);
  for (int64_t r = 0; r < nr; ++r) std::copy_n(&m[(r0 + r) * cols + c0], nc, &o[r * nc]);
  return o;
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

  layer_norm(cx, sv.x, P[P_LN1G], P[P_LN1B], sv.ln1, sv.mean1, sv.rstd1, D.M, D.h, d.ln_eps);
  // column-parallel QKV: the full output is the concatenation of the TP shards, so it is computed
  // at once (rows of the global weight in (head, {q,k,v}, hd) order).
  sv.qkv.assign(D.M * 3 * D.h, 0.f);
  gemm_nt(sv.ln1.data(), D.h, P[P_QKVW].data(), D.h, sv.qkv.data(), 3 * D.h, D.M, 3 * D.h, D.h);
  for (int64_t r = 0; r < D.M; ++r)
    for (int64_t c = 0; c < 3 * D.h; ++c) sv.qkv[r * 3 * D.h + c] += P[P_QKVB][c];
  cx.round(sv.qkv);

  // attention per (microbatch row bb, head)
  const int64_t s = D.s, hd = D.hd;
  sv.S.assign(D.b * D.H * s * s, 0.f);
  sv.P.assign(D.b * D.H * s * s, 0.f);
  sv.lse.assign(D.b * D.H * s, 0.f);
  sv.ctx.assign(D.M * D.h, 0.f);
  const uint64_t site_a = site(d, "attn.probs", mb);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t bb = 0; bb < D.b; ++bb) {
    for (int64_t hh = 0; hh < D.H; ++hh) {
      const float* q = &sv.qkv[bb * s * 3 * D.h + hh * 3 * hd];
      const float* k = q + hd;
      const float* v = q + 2 * hd;
      float* S = &sv.S[(bb * D.H + hh) * s * s];
      float* Pm = &sv.P[(bb * D.H + hh) * s * s];
      for (int64_t i = 0; i < s; ++i) {
        float mx = -INFINITY;
        for (int64_t j = 0; j <= i; ++j) {
          float acc = 0.f;
          for (int64_t e = 0; e < hd; ++e) acc += q[i * 3 * D.h + e] * k[j * 3 * D.h + e];
          acc *= alpha;
          if (cx.emu) acc = bf16_round(acc);
          S[i * s + j] = acc;
          mx = std::max(mx, acc);
        }
        float sum = 0.f;
        for (int64_t j = 0; j <= i; ++j) sum += std::exp(S[i * s + j] - mx);
        const float lse = mx + std::log(sum);
        sv.lse[(bb * D.H + hh) * s + i] = lse;
        const uint64_t base = ((static_cast<uint64_t>(bb) * D.H + hh) * s + i) * static_cast<uint64_t>(s);
        for (int64_t j = 0; j <= i; ++j) {
          float pv = std::exp(S[i * s + j] - mx) / sum;
          pv = curator::dropout_keep(site_a, base + j, th_a) ? pv * scale_a : 0.f;
          Pm[i * s + j] = cx.emu ? bf16_round(pv) : pv;
        }
      }
      // ctx = P V
      for (int64_t i = 0; i < s; ++i)
        for (int64_t e = 0; e < hd; ++e) {
          float acc = 0.f;
          for (int64_t j = 0; j <= i; ++j) acc += Pm[i * s + j] * v[j * 3 * D.h + e];
          sv.ctx[(bb * s + i) * D.h + hh * hd + e] = acc;
        }
    }
  }
  cx.round(sv.ctx);

  // row-parallel attn-out: per TP shard partial (rounded like the GPU epilogue), summed (the all-reduce)
  auto row_parallel = [&](const Vec& in, int64_t in_cols, const Vec& W, int64_t shard_cols, Vec& out) {
    out.assign(D.M * D.h, 0.f);
    Vec part(D.M * D.h);
    for (int64_t r = 0; r < D.t; ++r) {
      const Vec in_s = slice(in, in_cols, 0, D.M, r * shard_cols, shard_cols);
      const Vec w_s = slice(W, in_cols, 0, D.h, r * shard_cols, shard_cols);
      gemm_nt(in_s.data(), shard_cols, w_s.data(), shard_cols, part.data(), D.h, D.M, D.h, shard_cols);
      cx.round(part);
      for (int64_t i = 0; i < D.M * D.h; ++i) out[i] += part[i];
    }
    cx.round(out);
  };
  Vec z;
  row_parallel(sv.ctx, D.h, P[P_PROJW], D.hl, z);
  bias_dropout_residual(cx, z, P[P_PROJB], sv.x, sv.x1, D.M, D.h, site(d, "attn.out", mb), th_h, scale_h);
  layer_norm(cx, sv.x1, P[P_LN2G], P[P_LN2B], sv.ln2, sv.mean2, sv.rstd2, D.M, D.h, d.ln_eps);
  sv.pre.assign(D.M * D.ff, 0.f);
  gemm_nt(sv.ln2.data(), D.h, P[P_FC1W].data(), D.h, sv.pre.data(), D.ff, D.M, D.ff, D.h);
  sv.act.assign(D.M * D.ff, 0.f);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < D.M * D.ff; ++i) {
    float pr = sv.pre[i] + P[P_FC1B][i % D.ff];
    if (cx.emu) pr = bf16_round(pr);
    sv.pre[i] = pr;
    const float a = gelu(pr);
    sv.act[i] = cx.emu ? bf16_round(a) : a;
  }
  Vec m;
  row_parallel(sv.act, D.ff, P[P_FC2W], D.ffl, m);
  Vec y;
  bias_dropout_residual(cx, m, P[P_FC2B], sv.x1, y, D.M, D.h, site(d, "mlp.out", mb), th_h, scale_h);
  std::copy(y.begin(), y.end(), y_out);
}

namespace {

// dX = dY * W where W is [n, k] row-major (dY [M, n]) -> [M, k]; via the transposed weight.
void dgrad(const float* dY, int64_t n, const float* W, int64_t k, float* dX, int64_t M) {
  const Vec Wt = transpose(W, n, k, k);  // [k, n]
  gemm_nt(dY, n, Wt.data(), n, dX, k, M, k, n);
}

// dW[n][k] += sum_tok dY[tok][n] * X[tok][k]
void wgrad_acc(const float* dY, int64_t n, const float* X, int64_t k, float* dW, int64_t M) {
  const Vec dYt = transpose(dY, M, n, n);  // [n, M]
  const Vec Xt = transpose(X, M, k, k);    // [k, M]
  Vec tmp(n * k);
  gemm_nt(dYt.data(), M, Xt.data(), M, tmp.data(), k, n, k, M);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n * k; ++i) dW[i] += tmp[i];
}

void colsum_acc(const Vec& x, int64_t M, int64_t n, float* out) {
  for (int64_t c = 0; c < n; ++c) {
    double s = 0;
    for (int64_t r = 0; r < M; ++r) s += x[r * n + c];
    out[c] += static_cast<float>(s);
  }
}

// LayerNorm backward: returns dx (+resid), accumulates dgamma, dbeta.
void ln_backward(const Ctx& cx, const Vec& dy, const Vec& x, const Vec& g, const Vec& mean, const Vec& rstd,
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
  const int64_t M = D.M, h = D.h, ff = D.ff, s = D.s, hd = D.hd;
  Vec dy(dy_in, dy_in + M * h);

  // column-parallel "f" backward: per-shard dgrad partials rounded, summed, rounded (the TP all-reduce)
  auto col_parallel_dgrad = [&](const Vec& dout, int64_t out_cols, const Vec& W, int64_t shard_rows, Vec& din) {
    din.assign(M * h, 0.f);
    Vec part(M * h);
    for (int64_t r = 0; r < D.t; ++r) {
      const Vec do_s = slice(dout, out_cols, 0, M, r * shard_rows, shard_rows);
      const Vec w_s = slice(W, h, r * shard_rows, shard_rows, 0, h);
      dgrad(do_s.data(), shard_rows, w_s.data(), h, part.data(), M);
      cx.round(part);
      for (int64_t i = 0; i < M * h; ++i) din[i] += part[i];
    }
    cx.round(din);
  };

  // ---- MLP
  Vec dm;
  dropout_bwd(cx, dy, dm, M * h, site(d, "mlp.out", mb), th_h, scale_h);
  colsum_acc(dm, M, h, grads[P_FC2B]);
  Vec dpre(M * ff);
  dgrad(dm.data(), h, P[P_FC2W].data(), ff, dpre.data(), M);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M * ff; ++i) dpre[i] *= gelu_grad(sv.pre[i]);
  cx.round(dpre);
  wgrad_acc(dm.data(), h, sv.act.data(), ff, grads[P_FC2W], M);
  colsum_acc(dpre, M, ff, grads[P_FC1B]);
  wgrad_acc(dpre.data(), ff, sv.ln2.data(), h, grads[P_FC1W], M);
  Vec dln2;
  col_parallel_dgrad(dpre, ff, P[P_FC1W], D.ffl, dln2);
  Vec dx1;
  ln_backward(cx, dln2, sv.x1, P[P_LN2G], sv.mean2, sv.rstd2, &dy, dx1, grads[P_LN2G], grads[P_LN2B], M, h);

  // ---- attention
  Vec dz;
  dropout_bwd(cx, dx1, dz, M * h, site(d, "attn.out", mb), th_h, scale_h);
  colsum_acc(dz, M, h, grads[P_PROJB]);
  Vec dctx(M * h);
  dgrad(dz.data(), h, P[P_PROJW].data(), h, dctx.data(), M);
  cx.round(dctx);
  wgrad_acc(dz.data(), h, sv.ctx.data(), h, grads[P_PROJW], M);

  Vec dqkv(M * 3 * h, 0.f);
  const uint64_t site_a = site(d, "attn.probs", mb);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t bb = 0; bb < D.b; ++bb) {
    for (int64_t hh = 0; hh < D.H; ++hh) {
      const int64_t ld3 = 3 * h;
      const float* q = &sv.qkv[bb * s * ld3 + hh * 3 * hd];
      const float* k = q + hd;
      const float* v = q + 2 * hd;
      float* dq = &dqkv[bb * s * ld3 + hh * 3 * hd];
      float* dk = dq + hd;
      float* dv = dq + 2 * hd;
      const float* S = &sv.S[(bb * D.H + hh) * s * s];
      const float* Pm = &sv.P[(bb * D.H + hh) * s * s];
      const float* dc = &dctx[bb * s * h + hh * hd];
      Vec dS(s * s, 0.f);
      const uint64_t base0 = (static_cast<uint64_t>(bb) * D.H + hh) * s;
      for (int64_t i = 0; i < s; ++i) {
        const float lse = sv.lse[(bb * D.H + hh) * s + i];
        Vec y(i + 1), g(i + 1);
        float dot = 0.f;
        for (int64_t j = 0; j <= i; ++j) {
          float acc = 0.f;
          for (int64_t e = 0; e < hd; ++e) acc += dc[i * h + e] * v[j * ld3 + e];
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
      for (int64_t j = 0; j < s; ++j)
        for (int64_t e = 0; e < hd; ++e) {
          float av = 0.f, ak = 0.f;
          for (int64_t i = j; i < s; ++i) {
            av += Pm[i * s + j] * dc[i * h + e];
            ak += dS[i * s + j] * q[i * ld3 + e];
          }
          dv[j * ld3 + e] = av;
          dk[j * ld3 + e] = ak;
        }
      for (int64_t i = 0; i < s; ++i)
        for (int64_t e = 0; e < hd; ++e) {
          float aq = 0.f;
          for (int64_t j = 0; j <= i; ++j) aq += dS[i * s + j] * k[j * ld3 + e];
          dq[i * ld3 + e] = aq;
        }
    }
  }
  cx.round(dqkv);
  colsum_acc(dqkv, M, 3 * h, grads[P_QKVB]);
  wgrad_acc(dqkv.data(), 3 * h, sv.ln1.data(), h, grads[P_QKVW], M);
  Vec dln1;
  col_parallel_dgrad(dqkv, 3 * h, P[P_QKVW], 3 * D.hl, dln1);
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
