// Launchers of the HBM-bound kernels of the tensor-sliced layer (LayerNorm fwd/bwd, causal
// scaled-masked softmax fwd/bwd with attention dropout, bias+dropout+residual, bias-grad column
// sums, synthetic loss, seeded init). All take bf16 activations and an explicit stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mt {

typedef unsigned short bf16_t;  // raw bf16 bits on the host side of the launchers

// y = LN(x) * gamma + beta ; saves mean and rstd (fp32, one per row).
void ln_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows, int h,
            float eps, cudaStream_t s);
// dx = rstd * (g - mean(g) - xhat * mean(g * xhat)) [+ resid], g = dy * gamma.
void ln_bwd_dx(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
               const void* resid, void* dx, int rows, int h, cudaStream_t s);
// dgamma (+)= sum_rows dy * xhat ; dbeta (+)= sum_rows dy   (fp32, deterministic; += when accumulate)
void ln_bwd_params(const void* dy, const void* x, const float* mean, const float* rstd, float* dgamma, float* dbeta,
                   int rows, int h, float* workspace, bool accumulate, cudaStream_t s);

// out = resid + dropout(z + bias); mask index = elem_offset + (row * h + col) of the rows passed
// keep_out (optional): the dropout keep bits, one byte per 8 consecutive elements of a row
// ([rows][h / 8], bit j = element 8 v + j kept), for the backward to read instead of re-hashing
void bias_dropout_residual(const void* z, const void* bias, const void* resid, void* out, int rows, int h,
                           uint64_t site_seed, uint32_t thresh16, float scale, cudaStream_t s,
                           uint64_t elem_offset = 0, uint8_t* keep_out = nullptr);
// dz = dropout'(dy) ; dbias (+)= sum_rows dz   (keep_in: the forward's keep bytes, or nullptr: re-hash)
void dropout_bwd_bias_grad(const void* dy, void* dz, float* dbias, int rows, int h, uint64_t site_seed,
                           uint32_t thresh16, float scale, float* workspace, bool accumulate, cudaStream_t s,
                           uint64_t elem_offset = 0, const uint8_t* keep_in = nullptr);
// dbias (+)= sum_rows x   (x bf16 [rows, n])
void bias_grad(const void* x, float* dbias, int rows, int n, long long ldx, float* workspace, bool accumulate,
               cudaStream_t s);
size_t colsum_workspace_floats(int rows, int n);

// Fused LayerNorm backward: dx (= ln_bwd_dx) and dgamma/dbeta (= ln_bwd_params) in one pass over dy
// and x (TMA-fed persistent row kernel, rows_sm100.cu; falls back to the two kernels above).
int ln_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd, const void* resid,
            void* dx, float* dgamma, float* dbeta, int rows, int h, float* workspace, bool accumulate, cudaStream_t s);
// out = resid + dropout(z + bias) and, if gamma != nullptr, y = LN(out) (one pass).
int bias_dropout_residual_ln(const void* z, const void* bias, const void* resid, void* out, const void* gamma,
                              const void* beta, void* y, float* mean, float* rstd, int rows, int h, float eps,
                              uint64_t site_seed, uint32_t thresh16, float scale, uint64_t elem_offset, cudaStream_t s,
                              uint8_t* keep_out = nullptr);
// dgamma/dbeta (+)= sum over `splits` fp32 partials ws[2][splits][h]
void colsum_partials(const float* ws, float* out0, float* out1, int n, int splits, bool accumulate, cudaStream_t s);
// rows_sm100.cu (return false when the shape does not fit; callers then use the per-row kernels)
int row_kernel_ctas(int rows);
bool ln_fwd_rows(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows, int h,
                 float eps, cudaStream_t s);
bool bdr_ln_rows(const void* z, const void* bias, const void* resid, void* out, const void* gamma, const void* beta,
                 void* y, float* mean, float* rstd, int rows, int h, float eps, uint64_t seed, uint32_t thresh16,
                 float scale, uint64_t elem_offset, cudaStream_t s, uint8_t* keep_out = nullptr);
bool ln_bwd_rows(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                 const void* resid, void* dx, float* dgamma, float* dbeta, int rows, int h, float* ws, bool accumulate,
                 cudaStream_t s);

// Causal softmax over S (already scaled by 1/sqrt(hd)), rows of `batch_heads` independent
// [seq x seq] blocks. P = dropout(softmax(S)); zeros above the diagonal up to the next
// multiple of 256 columns (what the causal GEMMs read); lse saved per row.
// Attention dropout element index = ((head_base + bh) * seq + i) * seq + j, where bh is the
// block index and head_base maps local blocks to global (microbatch-row, head) ids.
void softmax_fwd(const void* S, void* P, float* lse, int batch_heads, int seq, long long head_base,
                 uint64_t site_seed, uint32_t thresh16, float scale, cudaStream_t s);

// One-pass softmax backward with the row term precomputed: D[bh * seq + i] = dctx_i . ctx_i of the
// head (= sum_j P_ij dP_ij), so dS = alpha * p * (dP' - D) needs no in-kernel row reduction.
void softmax_bwd_rowdot(const void* S, const float* lse, const float* D, void* dP, int batch_heads, int seq,
                        long long head_base, uint64_t site_seed, uint32_t thresh16, float scale, float alpha,
                        cudaStream_t s);
void attn_rowdot(const void* dout, const void* out, long long ld, int hd, int heads, int seq, float* D, cudaStream_t s);

// Fused causal flash attention on tcgen05 (attention_sm100.cu). Return 0 ok, 1 unsupported shape
// (seq % 128 or head dim not in {64, 128, 160}), 2 CUDA error.
int attention_fwd(const void* qkv, long long ld_qkv, int heads, int seq, int hd, long long head_base, float alpha,
                  uint64_t seed, uint32_t thresh16, float drop_scale, void* out, long long ld_out, float* lse,
                  uint32_t* mask, int* mask_written, cudaStream_t s);
int attention_bwd(const void* qkv, long long ld_qkv, const void* ctx, const void* dctx, long long ld_ctx, int heads,
                  int seq, int hd, long long head_base, float alpha, uint64_t seed, uint32_t thresh16,
                  float drop_scale, const float* lse, float* D, void* dqkv, const uint32_t* mask, float* dq_acc,
                  cudaStream_t s);

// loss += sum 0.5 (y - t)^2 / n ; dy = (y - t) / n     (n = rows * h)
// n_total: the element count the mean is over when y/t are one rank's rows of a larger tensor (0 = n)
void mse_loss(const void* y, const void* t, void* dy, float* loss, long long n, cudaStream_t s, long long n_total = 0);

// Seeded normal init of a TP shard of a row-major [global_rows x global_cols] tensor:
// out[r][c] = bf16(mean + std * normal_at(key, (row0 + r) * global_cols + col0 + c)).
void fill_normal(void* out, long long rows, long long cols, long long global_cols, long long row0, long long col0,
                 uint64_t key, float mean, float std, cudaStream_t s);
void fill_zero_f32(float* p, size_t n, cudaStream_t s);

}  // namespace mt
