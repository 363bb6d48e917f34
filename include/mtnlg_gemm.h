/* mtnlg_gemm.h — C ABI of the sm_100a tcgen05 GEMM used by every contraction of the
 * tensor-sliced transformer layer (column-parallel QKV / fc1, row-parallel attention-out /
 * fc2, their dgrad and wgrad, and the batched attention contractions).
 *
 * The reference (arxiv/paper_2201_11990, `proj/`) has no GEMM: the layer math is restated
 * from PAPER.md:133-150 (Megatron tensor slicing). This header is the kernel-level boundary;
 * the layer-level boundary is mtnlg.h.
 *
 * Logical problem, per batch index b in [0, batch):
 *     D[b][m][n] = epilogue( alpha * sum_k A[b][m][k] * B[b][n][k] )
 * A and B are bf16. "K-major" means k is the contiguous index:
 *     A(m,k) = a[b*a_batch_stride + m*lda + k]          (a_mn_major = 0)
 *     A(m,k) = a[b*a_batch_stride + k*lda + m]          (a_mn_major = 1)
 * and likewise for B(n,k). D(m,n) = d[b*d_batch_stride + m*ldd + n]. All strides in elements.
 * Requirements: 16-byte aligned base pointers and leading dimensions (multiples of 8 elements).
 */
#ifndef MTNLG_GEMM_H
#define MTNLG_GEMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mt_epilogue {
  MT_EPI_STORE_BF16 = 0,   /* D = bf16(alpha*acc [+ bias[n]])                                  */
  MT_EPI_BIAS_GELU = 1,    /* aux = bf16(acc + bias[n]) (pre-activation), D = bf16(gelu(aux))   */
  MT_EPI_GELU_BWD = 2,     /* D = bf16(acc * gelu'(aux[m][n]))   (aux = saved pre-activation)    */
  MT_EPI_STORE_F32 = 3,    /* D(f32) = alpha*acc                                                */
  MT_EPI_ACCUM_F32 = 4     /* D(f32) += alpha*acc   (fp32 gradient accumulation across microbatches) */
};

enum mt_causal {
  MT_CAUSAL_NONE = 0,
  MT_CAUSAL_SKIP_UPPER_TILES = 1, /* skip D tiles entirely above the diagonal (n_begin > m_end-1)   */
  MT_CAUSAL_K_LE_M = 2,           /* A is lower-triangular in (m,k): contract k < m_tile_end only    */
  MT_CAUSAL_K_GE_M = 3            /* A is upper-triangular in (m,k): contract k >= m_tile_begin only */
};

/* Fused all-reduce of the output over a tensor-parallel group (NVLink SHARP / multimem): every rank
 * launches the same GEMM on its partial operands with d in symmetric memory. The GEMM counts each
 * finished 128-row x BN output unit on its column group's local counter (column blocks complete in
 * raster order); mt_gemm_allreduce_reduce_groups, running concurrently on the SMs the GEMM leaves free
 * (max_ctas), waits per group for this rank's GEMM and a cross-rank barrier, then sums this rank's
 * 1/ranks of the group's rows over all ranks with multimem.ld_reduce (fp32 accumulation, one rounding)
 * and writes the sum to every rank with multimem.st — so all but the last group's reduction overlap
 * the GEMM. mt_gemm_allreduce_wait(counter, target) then orders the consumers after every rank's
 * reducer. Every cross-rank wait is bounded by timeout_ns: a peer that never arrives raises
 * *error_flag and the kernels finish (with undefined data) instead of wedging the GPU.
 * Requirements: STORE_BF16 epilogue, batch 1, no causal mode, M a multiple of ranks, m-fastest raster
 * (M <= N); d is the local address of offset 0 of the symmetric buffer whose multicast address is
 * d_multicast. */
typedef struct mt_gemm_allreduce {
  void* d_multicast;             /* multicast address of d */
  uint32_t* group_counters;      /* local per-group unit counters, zeroed before each launch (<= 64) */
  uint32_t* counter_multicast;   /* multicast address of the per-rank completion counter */
  int32_t rank, ranks;
  int32_t groups;                /* column groups (1..64) */
  uint32_t* error_flag;          /* host-mapped word raised on a peer timeout (may be NULL) */
  uint64_t timeout_ns;           /* bound of every cross-rank wait (> 0) */
  int64_t units;                 /* out: number of output units of this launch */
  int64_t geom[8];               /* out: unit geometry of the launch, read by the reducer */
  int64_t group_cols;            /* out: column blocks per group */
} mt_gemm_allreduce;
typedef struct mt_gemm_args {
  const void* a;
  int64_t lda, a_batch_stride;
  int32_t a_mn_major;
  const void* b;
  int64_t ldb, b_batch_stride;
  int32_t b_mn_major;
  void* d;
  int64_t ldd, d_batch_stride;
  int64_t m, n, k, batch;
  float alpha;
  int32_t epilogue; /* enum mt_epilogue */
  int32_t causal;   /* enum mt_causal */
  const void* bias; /* bf16[n] or NULL */
  void* aux;        /* bf16, ld = ld_aux (pre-activation for the GeLU epilogues) */
  int64_t ld_aux;
  int32_t block_n;  /* 0 = auto; else 64/128/160/192/256 */
  int32_t max_ctas; /* 0 = one CTA per SM; else cap (leaves SMs free for a concurrent collective) */
  /* Optional zero-initialised device workspace enabling the split-K tail (the last, partial wave of
   * tiles is split over k and reduced by the last-arriving split) and the dynamic tile scheduler (tiles
   * handed out in raster order from a counter, so the CTAs sharing an operand tile stay in step and
   * read it from L2 once). The first 64 KB hold counters, which the kernel leaves zeroed. GEMMs that
   * share a workspace must be stream-ordered. NULL disables both. MT_GEMM_WORKSPACE_BYTES suggests a
   * size. */
  void* workspace;
  int64_t workspace_bytes;
  mt_gemm_allreduce* allreduce; /* NULL, or the fused TP all-reduce of d (see above) */
} mt_gemm_args;

#define MT_GEMM_WORKSPACE_BYTES (64ll << 20)

/* Launches on `stream` (a cudaStream_t). Returns 0 on success, 1 on bad arguments, 2 on CUDA error. */
int mt_gemm(const mt_gemm_args* args, void* stream);

/* Reducer of the column-group mode: `ctas` CTAs; per group, waits for this rank's GEMM (group_counters),
 * a cross-rank barrier on the counter, then reduces this rank's rows of the group's columns; counts
 * one exit per CTA. Counter after the launch = base + ranks * groups + ranks * ctas. */
int mt_gemm_allreduce_reduce_groups(const mt_gemm_allreduce* ar, int64_t ldd, uint32_t* group_counters,
                                    const uint32_t* counter_local, uint32_t base, int32_t ctas, void* stream);
/* Stream-ordered (bounded) wait until the local completion counter reaches `target`; 1 launch. */
int mt_gemm_allreduce_wait(const mt_gemm_allreduce* ar, const uint32_t* counter_local, uint32_t target,
                           void* stream);
/* Number of kernel launches mt_gemm issues per call (always 1). */
int mt_gemm_launches_per_call(void);

#ifdef __cplusplus
}
#endif
#endif
