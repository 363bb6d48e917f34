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
  MT_EPI_ACCUM_F32 = 4,    /* D(f32) += alpha*acc   (fp32 gradient accumulation across microbatches) */
  MT_EPI_STORE_BF16_ROWSTATS = 5 /* D = bf16(alpha*acc), plus per (row, BN-column block) softmax statistics
                                    of the stored values: aux = float2 [batch][m][ld_aux] {max, sum exp(x - max)}
                                    over the block's columns (causal modes: columns <= row only); requires
                                    block_n = 128 or 256 and ld_aux >= ceil(n / block_n) */
};

enum mt_causal {
  MT_CAUSAL_NONE = 0,
  MT_CAUSAL_SKIP_UPPER_TILES = 1, /* skip D tiles entirely above the diagonal (n_begin > m_end-1)   */
  MT_CAUSAL_K_LE_M = 2,           /* A is lower-triangular in (m,k): contract k < m_tile_end only    */
  MT_CAUSAL_K_GE_M = 3            /* A is upper-triangular in (m,k): contract k >= m_tile_begin only */
};

/* Fused all-reduce of the output over a tensor-parallel group (NVLink SHARP / multimem): every rank
 * launches the same GEMM on its partial operands with d in symmetric memory; each 128-row x BN output
 * unit is published with a flag once stored, and its owner rank (round-robin over units) sums all
 * ranks' copies with multimem.ld_reduce (fp32 accumulation, one rounding) and writes the sum to every
 * rank with multimem.st from its epilogue warps while the tensor cores continue with later tiles.
 * mt_gemm_allreduce_wait(counter, target) then orders the consumers after all units of all ranks.
 * Requirements: STORE_BF16 epilogue, batch 1, no causal mode; d is the local address of offset 0 of
 * the symmetric buffer whose multicast address is d_multicast. */
typedef struct mt_gemm_allreduce {
  void* d_multicast;             /* multicast address of d */
  uint32_t* flags_local;         /* this rank's per-unit ready flags (symmetric memory) */
  const uint32_t* flags_peer[8]; /* each rank's flag array, load/store accessible, by rank */
  uint32_t* counter_multicast;   /* multicast address of the per-rank completion counter */
  int64_t flag_capacity;         /* units the flag arrays can hold */
  uint32_t epoch;                /* larger than every epoch used before on these flags */
  int32_t rank, ranks;
  int32_t reduce_in_epilogue;    /* 1: the GEMM's epilogue warps reduce the owned units; 0: the GEMM only
                                    publishes them and mt_gemm_allreduce_reduce (a concurrent kernel on
                                    the SMs the GEMM leaves free, max_ctas) reduces them */
  int32_t groups;                /* > 0: column-group mode — the GEMM counts finished units per group of
                                    column blocks on flags_local[g] (zeroed by the caller before the
                                    launch) and mt_gemm_allreduce_reduce_groups reduces group by group */
  int64_t units;                 /* out: number of output units of this launch (counter increments) */
  int64_t geom[8];               /* out: unit geometry of the launch, read by mt_gemm_allreduce_reduce */
  int64_t group_cols;            /* out: column blocks per group (0: group mode not applicable) */
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
   * tiles is split over k and reduced by the last-arriving split). The first 64 KB hold arrival
   * counters, which the kernel leaves zeroed. NULL disables. MT_GEMM_WORKSPACE_BYTES suggests a size. */
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
/* Stream-ordered wait until the local completion counter reaches `target` (all units of all ranks of
 * the fused all-reduce launches so far); 1 launch. */
int mt_gemm_allreduce_wait(const uint32_t* counter_local, uint32_t target, void* stream);
/* Reducer for a launch with reduce_in_epilogue = 0: `ctas` CTAs reduce this rank's owned units in
 * publication order as the GEMM (running concurrently, e.g. on another stream) publishes them, then
 * wait until the local counter reaches `target`. 1 launch. */
int mt_gemm_allreduce_reduce(const mt_gemm_allreduce* ar, void* d, int64_t ldd, const uint32_t* counter_local,
                             uint32_t target, int32_t ctas, void* stream);

/* Number of kernel launches mt_gemm issues per call (always 1). */
int mt_gemm_launches_per_call(void);

#ifdef __cplusplus
}
#endif
#endif
