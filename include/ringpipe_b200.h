/*
 * ringpipe-b200 C ABI.
 *
 * The drop-in boundary for the Ouroboros training step (arXiv 1909.06695) of
 * the reference `ringpipe` package.  The reference has no FFI: its seams are
 * the Python layer protocol (reference pkg/src/ringpipe/layers.py:28-37,
 * 96-280), the numba contraction kernels `kernels.mm/bmm`
 * (kernels.py:68-81) and the optimizer `apply` (optim.py:60-75, 114-126).
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - All pointers are device pointers unless stated; the library BORROWS them
 *    for the duration of the (asynchronous) call and never frees caller memory.
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *    it.  Handles are thread-compatible, not thread-safe (one owner).
 *  - Return value: rp_status.  On failure rp_last_error() gives the message.
 *    The Python host maps statuses onto the reference exception classes
 *    (tensor.py:20-25, model.py:28-33, engine.py:138-139).
 */
#ifndef RINGPIPE_B200_H
#define RINGPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rp_status {
  RP_OK = 0,
  RP_ERR_DIMENSION = 1, /* DimensionError   tensor.py:20-21 */
  RP_ERR_NONFINITE = 2, /* NonFiniteError   tensor.py:24-25 */
  RP_ERR_SCHEDULE = 3,  /* ScheduleViolation model.py:32-33 */
  RP_ERR_PARTITION = 4, /* PartitionError   model.py:28-29 */
  RP_ERR_CUDA = 5,
  RP_ERR_NCCL = 6,
  RP_ERR_INVALID = 7 /* ValueError */
} rp_status;

typedef enum rp_dtype { RP_F32 = 0, RP_BF16 = 1 } rp_dtype;

/* Contraction arithmetic.  BF16: bf16 operands, fp32 accumulate (production).
 * TF32X3: fp32 operands split hi/lo, three tf32 passes, fp32 accumulate
 * (check mode, ~fp32 accuracy).  TF32: single tf32 pass. */
typedef enum rp_math { RP_MATH_BF16 = 0, RP_MATH_TF32 = 1, RP_MATH_TF32X3 = 2 } rp_math;

typedef enum rp_epilogue {
  RP_EPI_STORE = 0,                 /* C = alpha*AB                                   */
  RP_EPI_BIAS_RELU = 1,             /* C = relu(alpha*AB + bias)        layers.py:190-191 */
  RP_EPI_BIAS_DROPOUT_RESIDUAL = 2, /* C = resid + (alpha*AB+bias)*mask layers.py:184-187,192-195 */
  RP_EPI_LSE_PARTIAL = 3,           /* per-(row, N-tile) (max, sumexp) + target logit  layers.py:310-316 */
  RP_EPI_CE_GRAD = 4                /* C = (exp(AB - lse[row]) - onehot) * ce_scale    layers.py:317-319 */
} rp_epilogue;

/* C[b] = epilogue(alpha * opA(A[b]) * opB(B[b])).
 * a_mn_major = 0: A is [M,K] row-major (ld = lda); 1: A is stored [K,M].
 * b_mn_major = 0: B is stored [N,K] row-major;      1: B is [K,N].
 * Replaces kernels.mm / kernels.bmm (kernels.py:68-81). */
typedef struct rp_gemm_args {
  int32_t math;      /* rp_math */
  int32_t out_dtype; /* rp_dtype of C (operands are bf16 for BF16 math, fp32 otherwise) */
  int32_t a_mn_major, b_mn_major;
  int64_t M, N, K, batch;
  const void* A;
  const void* A_lo; /* TF32X3 only: low halves (rp_tf32_split) */
  int64_t lda, stride_a;
  const void* B;
  const void* B_lo;
  int64_t ldb, stride_b;
  void* C;
  int64_t ldc, stride_c;
  int32_t epilogue; /* rp_epilogue */
  int32_t tile_n;   /* 0 = auto (see rp_gemm_tile_n) */
  float alpha;
  const float* bias;    /* [N] or NULL */
  const void* residual; /* same dtype as C, or NULL */
  int64_t ld_residual, stride_residual;
  int32_t drop_enabled;
  float drop_scale;         /* 1/(1-p) */
  uint64_t drop_seed;       /* layer stream seed, model.py:218-219 */
  uint64_t drop_threshold;  /* ceil(p * 2^53)                  */
  uint64_t drop_pos0;       /* stream position of element (0,0) */
  const int64_t* targets;   /* [batch*M] */
  const float* lse;         /* [batch*M] */
  float* partial;           /* [batch*M, n_tiles, 2] */
  float* target_logit;      /* [batch*M] */
  float ce_scale;
} rp_gemm_args;

const char* rp_version(void);
int rp_last_error(char* buf, size_t len);

int rp_gemm(const rp_gemm_args* args, void* stream);
int rp_gemm_tile_n(int64_t N);
int rp_tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src,
                  int64_t ld_dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RINGPIPE_B200_H */
