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
 *  - Row pitches ("ld*", in elements; 0 = the row length): bf16 rows that are
 *    operands of the TMA-fed GEMM need 16-byte pitches, so widths that are not
 *    multiples of 8 (BASELINE configs[3]: d 410, heads of 41, d_ff 2100) live
 *    in rows padded to the next multiple of 8.
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

/* compute dtypes (RP_F32, RP_BF16); the integer / f64 tags appear only in
 * state entries (rp_state_entry) */
typedef enum rp_dtype { RP_F32 = 0, RP_BF16 = 1, RP_I64 = 2, RP_U64 = 3, RP_F64 = 4 } rp_dtype;

/* Contraction arithmetic.  BF16: bf16 operands, fp32 accumulate (production).
 * TF32X3: fp32 operands split hi/lo, three tf32 passes, fp32 accumulate
 * (check mode, ~fp32 accuracy).  TF32: single tf32 pass. */
typedef enum rp_math { RP_MATH_BF16 = 0, RP_MATH_TF32 = 1, RP_MATH_TF32X3 = 2 } rp_math;

typedef enum rp_epilogue {
  RP_EPI_STORE = 0,                 /* C = alpha*AB                                   */
  RP_EPI_BIAS_RELU = 1,             /* C = relu(alpha*AB + bias)        layers.py:190-191 */
  RP_EPI_BIAS_DROPOUT_RESIDUAL = 2, /* C = resid + (alpha*AB+bias)*mask layers.py:184-187,192-195 */
  RP_EPI_LSE_PARTIAL = 3,           /* per-(row, N-tile, column half) (max, sumexp) + target logit  layers.py:310-316 */
  RP_EPI_CE_GRAD = 4,               /* C = (exp(AB - lse[row]) - onehot) * ce_scale    layers.py:317-319 */
  RP_EPI_RELU_GRAD = 5,             /* C = alpha*AB * (residual > 0)                   layers.py:221 */
  RP_EPI_GELU_GRAD = 6              /* C = alpha*AB * gelu'(residual), residual = the pre-activation z1 */
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
  float* partial;           /* [batch*M, 2*n_tiles, 2]: (max, sumexp) per N tile and column half */
  float* target_logit;      /* [batch*M] */
  float ce_scale;
  int32_t k_splits; /* > 1: C = [k_splits, M, N] fp32 partials over K ranges (rp_splitk_reduce) */
  int32_t max_ctas; /* > 0: cap the persistent grid (SM budget when sharing the GPU with another stream) */
  /* Banded A (causal / memory-window attention matrices): k_lo_sign = +1 means
   * row m of op(A) is zero for k < m + k_lo_off, so each output tile starts its
   * K loop at the first k-block any of its rows needs (adding the skipped
   * zeros would not change one bit of the fp32 sums); 0 = dense. */
  int32_t k_lo_sign;
  int64_t k_lo_off;
} rp_gemm_args;

const char* rp_version(void);
int rp_last_error(char* buf, size_t len);

int rp_gemm(const rp_gemm_args* args, void* stream);
/* N tile the library picks for an (M, N, batch) GEMM (sizes RP_EPI_LSE_PARTIAL partials) */
int rp_gemm_tile_n(int64_t M, int64_t N, int64_t batch);
/* K splits the library uses for an fp32 store GEMM of `batch` matrices with cap_bytes of partial scratch
 * (1 = none).  Split-K partials are laid out [split][matrix][M][N]; a batched GEMM finishes with one
 * rp_splitk_reduce over batch*M rows, so its output rows must be contiguous across the batch. */
int rp_gemm_choose_splits(int64_t M, int64_t N, int64_t K, int64_t batch, int64_t cap_bytes);
/* out[m,n] = sum_s part[s][m,n] in fixed order (deterministic split-K finish) */
int rp_splitk_reduce(const float* part, int32_t splits, int64_t M, int64_t N, float* out, int64_t ldo, void* stream);
int rp_tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src,
                  int64_t ld_dst, void* stream);


/* Device status word bits, OR-ed by kernels (a device int32 owned by the caller);
 * the host polls it once per step and raises the matching reference exception. */
#define RP_FLAG_NONFINITE 1 /* NonFiniteError: check_finite, tensor.py:93-96 / optim.py:47-49 */
#define RP_FLAG_DIMENSION 2 /* DimensionError: token/target range, layers.py:116-117, 292-293 */

/* ---- LayerNorm (layers.py:62-79) ----------------------------------------- */
/* y = (x-mu)*rstd*g + b over rows of d; saves mean/rstd (fp32). dtype: rp_dtype of x/y;
 * gain/bias are fp32. */
int rp_layernorm_fwd(int32_t dtype, const void* x, const float* gain, const float* bias, void* y, float* mean,
                     float* rstd, int64_t rows, int64_t d, int64_t ld_x, int64_t ld_y, int32_t* flag, void* stream);
/* dx = LN-backward(dy) + resid_grad (fp32), or not written when dx is NULL (rows that only add to
 * the gain / bias sums, as XL's stop-gradient memory rows); dx_masked = dx*dropout-mask (dtype) if
 * non-NULL; writes rp_layernorm_bwd_blocks(rows) partial rows of dgain/dbias. */
int rp_layernorm_bwd(int32_t dtype, const float* dy, const void* x, const float* mean, const float* rstd,
                     const float* gain, const float* resid_grad, float* dx, void* dx_masked, uint64_t seed,
                     uint64_t threshold, float scale, int32_t drop_enabled, float* partial_gain,
                     float* partial_bias, int64_t rows, int64_t d, int64_t ld_x, int64_t ld_masked, void* stream);
int rp_layernorm_bwd_blocks(int64_t rows);

/* ---- deterministic column sums (bias/gain gradients, layers.py:72-73,220,223) ---- */
int rp_colsum_blocks(int64_t rows);
int rp_colsum_partial(int32_t dtype, const void* x, int64_t rows, int64_t cols, int64_t ld, float* partial,
                      void* stream);
int rp_colsum_finish(const float* partial, int32_t nblocks, int64_t cols, float* out, void* stream);
/* up to 8 rp_colsum_finish jobs in one launch (bitwise equal to separate calls) */
int rp_colsum_finish_multi(const float* const* partials, const int32_t* nblocks, const int64_t* cols, float* const* outs,
                           int32_t n, void* stream);
/* out = g * mask(seed, pos0 + r*d + j) (dtype), partial column sums of the masked values
 * (layers.py:209-220). */
int rp_mask_grad_blocks(int64_t rows, int64_t d); /* partial rows rp_mask_grad writes */
int rp_mask_grad(int32_t dtype, const float* g, void* out, int64_t rows, int64_t d, uint64_t seed, uint64_t pos0,
                 uint64_t threshold, float scale, int32_t drop_enabled, float* partial, int64_t ld_out, void* stream);
/* partial rows rp_mask_grad writes when its output pitch ld_out differs from d */
int rp_mask_grad_blocks_ld(int64_t rows, int64_t d, int64_t ld_out);

/* ---- causal single-head attention softmax (layers.py:180-183, 237) ---------- */
/* rows = B*T rows of length T, row stride ld (>= T) */
int rp_softmax_causal(int32_t dtype, const float* scores, void* probs, int64_t rows, int64_t T, int64_t ld,
                      void* stream);
/* g_s = (g_p - rowsum(g_p*P)) * P * scale */
int rp_softmax_bwd(int32_t dtype, const float* grad_probs, const void* probs, void* grad_scores, float scale,
                   int64_t rows, int64_t T, int64_t ld, void* stream);

/* ---- Transformer-XL attention glue (oracle/xl.py) --------
 * No reference interface exists (the reference has no XL path): these are the
 * HBM-bound pieces around the tcgen05 GEMMs of relative-position multi-head
 * attention with segment memory.  xa rows: B*M memory rows, then B*T current
 * rows; head-major layouts qu/qv [H,B,T,dh], kh/vh [H,B,M+T,dh]. */
int rp_xl_split_qkv(int32_t dtype, const void* qkv, const float* r_w_bias, const float* r_r_bias, void* qu, void* qv,
                    void* kh, void* vh, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t ld_qkv,
                    int64_t ld_h, void* stream);
/* dst[h, r, c] = src[r*ld + h*dh + c] */
int rp_xl_split_heads(int32_t src_dtype, const void* src, int64_t ld, int32_t dst_dtype, void* dst, int64_t rows,
                      int32_t H, int32_t dh, int64_t ld_h, void* stream);
/* dst[r*ld + h*dh + c] = src[h, r, c] */
int rp_xl_merge_heads(int32_t src_dtype, const void* src, int32_t dst_dtype, void* dst, int64_t ld, int64_t rows,
                      int32_t H, int32_t dh, int64_t ld_h, void* stream);
/* g_qkv (xa row layout, [B*(M+T), 3d], row pitch ld_qkv, dtype) from head-major fp32 dQu, dQv
   (row pitch ld_g; 0 = dh) and dK, dV in `dtype` (row pitch ld_kv) */
int rp_xl_merge_grads(int32_t dtype, const float* g_qu, const float* g_qv, const void* g_kh, const void* g_vh,
                      void* g_qkv, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t ld_qkv,
                      int64_t ld_g, int64_t ld_kv, void* stream);
/* P = softmax((AC + relshift(BD)) * scale) over keys M-mem_len <= j <= M+i; rows = H*B*T */
int rp_xl_softmax_fwd(int32_t dtype, const float* ac, const float* bd, int64_t ld_scores, void* probs, int64_t ld_p,
                      int64_t rows, int64_t T, int64_t M, int64_t mem_len, float scale, void* stream);
/* Fused relative-position scores + softmax (bf16, dh = 64, tcgen05): P [H*B, T, ld_p] from
 * qu = q+u, qv = q+v [H*B, T, dh], kh [H*B, M+T, dh], r_h [H, M+T, dh]; the same P as
 * rp_xl_softmax_fwd over the AC / BD GEMM outputs, without materialising them */
int rp_xl_attn_fwd(const void* qu, const void* qv, const void* kh, const void* rh, void* probs, int64_t ld_p, int64_t B,
                   int64_t T, int64_t M, int32_t H, int32_t dh, int64_t mem_len, float scale, void* stream);
/* rp_xl_attn_fwd with P.V folded in (operand head dim dh = 64): also ctx = P v written as merged
 * rows (the normalised P tile stays in shared memory as the A operand of a second tcgen05 MMA into a
 * TMEM accumulator); P is still written for the backward.  A model head dim dh_out < 64 (e.g. 41)
 * rides with its q / k / v / r rows zero-padded to 64: ctx then holds head h's dh_out columns at
 * h * dh_out, rows at pitch ld_ctx (0, 0 = 64, H * 64) */
int rp_xl_attn_fwd_pv(const void* qu, const void* qv, const void* kh, const void* vh, const void* rh, void* probs,
                      int64_t ld_p, void* ctx, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t mem_len,
                      float scale, int32_t dh_out, int64_t ld_ctx, void* stream);
/* Fused backward of rp_xl_attn_fwd's softmax (bf16, dh = 64, tcgen05): dP = g_ctx_h v^T on the tensor
 * cores, D_i = <g_ctx_i, ctx_i> from the merged [B*T, H*dh] rows, dAC = P (dP - D) * scale and the
 * un-shifted dBD, both [H*B, T, ld_p]; replaces the dP GEMM + rp_xl_softmax_bwd */
int rp_xl_attn_bwd(const void* grad_ctx_h, const void* vh, const void* probs, void* grad_ac, void* grad_bd, int64_t ld_p,
                   const void* grad_ctx, const void* ctx, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh,
                   int64_t mem_len, float scale, void* stream);
/* rp_xl_attn_bwd plus the query gradients on the tensor cores (dh = 64, T % 128 == 0):
 * grad_qu = dAC kh and grad_qv = dBD r_h, fp32 [H*B*T, dh] -- the two head-dim-wide GEMMs
 * over the dAC / dBD matrices are folded into the kernel (dS stays in shared memory).
 * grad_ac NULL: dAC is not written (rp_xl_attn_bwd_kv forms the key gradient itself);
 * d_rows (or NULL): D_i = <g_ctx_i, ctx_i> per query row, fp32 [H*B*T], for rp_xl_attn_bwd_kv.
 * grad_qkv (or NULL; with grad_ac NULL and d_rows): bf16(grad_qu + grad_qv) goes straight into the
 * query columns of the merged bf16 g_qkv rows ([B*M memory rows; B*T current rows] x 3*H*dh, the
 * layout rp_xl_merge_grads writes) instead of grad_qu / grad_qv, which may then be NULL */
int rp_xl_attn_bwd_dq(const void* grad_ctx_h, const void* vh, const void* kh, const void* rh, const void* probs,
                      void* grad_ac, void* grad_bd, int64_t ld_p, const void* grad_ctx, const void* ctx, float* grad_qu,
                      float* grad_qv, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t mem_len,
                      float scale, float* bias_part, float* d_rows, void* grad_qkv, void* stream);
/* Key-major key / value gradients (bf16, dh = 64, T % 128 == 0; after rp_xl_attn_bwd_dq with
 * d_rows): one CTA per (head*batch, 128-key tile) recomputes dP = g_ctx_h v^T and dS on the
 * tensor cores and accumulates grad_vh = P^T g_ctx_h and grad_kh = dS^T qu in TMEM, written as
 * bf16 [H*B, M+T, dh] -- bitwise the banded GEMMs over P and dAC it replaces (kernels.bmm,
 * kernels.py:68-81, on the XL score matrices), without the dAC matrix.  grad_qkv (or NULL): dK and
 * dV go straight into the key / value columns of the merged g_qkv rows (as rp_xl_attn_bwd_dq), and
 * the memory rows' query columns are zeroed -- with rp_xl_attn_bwd_dq's grad_qkv this replaces
 * rp_xl_merge_grads; grad_kh / grad_vh may then be NULL */
/* 1 when rp_xl_attn_bwd_dq runs its persistent kernel for the no-dAC path (RP_XL_DQ_PERSIST != 0),
 * the one that takes grad_qkv */
int rp_xl_dq_persistent(void);
int rp_xl_attn_bwd_kv(const void* grad_ctx_h, const void* vh, const void* qu, const void* probs, int64_t ld_p,
                      const float* d_rows, void* grad_kh, void* grad_vh, int64_t B, int64_t T, int64_t M, int32_t H,
                      int32_t dh, int64_t mem_len, float scale, void* grad_qkv, void* stream);
/* bias_part of rp_xl_attn_bwd_dq (or NULL): per-CTA column sums of grad_qu / grad_qv, which
 * rp_xl_dq_bias_finish turns into the r_w_bias / r_r_bias gradients ([H, 64] each) without
 * re-reading the query gradients (the column sums of rp_xl_bias_grad) */
int64_t rp_xl_dq_bias_part_bytes(int32_t H, int64_t B, int64_t T);
int rp_xl_dq_bias_finish(const float* bias_part, float* g_r_w_bias, float* g_r_r_bias, int32_t H, int64_t B, int64_t T,
                         void* stream);
/* dAC = P (dP - <dP,P>) * scale; dBD = the same values un-shifted */
int rp_xl_softmax_bwd(int32_t dtype, const float* grad_p, int64_t ld_scores, const void* probs, int64_t ld_p,
                      void* grad_ac, void* grad_bd, int64_t rows, int64_t T, int64_t M, int64_t mem_len, float scale,
                      void* stream);
/* per-head column sums of dQu / dQv [H, R, dh] -> d r_w_bias, d r_r_bias [H, dh] (deterministic) */
int64_t rp_xl_bias_grad_workspace_bytes(int32_t H, int32_t dh);

/* ---- adaptive tied softmax head (oracle/adaptive.py; BASELINE configs[3]) ----
 * The contractions run on rp_gemm (RP_EPI_LSE_PARTIAL / RP_EPI_CE_GRAD); these move rows.
 * rows_copy: dst[r, :cols] = src[r, :cols]; with aug, dst[r, cols] = val ? val[r] : val_const;
 *            zeros up to ld_dst (builds [h | 1] and [V_head ; W_c | b_c]).
 * rows_gather: dst[r] = src[idx[r]].  rows_scatter_add (fp32): dst[idx[r]] += src[r], rows unique. */
int rp_rows_copy(int32_t src_dtype, const void* src, int64_t ld_src, int64_t rows, int64_t cols, const float* val,
                 float val_const, int32_t aug, int32_t dst_dtype, void* dst, int64_t ld_dst, void* stream);
int rp_rows_gather(int32_t dtype, const void* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols,
                   void* dst, int64_t ld_dst, void* stream);
int rp_rows_scatter_add(const float* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols, float* dst,
                        int64_t ld_dst, void* stream);
/* u / v gradients: column sums of dQu / dQv [H, R, dh] (row pitch ld_g; 0 = dh) */
int rp_xl_bias_grad(const float* g_qu, const float* g_qv, float* workspace, float* g_r_w_bias, float* g_r_r_bias,
                    int32_t H, int64_t R, int32_t dh, int64_t ld_g, void* stream);

/* ---- embedding (layers.py:114-136) ---------------------------------------- */
int rp_embed_fwd(int32_t dtype, const int64_t* tokens, const void* tied, const void* pos, void* out, int64_t B,
                 int64_t T, int64_t d, int64_t vocab, uint64_t seed, uint64_t threshold, float scale,
                 int32_t drop_enabled, int32_t* flag, int64_t ld, void* stream);
/* grad_pos [Tmax,d] (fully written); emb[tok] += beta * sum of masked rows (deterministic
 * sorted, chunked scatter; replaces np.add.at, layers.py:135).  Ids outside [0, vocab)
 * are skipped (rp_embed_fwd already raised RP_FLAG_DIMENSION for them; the reference
 * raises DimensionError, layers.py:116-117).
 * workspace: rp_embed_bwd_workspace_bytes(B*T, d) bytes. */
int rp_embed_bwd(const float* grad, const int64_t* tokens, int64_t B, int64_t T, int64_t Tmax, int64_t d,
                 int64_t vocab, uint64_t seed, uint64_t threshold, float scale, int32_t drop_enabled, float* grad_pos,
                 float* emb_grad, float beta, void* workspace, int64_t ld_out, void* stream);
int64_t rp_embed_bwd_workspace_bytes(int64_t n_tokens, int64_t d);

/* ---- tied-head cross-entropy finish (layers.py:287-296, 310-316) ------------ */
int rp_ce_finish(const float* partial, int32_t ntiles, const float* target_logit, const int64_t* targets,
                 int64_t vocab, int64_t rows, float* lse, float* loss_rows, float* loss, double* loss64,
                 int32_t* flag, void* stream);

/* ---- optimizers over flat fp32 master buffers (optim.py:52-126) ------------- */
/* copy (compute dtype) receives the updated weights: the next snapshot-ring slot. */
int rp_adam_step(float* w, const float* g, float* m, float* v, void* copy, int32_t copy_dtype, int64_t n, float lr,
                 float beta1, float beta2, float eps, float bias_corr1, float bias_corr2, int32_t* flag,
                 void* stream);
int rp_sgd_step(float* w, const float* g, void* copy, int32_t copy_dtype, int64_t n, float lr, int32_t* flag,
                void* stream);

/* ---- mixed tied gradient (engine.py:54-69) ---------------------------------
 * out = 1/2 vo + 1/2 vi (convention 0, "half_avg") or vo + vi (1, "sum");
 * zeros while t-K+1 < 0 (vi must then be NULL: RP_ERR_SCHEDULE otherwise, and
 * when it is missing later).  The engines fuse this into the head / embedding
 * backward epilogues; this is the standalone form of the reference function. */
int rp_embedding_gradient(int64_t t, int64_t K, const float* vo, const float* vi, float* out, int64_t n,
                          int32_t convention, void* stream);

/* ---- misc ----------------------------------------------------------------- */
/* uniform_signed init from the reference stream (tensor.py:72-74), fp64 math, fp32 out */
int rp_init_uniform(float* out, int64_t n, uint64_t seed, uint64_t pos0, double scale, void* stream);
int rp_cast(const void* in, int32_t in_dtype, void* out, int32_t out_dtype, int64_t n, void* stream);
/* out (+)= sum x^2 in fp64; part: >= 296 doubles of scratch (engine.py:72-80) */
int rp_sq_norm(const float* x, int64_t n, double* part, double* out, int32_t accumulate, void* stream);


/* ---- layer-level entry points: the reference layer protocol ------------------
 * TransformerBlockLayer.forward/backward (layers.py:168-253) and the projection
 * layer + loss_and_head_backward (layers.py:268-322) as single native calls. */
typedef struct rp_block_desc {
  int64_t B, T, d, f;
  int32_t dtype;        /* rp_dtype of activations and matrix weights */
  int32_t drop_enabled; /* train && p > 0 */
  uint64_t drop_seed;   /* mix64(dropout_seed, step, layer), model.py:218-219 */
  uint64_t drop_threshold;
  float drop_scale;
  int32_t max_ctas; /* SM budget for every GEMM of the layer (0 = whole GPU) */
  /* Rows (B*T) of the whole batch when this call is one row block of it (the
   * micro-batched relay, paper_1909_06695_b200/distributed.py); 0 = B*T.  The
   * second dropout mask then starts at drop_rows_total*d (layers.py:209-212);
   * the block's own row offset r0 is folded into drop_seed by the caller:
   * seed + r0*d*0x9E3779B97F4A7C15 addresses positions r0*d + i (tensor.py:41-48). */
  int64_t drop_rows_total;
  /* FFN activation: 0 = ReLU (the reference, layers.py:191), 1 = GELU (exact
   * erf form, a production option): the tape then also keeps z1 */
  int32_t activation;
} rp_block_desc;

typedef struct rp_block_weights {
  const void* wqkv; /* [d, 3d] = [wq | wk | wv] (dtype) */
  const void* wo;   /* [d, d] */
  const void* w1;   /* [d, f] */
  const void* w2;   /* [f, d] */
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b, *b1, *b2;
} rp_block_weights;

/* forward intermediates kept in a stale slot ("store-all"; the reference
 * recomputes them, model.py:250-268, and proves the two bitwise equal) */
typedef struct rp_block_tape {
  void *a, *qkv, *probs, *ctx, *x1, *m, *h1; /* probs: [B, T, pad8(T)] */
  float *mean1, *rstd1, *mean2, *rstd2;
  void* z1; /* [B*T, f] FFN pre-activation (GELU only; NULL for ReLU) */
} rp_block_tape;

typedef struct rp_block_grads {
  float *wqkv, *wo, *w1, *w2, *ln1_g, *ln1_b, *ln2_g, *ln2_b, *b1, *b2;
} rp_block_grads;

int64_t rp_block_workspace_bytes(const rp_block_desc* desc);
int rp_block_forward(const rp_block_desc* desc, const rp_block_weights* w, const void* x, void* out,
                     const rp_block_tape* tape, void* workspace, int64_t workspace_bytes, int32_t* flag,
                     void* stream);
/* g_x = dL/dx (fp32) from g_out = dL/dout (fp32); parameter grads (fp32) overwritten */
int rp_block_backward(const rp_block_desc* desc, const rp_block_weights* w, const void* x, const rp_block_tape* tape,
                      const float* g_out, float* g_x, const rp_block_grads* grads, void* workspace,
                      int64_t workspace_bytes, void* stream);

typedef struct rp_head_desc {
  int64_t rows, d, vocab;
  int32_t dtype;
  /* rows of the whole batch when this call is one row block of it: the
   * cross-entropy gradient is scaled by 1/rows_total (layers.py:319); 0 = rows */
  int64_t rows_total;
} rp_head_desc;

int64_t rp_head_workspace_bytes(const rp_head_desc* desc);
/* mean CE of x @ tied^T vs targets without materialising logits; lse kept for backward */
int rp_head_forward(const rp_head_desc* desc, const void* x, const void* tied, const int64_t* targets, float* lse,
                    float* loss, double* loss64, void* workspace, int64_t workspace_bytes, int32_t* flag,
                    void* stream);
/* g_x = dL/dx (fp32); vo (if non-NULL) = vo_alpha * dL/dtied from the output side
 * (the fresh half of the mixed tied gradient, engine.py:54-69), or vo += that when
 * vo_accumulate (the input-side half may already be there: 0 + a + b == 0 + b + a) */
int rp_head_backward(const rp_head_desc* desc, const void* x, const void* tied, const int64_t* targets,
                     const float* lse, float* g_x, float* vo, float vo_alpha, int32_t vo_accumulate,
                     void* workspace, int64_t workspace_bytes, void* stream);

/* ---- module-level entry points: ModuleState.forward / recompute_backward -----
 * (model.py:224-304).  One call runs a module's contiguous layer slice --
 * optional embedding, n_blocks transformer blocks, optional projection + loss
 * -- over caller-owned weights (the ring snapshot of the slot's step) and the
 * slot's device storage.  The host keeps the schedule bookkeeping (rings,
 * slot queue, boundary hand-off), exactly as the reference keeps it in
 * ModuleState / PipelineEngine. */
/* ---- Transformer-XL block composite (paper_1909_06695_b200/xl.py; restated in
 * oracle/xl.py -- the reference has no XL path): relative-position multi-head
 * attention over [memory; segment] inside the reference's pre-LN block, the
 * same kernels in the same order as the Python host loop (bitwise equal).
 * The host fills tape.xa = [memory rows; current rows] before the forward
 * (the memory is the previous segment's layer input, stop-gradient). */
#define RP_XL_FUSED_FWD 1 /* rp_xl_attn_fwd (bf16, dh 64 / 128) */
#define RP_XL_FUSED_BWD 2 /* rp_xl_attn_bwd (bf16, dh 64 / 128, T % 8 == 0) */
#define RP_XL_FUSED_PV 4  /* rp_xl_attn_fwd_pv (bf16, dh 64) */
#define RP_XL_FUSED_DQ 8  /* rp_xl_attn_bwd_dq (bf16, dh 64, T % 128 == 0) */
#define RP_XL_BANDED 16   /* dK / dV GEMMs skip the causal window's all-zero query blocks (bitwise the dense result) */
#define RP_XL_FUSED_KV 32 /* rp_xl_attn_bwd_kv after rp_xl_attn_bwd_dq (no dAC; needs RP_XL_FUSED_DQ) */
typedef struct rp_xl_block_desc {
  int64_t B, T, M, d, f;
  int32_t H, dtype;
  int32_t drop_enabled, activation, max_ctas;
  int32_t mem_len;    /* valid memory rows (M - mem_len leading keys are masked) */
  uint64_t drop_seed, drop_threshold;
  float drop_scale;
  int64_t drop_rows_total;
  int64_t ldk;        /* row pitch of the probabilities: pad8(M + T) */
  int32_t fused;      /* RP_XL_FUSED_* (0: the unfused GEMM + softmax path, also the fp32 check mode) */
  int32_t score_tile; /* N tile of the unfused score GEMMs (0: default) */
} rp_xl_block_desc;
typedef struct rp_xl_block_weights {
  const void *wqkv, *wo, *w1, *w2, *wr; /* matrices (dtype); wr [d, d] projects the sinusoid R */
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b, *b1, *b2, *r_w_bias, *r_r_bias; /* u, v: [H, dh] */
} rp_xl_block_weights;
typedef struct rp_xl_block_tape {
  void *xa, *a, *qkv, *qu, *qv, *kh, *vh, *rh, *probs, *ctx, *x1, *m, *h1, *z1;
  float *mean1, *rstd1, *mean2, *rstd2;
} rp_xl_block_tape;
typedef struct rp_xl_block_grads {
  float *wqkv, *wo, *w1, *w2, *wr, *ln1_g, *ln1_b, *ln2_g, *ln2_b, *b1, *b2, *r_w_bias, *r_r_bias;
} rp_xl_block_grads;
int64_t rp_xl_block_workspace_bytes(const rp_xl_block_desc* desc);
/* R: the sinusoid relative encodings [M+T, d] (dtype); out: [B*T, d] */
int rp_xl_block_forward(const rp_xl_block_desc* desc, const rp_xl_block_weights* w, const void* R, void* out,
                        const rp_xl_block_tape* tape, void* workspace, int64_t workspace_bytes, int32_t* flag,
                        void* stream);
int rp_xl_block_backward(const rp_xl_block_desc* desc, const rp_xl_block_weights* w, const void* R,
                         const rp_xl_block_tape* tape, const float* g_out, float* g_x, const rp_xl_block_grads* grads,
                         void* workspace, int64_t workspace_bytes, void* stream);

typedef struct rp_module_desc {
  int64_t B, T, d, f, vocab;
  int64_t t_max;            /* rows of the embedding position table */
  int32_t n_blocks, has_embedding, has_projection;
  int32_t dtype;            /* rp_dtype of activations / matrix weights */
  int32_t max_ctas;         /* SM budget of every GEMM (0 = whole GPU) */
  int32_t drop_enabled;     /* train && p > 0 */
  uint64_t drop_threshold;  /* ceil(p * 2^53) */
  float drop_scale;         /* 1 / (1 - p) */
  const uint64_t* layer_seeds; /* host array, one per layer of the slice: mix64(dropout_seed, step, layer) */
  int32_t activation;       /* FFN activation of every block: 0 = ReLU, 1 = GELU (rp_block_desc) */
  /* Transformer-XL modules (n_heads > 0): every block is an XL block with M
   * memory rows, mem_len of them valid; xl_fused / score_tile as in
   * rp_xl_block_desc.  The host keeps the memory: it writes each block's
   * memory rows into its tape's xa before the forward. */
  int32_t n_heads, mem_len;
  int64_t M;
  int32_t xl_fused, score_tile;
} rp_module_desc;

typedef struct rp_module_weights {
  const rp_block_weights* blocks; /* host array [n_blocks] */
  const void* tied;               /* compute copy of the tied matrix [vocab, d] */
  const void* pos;                /* embedding position table [t_max, d] (dtype) */
  const rp_xl_block_weights* xl_blocks; /* host array [n_blocks] (XL modules) */
  const void* R;                  /* sinusoid relative encodings [M+T, d] (XL modules) */
} rp_module_weights;

/* one stale slot (model.py:162-168): acts[j] = input of block j (acts[0] is
 * written by the embedding or by the upstream module), acts[n_blocks] = head
 * input when has_projection */
typedef struct rp_module_slot {
  const int64_t* tokens;       /* [B, T] (embedding modules) */
  const int64_t* targets;      /* [B*T]  (projection modules) */
  void* const* acts;           /* host array [n_blocks + has_projection] of [B*T, d] (dtype) */
  const rp_block_tape* tapes;  /* host array [n_blocks] */
  float* lse;                  /* [B*T] head log-sum-exp (projection) */
  float* loss;                 /* 0-d mean cross entropy (projection) */
  double* loss64;
  const rp_xl_block_tape* xl_tapes; /* host array [n_blocks] (XL modules; acts[j] = the current rows of xa) */
} rp_module_slot;

typedef struct rp_module_grads {
  const rp_block_grads* blocks; /* host array [n_blocks], overwritten */
  float* pos;                   /* embedding position-table gradient, overwritten */
  float* tied;                  /* tied gradient [vocab, d] (fp32) or NULL */
  float tied_alpha;             /* output half: tied (+)= alpha * dV_out (skipped when 0) */
  float tied_beta;              /* input half:  tied  += beta * dV_in   (skipped when 0) */
  int32_t tied_accumulate;      /* 1: add the output half onto tied; 0: overwrite */
  const rp_xl_block_grads* xl_blocks; /* host array [n_blocks] (XL modules) */
} rp_module_grads;

int64_t rp_module_workspace_bytes(const rp_module_desc* desc);
/* forward at the given weights; `out` receives the last block's output when
 * the module has no projection (the downstream module's input buffer) */
int rp_module_forward(const rp_module_desc* desc, const rp_module_weights* w, const rp_module_slot* slot, void* out,
                      void* workspace, int64_t workspace_bytes, int32_t* flag, void* stream);
/* delayed backward from the slot's stored intermediates; g_out = boundary
 * gradient dL/d(output) (fp32, NULL for projection modules); g_in (may be
 * NULL) receives dL/d(input) for non-embedding modules */
int rp_module_backward(const rp_module_desc* desc, const rp_module_weights* w, const rp_module_slot* slot,
                       const float* g_out, float* g_in, const rp_module_grads* grads, void* workspace,
                       int64_t workspace_bytes, void* stream);

/* GELU (exact erf form): y = 0.5 z (1 + erf(z / sqrt 2)) over n elements of
 * `dtype`, vectorised (the FFN activation option; its gradient is the GEMM
 * epilogue RP_EPI_GELU_GRAD) */
int rp_gelu_fwd(int32_t dtype, const void* z, void* y, int64_t n, void* stream);

/* y += alpha * x over n fp32 elements (weight-gradient accumulation over the
 * row blocks of a micro-batched slot, in a fixed order) */
int rp_axpy(float* y, const float* x, float alpha, int64_t n, void* stream);

/* ---- distributed context and point-to-point transfers ---------
 * The reference's module threads hand activations and boundary gradients over
 * by reference (engine.py:246-265, 313-373; ring placement model.py:137-140);
 * across GPUs these are NCCL send/recv over NVLink between the ranks of one
 * node.  NCCL is loaded at run time: RP_NCCL_LIB, else libnccl.so.2.
 * Every rank calls rp_ctx_create with the same 128-byte id (rank 0 draws it
 * with rp_nccl_unique_id and shares it out of band).  Transfers are
 * asynchronous on `stream`; ordering per peer pair follows issue order, so
 * every rank issues its relay hops in the global order k = 1..K-1 and its
 * boundary hops in the order k = K..2 (paper_1909_06695_b200/distributed.py).
 * A send and a receive that must progress together (including a transfer to
 * the same rank) go between rp_group_start / rp_group_end. */
typedef struct rp_ctx rp_ctx;
int rp_nccl_unique_id(void* id128);
int rp_ctx_create(int32_t device, const void* nccl_unique_id, int32_t rank, int32_t nranks, rp_ctx** out);
int rp_ctx_destroy(rp_ctx* ctx);
int rp_ctx_rank(const rp_ctx* ctx);
int rp_ctx_nranks(const rp_ctx* ctx);
/* activation relay module k -> k+1 / boundary gradient k -> k-1 (engine.py:224, 239-245) */
int rp_send(rp_ctx* ctx, const void* buf, int64_t bytes, int32_t peer, void* stream);
int rp_recv(rp_ctx* ctx, void* buf, int64_t bytes, int32_t peer, void* stream);
int rp_group_start(void);
int rp_group_end(void);

/* ---- state export / import (checkpoint of the device state) ------------------
 * The reference checkpoints weights, optimizer moments, snapshot rings, pending
 * slots and boundary gradients under fixed names (runner.py:111-226) in the
 * RPCK container (checkpoint.py:1-70).  A C host describes the buffers it
 * owns (device or host) and exports them into / imports them from that
 * container in memory; fp32 / bf16 widen to f8 exactly, so an export ->
 * import round trip is bit-exact, and the Python host's and the reference's
 * loaders read the result. */
typedef struct rp_state_entry {
  const char* name;   /* entry name, e.g. "stack.L3.wq", "m2.ring.7.L3.w1", "boundary.1" */
  void* ptr;          /* the buffer (contiguous) */
  int32_t dtype;      /* rp_dtype */
  int32_t on_host;    /* 1: ptr is host memory; 0: device memory */
  int32_t ndim;       /* <= 4 */
  int64_t shape[4];
} rp_state_entry;
/* bytes of the container holding `entries` (-1 on a malformed entry) */
int64_t rp_state_bytes(const rp_state_entry* entries, int32_t n);
/* device/host buffers -> container in host memory `blob` (synchronous on stream) */
int rp_export_state(const rp_state_entry* entries, int32_t n, void* blob, int64_t blob_bytes, void* stream);
/* container -> the named buffers (by name; element counts must match) */
int rp_import_state(const rp_state_entry* entries, int32_t n, const void* blob, int64_t blob_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RINGPIPE_B200_H */
