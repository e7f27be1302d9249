// Internal declarations shared by the ringpipe-b200 translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ringpipe_b200.h"

#include <mutex>

namespace rp {

// Function attributes (e.g. the dynamic shared-memory opt-in) are per device:
// returns true the first time a call site asks on the current device.  `done`
// is a per-call-site bitmask of devices (a static at the call site).
inline bool first_on_device(uint64_t& done) {
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  if (done & bit) return false;
  done |= bit;
  return true;
}

// Records a formatted error message (thread-local) and returns `status`.
int set_error(int status, const char* fmt, ...);
// Returns RP_OK or RP_ERR_CUDA with the launch error recorded.
int check_launch(const char* what);

int gemm(const rp_gemm_args& a, cudaStream_t stream);
// 3-d bf16 TMA map (128B swizzle): dims {inner, rows, batch}; OOB reads fill zeros
int tma_map_bf16(CUtensorMap* map, const void* ptr, int64_t inner, int64_t rows, int64_t ld, int64_t batch,
                 int64_t bstride, int box_inner, int box_rows, bool swizzle = true);
// 3-d bf16 map {inner, rows, batch} for 32 x 32 TMA store tiles staged with the 64B swizzle
int tma_map_bf16_store32(CUtensorMap* map, const void* ptr, int64_t inner, int64_t rows, int64_t ld, int64_t batch);
int gemm_tile_n(int64_t M, int64_t N, int64_t batch);
// split count for an fp32 store GEMM of `batch` matrices (layers.cpp choose_splits); 1 = no split
int gemm_choose_splits(int64_t M, int64_t N, int64_t K, int64_t cap_bytes, int64_t batch = 1);
int splitk_reduce(const float* part, int S, int64_t M, int64_t N, float* out, int64_t ldo, cudaStream_t st);
int tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
               cudaStream_t stream);

// ldx / ldy / ldm / ldo: row pitches in elements (0 = d); a pitch wider than d
// (d not a multiple of 8: bf16 rows padded to 16 bytes) takes the scalar kernels
int layernorm_fwd(int dtype, const void* x, const float* g, const float* b, void* y, float* mean, float* rstd,
                  int64_t rows, int64_t d, int32_t* flag, cudaStream_t st, int64_t ldx = 0, int64_t ldy = 0);
int layernorm_bwd(int dtype, const float* dy, const void* x, const float* mean, const float* rstd, const float* g,
                  const float* resid_grad, float* dx, void* dx_masked, uint64_t seed, uint64_t thr, float scale,
                  int drop_on, float* part_g, float* part_b, int64_t rows, int64_t d, cudaStream_t st,
                  int64_t ldx = 0, int64_t ldm = 0);
int ln_bwd_blocks(int64_t rows);
int colsum_blocks(int64_t rows);
int mask_grad_blocks(int64_t rows, int64_t d);
int colsum_partial(int dtype, const void* x, int64_t rows, int64_t cols, int64_t ld, float* part, cudaStream_t st);
int colsum_finish(const float* part, int nblk, int64_t cols, float* out, cudaStream_t st);
struct ColsumJob {
  const float* part;
  int nblk;
  int64_t cols;
  float* out;
};
constexpr int kMaxColsumJobs = 8;
struct ColsumJobs {
  ColsumJob job[kMaxColsumJobs];
  int first_block[kMaxColsumJobs];
  int n;
};
// up to kMaxColsumJobs colsum_finish operations in one launch (bitwise equal)
int colsum_finish_multi(const ColsumJob* jobs, int n, cudaStream_t st);
int mask_grad(int dtype, const float* g, void* out, int64_t rows, int64_t d, uint64_t seed, uint64_t pos0,
              uint64_t thr, float scale, int drop_on, float* part, cudaStream_t st, int64_t ldo = 0);
int mask_grad_blocks_ld(int64_t rows, int64_t d, int64_t ldo);
int softmax_causal(int dtype, const float* s, void* p, int64_t rows, int64_t Tn, int64_t ld, cudaStream_t st);
int softmax_bwd(int dtype, const float* gp, const void* p, void* gs, float scale, int64_t rows, int64_t Tn,
                int64_t ld, cudaStream_t st);
// ld: row pitch of V, pos and out (0 = d)
int embed_fwd(int dtype, const int64_t* tok, const void* V, const void* pos, void* out, int64_t B, int64_t Tn,
              int64_t d, int64_t vocab, uint64_t seed, uint64_t thr, float scale, int drop_on, int32_t* flag,
              cudaStream_t st, int64_t ld = 0);
int64_t embed_bwd_workspace_bytes(int64_t n_tokens, int64_t d);
int embed_bwd(const float* g, const int64_t* tok, int64_t B, int64_t Tn, int64_t Tmax, int64_t d, int64_t vocab,
              uint64_t seed,
              uint64_t thr, float scale, int drop_on, float* gpos, float* emb, float beta, void* workspace,
              cudaStream_t st, int64_t ld_out = 0);  // ld_out: row pitch of gpos and emb
int ce_finish(const float* partial, int ntiles, const float* zy, const int64_t* tgt, int64_t vocab, int64_t rows,
              float* lse, float* loss_rows, float* loss, double* loss64, int32_t* flag, cudaStream_t st);
int adam_step(float* w, const float* g, float* m, float* v, void* copy, int copy_dtype, int64_t n, float lr, float b1,
              float b2, float eps, float c1, float c2, int32_t* flag, cudaStream_t st);
int sgd_step(float* w, const float* g, void* copy, int copy_dtype, int64_t n, float lr, int32_t* flag,
             cudaStream_t st);
int init_uniform(float* out, int64_t n, uint64_t seed, uint64_t pos0, double scale, cudaStream_t st);
int embedding_gradient(int64_t t, int64_t K, const float* vo, const float* vi, float* out, int64_t n,
                       int convention, cudaStream_t st);
int cast(const void* in, int in_dtype, void* out, int out_dtype, int64_t n, cudaStream_t st);
int axpy(float* y, const float* x, float alpha, int64_t n, cudaStream_t st);
int gelu_fwd(int dtype, const void* z, void* y, int64_t n, cudaStream_t st);
int sq_norm(const float* x, int64_t n, double* part, double* out, int accumulate, cudaStream_t st);

// ldq: row pitch of qkv / g_qkv (0 = 3*H*dh); ldh: row pitch of the
// head-major [H, rows, dh] tensors (0 = dh)
int xl_split_qkv(int dtype, const void* qkv, const float* u, const float* v, void* qu, void* qv, void* kh, void* vh,
                 int64_t B, int64_t Tn, int64_t M, int H, int dh, cudaStream_t st, int64_t ldq = 0, int64_t ldh = 0);
int xl_split_heads(int src_dtype, const void* src, int64_t ld, int dst_dtype, void* dst, int64_t rows, int H, int dh,
                   cudaStream_t st, int64_t ldh = 0);
int xl_merge_heads(int src_dtype, const void* src, int dst_dtype, void* dst, int64_t ld, int64_t rows, int H, int dh,
                   cudaStream_t st, int64_t ldh = 0);
// gkh / gvh in the compute dtype (the dK / dV GEMMs store them rounded like g_qkv)
int xl_merge_grads(int dtype, const float* gqu, const float* gqv, const void* gkh, const void* gvh, void* gqkv,
                   int64_t B, int64_t Tn, int64_t M, int H, int dh, cudaStream_t st, int64_t ldq = 0,
                   int64_t ldg = 0, int64_t ldkv = 0);
int xl_softmax_fwd(int dtype, const float* ac, const float* bd, int64_t lds, void* p, int64_t ldp, int64_t rows,
                   int64_t Tn, int64_t M, int64_t mem_len, float scale, cudaStream_t st);
int xl_softmax_bwd(int dtype, const float* gp, int64_t lds, const void* p, int64_t ldp, void* gac, void* gbd,
                   int64_t rows, int64_t Tn, int64_t M, int64_t mem_len, float scale, cudaStream_t st);
// fused XL scores + softmax (xl_attn.cu): bf16, dh = 64
int xl_attn_fwd(const void* qu, const void* qv, const void* kh, const void* rh, void* probs, int64_t ldp, int64_t B,
                int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale, cudaStream_t st);
int xl_attn_bwd(const void* gctx_h, const void* vh, const void* probs, void* gac, void* gbd, int64_t ldp,
                const void* gctx, const void* ctx, int64_t B, int64_t Tn, int64_t M, int H, int dh, int mem_len,
                float scale, cudaStream_t st);
// fused forward with P.V (operands dh = 64; a smaller model head dim dh_out
// rides zero-padded to 64): also ctx (merged rows, head h at h * dh_out, pitch ld_ctx) = P v
int xl_attn_fwd_pv(const void* qu, const void* qv, const void* kh, const void* vh, const void* rh, void* probs,
                   int64_t ldp, void* ctx, int64_t B, int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale,
                   cudaStream_t st, int dh_out = 0, int64_t ld_ctx = 0);
// fused backward with the query gradients on the tensor cores (dh = 64, T % 128 == 0):
// also gqu = dAC K, gqv = dBD R as fp32 [H*B*T, 64]
// bias_part (optional, xl_dq_bias_part_bytes): per-CTA column sums of gqu / gqv, finished
// into the r_w_bias / r_r_bias gradients by xl_dq_bias_finish (no re-read of gqu / gqv)
int xl_attn_bwd_dq(const void* gctx_h, const void* vh, const void* kh, const void* rh, const void* probs, void* gac,
                   void* gbd, int64_t ldp, const void* gctx, const void* ctx, float* gqu, float* gqv, int64_t B,
                   int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale, cudaStream_t st,
                   float* bias_part = nullptr, float* d_rows = nullptr, void* gqkv = nullptr);
bool xl_dq_persistent();  // RP_XL_DQ_PERSIST (default on): the no-dAC bwd_dq runs the persistent kernel
// key-major dK / dV (dh = 64, T % 128 == 0) from P, g_ctx_h, v, q+u and xl_attn_bwd_dq's D
// rows: gk = dS^T (q+u), gv = P^T g_ctx_h as bf16 [H*B, Kl, 64] -- bitwise the banded GEMMs
// over dAC and P, so xl_attn_bwd_dq can skip dAC (gac = NULL)
int xl_attn_bwd_kv(const void* gctx_h, const void* vh, const void* qu, const void* probs, int64_t ldp,
                   const float* d_rows, void* gk, void* gv, int64_t B, int64_t Tn, int64_t M, int H, int dh, int mem_len,
                   float scale, cudaStream_t st, void* gqkv = nullptr);
int64_t xl_dq_bias_part_bytes(int H, int64_t B, int64_t Tn);
int xl_dq_bias_finish(const float* part, float* gu, float* gv, int H, int64_t B, int64_t Tn, cudaStream_t st);
// adaptive softmax row movers (adaptive.cu)
int rows_copy(int src_dtype, const void* src, int64_t ld_src, int64_t rows, int64_t cols, const float* val,
              float val_const, int aug, int dst_dtype, void* dst, int64_t ld_dst, cudaStream_t st);
int rows_gather(int dtype, const void* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols, void* dst,
                int64_t ld_dst, cudaStream_t st);
int rows_scatter_add(const float* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols, float* dst,
                     int64_t ld_dst, cudaStream_t st);
int64_t xl_bias_grad_workspace_bytes(int H, int dh);
int xl_bias_grad(const float* gqu, const float* gqv, float* part, float* gu, float* gv, int H, int64_t R, int dh,
                 cudaStream_t st, int64_t ldg = 0);

int64_t block_workspace_bytes(const rp_block_desc& d);
int block_forward(const rp_block_desc& d, const rp_block_weights& w, const void* x, void* out, const rp_block_tape& tp,
                  void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st);
int block_backward(const rp_block_desc& d, const rp_block_weights& w, const void* x, const rp_block_tape& tp,
                   const float* g_out, float* g_x, const rp_block_grads& G, void* ws, int64_t ws_bytes,
                   cudaStream_t st);
int64_t head_workspace_bytes(const rp_head_desc& h);
int head_forward(const rp_head_desc& h, const void* x, const void* tied, const int64_t* targets, float* lse,
                 float* loss, double* loss64, void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st);
int head_backward(const rp_head_desc& h, const void* x, const void* tied, const int64_t* targets, const float* lse,
                  float* g_x, float* vo, float vo_alpha, int vo_accumulate, void* ws, int64_t ws_bytes,
                  cudaStream_t st);

int64_t xl_block_workspace_bytes(const rp_xl_block_desc& d);
int xl_block_forward(const rp_xl_block_desc& d, const rp_xl_block_weights& w, const void* R, void* out,
                     const rp_xl_block_tape& tp, void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st);
int xl_block_backward(const rp_xl_block_desc& d, const rp_xl_block_weights& w, const void* R,
                      const rp_xl_block_tape& tp, const float* g_out, float* g_x, const rp_xl_block_grads& G,
                      void* ws, int64_t ws_bytes, cudaStream_t st);

int64_t module_workspace_bytes(const rp_module_desc& m);
int module_forward(const rp_module_desc& m, const rp_module_weights& w, const rp_module_slot& s, void* out,
                   void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st);
int module_backward(const rp_module_desc& m, const rp_module_weights& w, const rp_module_slot& s, const float* g_out,
                    float* g_in, const rp_module_grads& G, void* ws, int64_t ws_bytes, cudaStream_t st);

}  // namespace rp
