// extern "C" entry points of libringpipe_b200.so (declared in include/ringpipe_b200.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "rp_internal.h"

namespace rp {

static thread_local char g_err[1024] = "";

int set_error(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(RP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return RP_OK;
}

}  // namespace rp

extern "C" {

const char* rp_version(void) { return "ringpipe-b200 0.1.0 (sm_100a)"; }

int rp_last_error(char* buf, size_t len) {
  if (buf && len) {
    strncpy(buf, rp::g_err, len - 1);
    buf[len - 1] = 0;
  }
  return (int)strlen(rp::g_err);
}

int rp_gemm(const rp_gemm_args* args, void* stream) {
  if (!args) return rp::set_error(RP_ERR_INVALID, "rp_gemm: null args");
  return rp::gemm(*args, static_cast<cudaStream_t>(stream));
}

int rp_gemm_tile_n(int64_t M, int64_t N, int64_t batch) { return rp::gemm_tile_n(M, N, batch); }

int rp_gemm_choose_splits(int64_t M, int64_t N, int64_t K, int64_t batch, int64_t cap_bytes) {
  return rp::gemm_choose_splits(M, N, K, cap_bytes, batch);
}

int rp_splitk_reduce(const float* part, int32_t splits, int64_t M, int64_t N, float* out, int64_t ldo, void* stream) {
  return rp::splitk_reduce(part, splits, M, N, out, ldo, static_cast<cudaStream_t>(stream));
}

int rp_tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
                  void* stream) {
  return rp::tf32_split(x, hi, lo, rows, cols, ld_src, ld_dst, static_cast<cudaStream_t>(stream));
}

#define RP_S(s) static_cast<cudaStream_t>(s)

int rp_layernorm_fwd(int32_t dtype, const void* x, const float* gain, const float* bias, void* y, float* mean,
                     float* rstd, int64_t rows, int64_t d, int64_t ld_x, int64_t ld_y, int32_t* flag, void* stream) {
  return rp::layernorm_fwd(dtype, x, gain, bias, y, mean, rstd, rows, d, flag, RP_S(stream), ld_x, ld_y);
}
int rp_layernorm_bwd(int32_t dtype, const float* dy, const void* x, const float* mean, const float* rstd,
                     const float* gain, const float* resid_grad, float* dx, void* dx_masked, uint64_t seed,
                     uint64_t threshold, float scale, int32_t drop_enabled, float* partial_gain,
                     float* partial_bias, int64_t rows, int64_t d, int64_t ld_x, int64_t ld_masked, void* stream) {
  return rp::layernorm_bwd(dtype, dy, x, mean, rstd, gain, resid_grad, dx, dx_masked, seed, threshold, scale,
                           drop_enabled, partial_gain, partial_bias, rows, d, RP_S(stream), ld_x, ld_masked);
}
int rp_layernorm_bwd_blocks(int64_t rows) { return rp::ln_bwd_blocks(rows); }
int rp_colsum_blocks(int64_t rows) { return rp::colsum_blocks(rows); }
int rp_mask_grad_blocks(int64_t rows, int64_t d) { return rp::mask_grad_blocks(rows, d); }
int rp_mask_grad_blocks_ld(int64_t rows, int64_t d, int64_t ld_out) { return rp::mask_grad_blocks_ld(rows, d, ld_out); }
int rp_colsum_partial(int32_t dtype, const void* x, int64_t rows, int64_t cols, int64_t ld, float* partial,
                      void* stream) {
  return rp::colsum_partial(dtype, x, rows, cols, ld, partial, RP_S(stream));
}
int rp_colsum_finish(const float* partial, int32_t nblocks, int64_t cols, float* out, void* stream) {
  return rp::colsum_finish(partial, nblocks, cols, out, RP_S(stream));
}
int rp_colsum_finish_multi(const float* const* partials, const int32_t* nblocks, const int64_t* cols, float* const* outs,
                           int32_t n, void* stream) {
  if (n < 1 || n > rp::kMaxColsumJobs)
    return rp::set_error(RP_ERR_INVALID, "colsum_finish_multi: 1..%d jobs", rp::kMaxColsumJobs);
  rp::ColsumJob jobs[rp::kMaxColsumJobs];
  for (int i = 0; i < n; ++i) jobs[i] = rp::ColsumJob{partials[i], nblocks[i], cols[i], outs[i]};
  return rp::colsum_finish_multi(jobs, n, RP_S(stream));
}
int rp_mask_grad(int32_t dtype, const float* g, void* out, int64_t rows, int64_t d, uint64_t seed, uint64_t pos0,
                 uint64_t threshold, float scale, int32_t drop_enabled, float* partial, int64_t ld_out, void* stream) {
  return rp::mask_grad(dtype, g, out, rows, d, seed, pos0, threshold, scale, drop_enabled, partial, RP_S(stream),
                       ld_out);
}
int rp_softmax_causal(int32_t dtype, const float* scores, void* probs, int64_t rows, int64_t T, int64_t ld,
                      void* stream) {
  return rp::softmax_causal(dtype, scores, probs, rows, T, ld, RP_S(stream));
}
int rp_softmax_bwd(int32_t dtype, const float* grad_probs, const void* probs, void* grad_scores, float scale,
                   int64_t rows, int64_t T, int64_t ld, void* stream) {
  return rp::softmax_bwd(dtype, grad_probs, probs, grad_scores, scale, rows, T, ld, RP_S(stream));
}
int rp_embed_fwd(int32_t dtype, const int64_t* tokens, const void* tied, const void* pos, void* out, int64_t B,
                 int64_t T, int64_t d, int64_t vocab, uint64_t seed, uint64_t threshold, float scale,
                 int32_t drop_enabled, int32_t* flag, int64_t ld, void* stream) {
  return rp::embed_fwd(dtype, tokens, tied, pos, out, B, T, d, vocab, seed, threshold, scale, drop_enabled, flag,
                       RP_S(stream), ld);
}
int rp_embed_bwd(const float* grad, const int64_t* tokens, int64_t B, int64_t T, int64_t Tmax, int64_t d,
                 int64_t vocab, uint64_t seed, uint64_t threshold, float scale, int32_t drop_enabled, float* grad_pos,
                 float* emb_grad, float beta, void* work, int64_t ld_out, void* stream) {
  return rp::embed_bwd(grad, tokens, B, T, Tmax, d, vocab, seed, threshold, scale, drop_enabled, grad_pos, emb_grad, beta,
                       work, RP_S(stream), ld_out);
}
int64_t rp_embed_bwd_workspace_bytes(int64_t n_tokens, int64_t d) { return rp::embed_bwd_workspace_bytes(n_tokens, d); }
int rp_ce_finish(const float* partial, int32_t ntiles, const float* target_logit, const int64_t* targets,
                 int64_t vocab, int64_t rows, float* lse, float* loss_rows, float* loss, double* loss64,
                 int32_t* flag, void* stream) {
  return rp::ce_finish(partial, ntiles, target_logit, targets, vocab, rows, lse, loss_rows, loss, loss64, flag,
                       RP_S(stream));
}
int rp_adam_step(float* w, const float* g, float* m, float* v, void* copy, int32_t copy_dtype, int64_t n, float lr,
                 float beta1, float beta2, float eps, float bias_corr1, float bias_corr2, int32_t* flag,
                 void* stream) {
  return rp::adam_step(w, g, m, v, copy, copy_dtype, n, lr, beta1, beta2, eps, bias_corr1, bias_corr2, flag,
                       RP_S(stream));
}
int rp_sgd_step(float* w, const float* g, void* copy, int32_t copy_dtype, int64_t n, float lr, int32_t* flag,
                void* stream) {
  return rp::sgd_step(w, g, copy, copy_dtype, n, lr, flag, RP_S(stream));
}
int rp_init_uniform(float* out, int64_t n, uint64_t seed, uint64_t pos0, double scale, void* stream) {
  return rp::init_uniform(out, n, seed, pos0, scale, RP_S(stream));
}
int rp_embedding_gradient(int64_t t, int64_t K, const float* vo, const float* vi, float* out, int64_t n,
                          int32_t convention, void* stream) {
  return rp::embedding_gradient(t, K, vo, vi, out, n, convention, RP_S(stream));
}
int rp_gelu_fwd(int32_t dtype, const void* z, void* y, int64_t n, void* stream) {
  return rp::gelu_fwd(dtype, z, y, n, RP_S(stream));
}
int rp_axpy(float* y, const float* x, float alpha, int64_t n, void* stream) {
  return rp::axpy(y, x, alpha, n, RP_S(stream));
}
int rp_cast(const void* in, int32_t in_dtype, void* out, int32_t out_dtype, int64_t n, void* stream) {
  return rp::cast(in, in_dtype, out, out_dtype, n, RP_S(stream));
}
int rp_sq_norm(const float* x, int64_t n, double* part, double* out, int32_t accumulate, void* stream) {
  return rp::sq_norm(x, n, part, out, accumulate, RP_S(stream));
}

int rp_xl_split_qkv(int32_t dtype, const void* qkv, const float* r_w_bias, const float* r_r_bias, void* qu, void* qv,
                    void* kh, void* vh, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t ld_qkv,
                    int64_t ld_h, void* stream) {
  return rp::xl_split_qkv(dtype, qkv, r_w_bias, r_r_bias, qu, qv, kh, vh, B, T, M, H, dh, RP_S(stream), ld_qkv, ld_h);
}
int rp_xl_split_heads(int32_t src_dtype, const void* src, int64_t ld, int32_t dst_dtype, void* dst, int64_t rows,
                      int32_t H, int32_t dh, int64_t ld_h, void* stream) {
  return rp::xl_split_heads(src_dtype, src, ld, dst_dtype, dst, rows, H, dh, RP_S(stream), ld_h);
}
int rp_xl_merge_heads(int32_t src_dtype, const void* src, int32_t dst_dtype, void* dst, int64_t ld, int64_t rows,
                      int32_t H, int32_t dh, int64_t ld_h, void* stream) {
  return rp::xl_merge_heads(src_dtype, src, dst_dtype, dst, ld, rows, H, dh, RP_S(stream), ld_h);
}
int rp_xl_merge_grads(int32_t dtype, const float* g_qu, const float* g_qv, const void* g_kh, const void* g_vh,
                      void* g_qkv, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t ld_qkv,
                      int64_t ld_g, int64_t ld_kv, void* stream) {
  return rp::xl_merge_grads(dtype, g_qu, g_qv, g_kh, g_vh, g_qkv, B, T, M, H, dh, RP_S(stream), ld_qkv, ld_g, ld_kv);
}
int rp_xl_softmax_fwd(int32_t dtype, const float* ac, const float* bd, int64_t ld_scores, void* probs, int64_t ld_p,
                      int64_t rows, int64_t T, int64_t M, int64_t mem_len, float scale, void* stream) {
  return rp::xl_softmax_fwd(dtype, ac, bd, ld_scores, probs, ld_p, rows, T, M, mem_len, scale, RP_S(stream));
}
int rp_xl_attn_fwd(const void* qu, const void* qv, const void* kh, const void* rh, void* probs, int64_t ld_p, int64_t B,
                   int64_t T, int64_t M, int32_t H, int32_t dh, int64_t mem_len, float scale, void* stream) {
  return rp::xl_attn_fwd(qu, qv, kh, rh, probs, ld_p, B, T, M, H, dh, (int)mem_len, scale, RP_S(stream));
}
int rp_xl_attn_bwd(const void* grad_ctx_h, const void* vh, const void* probs, void* grad_ac, void* grad_bd, int64_t ld_p,
                   const void* grad_ctx, const void* ctx, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh,
                   int64_t mem_len, float scale, void* stream) {
  return rp::xl_attn_bwd(grad_ctx_h, vh, probs, grad_ac, grad_bd, ld_p, grad_ctx, ctx, B, T, M, H, dh, (int)mem_len,
                         scale, RP_S(stream));
}
int rp_xl_attn_fwd_pv(const void* qu, const void* qv, const void* kh, const void* vh, const void* rh, void* probs,
                      int64_t ld_p, void* ctx, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t mem_len,
                      float scale, int32_t dh_out, int64_t ld_ctx, void* stream) {
  return rp::xl_attn_fwd_pv(qu, qv, kh, vh, rh, probs, ld_p, ctx, B, T, M, H, dh, (int)mem_len, scale, RP_S(stream),
                            dh_out, ld_ctx);
}
int rp_xl_attn_bwd_dq(const void* grad_ctx_h, const void* vh, const void* kh, const void* rh, const void* probs,
                      void* grad_ac, void* grad_bd, int64_t ld_p, const void* grad_ctx, const void* ctx, float* grad_qu,
                      float* grad_qv, int64_t B, int64_t T, int64_t M, int32_t H, int32_t dh, int64_t mem_len,
                      float scale, float* bias_part, float* d_rows, void* grad_qkv, void* stream) {
  return rp::xl_attn_bwd_dq(grad_ctx_h, vh, kh, rh, probs, grad_ac, grad_bd, ld_p, grad_ctx, ctx, grad_qu, grad_qv, B,
                            T, M, H, dh, (int)mem_len, scale, RP_S(stream), bias_part, d_rows, grad_qkv);
}
int rp_xl_dq_persistent(void) { return rp::xl_dq_persistent() ? 1 : 0; }
int rp_xl_attn_bwd_kv(const void* grad_ctx_h, const void* vh, const void* qu, const void* probs, int64_t ld_p,
                      const float* d_rows, void* grad_kh, void* grad_vh, int64_t B, int64_t T, int64_t M, int32_t H,
                      int32_t dh, int64_t mem_len, float scale, void* grad_qkv, void* stream) {
  return rp::xl_attn_bwd_kv(grad_ctx_h, vh, qu, probs, ld_p, d_rows, grad_kh, grad_vh, B, T, M, H, dh, (int)mem_len,
                            scale, RP_S(stream), grad_qkv);
}
int64_t rp_xl_dq_bias_part_bytes(int32_t H, int64_t B, int64_t T) { return rp::xl_dq_bias_part_bytes(H, B, T); }
int rp_xl_dq_bias_finish(const float* bias_part, float* g_r_w_bias, float* g_r_r_bias, int32_t H, int64_t B, int64_t T,
                         void* stream) {
  return rp::xl_dq_bias_finish(bias_part, g_r_w_bias, g_r_r_bias, H, B, T, RP_S(stream));
}
int rp_xl_softmax_bwd(int32_t dtype, const float* grad_p, int64_t ld_scores, const void* probs, int64_t ld_p,
                      void* grad_ac, void* grad_bd, int64_t rows, int64_t T, int64_t M, int64_t mem_len, float scale,
                      void* stream) {
  return rp::xl_softmax_bwd(dtype, grad_p, ld_scores, probs, ld_p, grad_ac, grad_bd, rows, T, M, mem_len, scale,
                            RP_S(stream));
}
int rp_rows_copy(int32_t src_dtype, const void* src, int64_t ld_src, int64_t rows, int64_t cols, const float* val,
                 float val_const, int32_t aug, int32_t dst_dtype, void* dst, int64_t ld_dst, void* stream) {
  return rp::rows_copy(src_dtype, src, ld_src, rows, cols, val, val_const, aug, dst_dtype, dst, ld_dst, RP_S(stream));
}
int rp_rows_gather(int32_t dtype, const void* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols,
                   void* dst, int64_t ld_dst, void* stream) {
  return rp::rows_gather(dtype, src, ld_src, idx, n, cols, dst, ld_dst, RP_S(stream));
}
int rp_rows_scatter_add(const float* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols, float* dst,
                        int64_t ld_dst, void* stream) {
  return rp::rows_scatter_add(src, ld_src, idx, n, cols, dst, ld_dst, RP_S(stream));
}
int64_t rp_xl_bias_grad_workspace_bytes(int32_t H, int32_t dh) { return rp::xl_bias_grad_workspace_bytes(H, dh); }
int rp_xl_bias_grad(const float* g_qu, const float* g_qv, float* workspace, float* g_r_w_bias, float* g_r_r_bias,
                    int32_t H, int64_t R, int32_t dh, int64_t ld_g, void* stream) {
  return rp::xl_bias_grad(g_qu, g_qv, workspace, g_r_w_bias, g_r_r_bias, H, R, dh, RP_S(stream), ld_g);
}

int64_t rp_module_workspace_bytes(const rp_module_desc* desc) { return rp::module_workspace_bytes(*desc); }
int rp_module_forward(const rp_module_desc* desc, const rp_module_weights* w, const rp_module_slot* slot, void* out,
                      void* workspace, int64_t workspace_bytes, int32_t* flag, void* stream) {
  return rp::module_forward(*desc, *w, *slot, out, workspace, workspace_bytes, flag, RP_S(stream));
}
int rp_module_backward(const rp_module_desc* desc, const rp_module_weights* w, const rp_module_slot* slot,
                       const float* g_out, float* g_in, const rp_module_grads* grads, void* workspace,
                       int64_t workspace_bytes, void* stream) {
  return rp::module_backward(*desc, *w, *slot, g_out, g_in, *grads, workspace, workspace_bytes, RP_S(stream));
}
int64_t rp_xl_block_workspace_bytes(const rp_xl_block_desc* desc) { return rp::xl_block_workspace_bytes(*desc); }
int rp_xl_block_forward(const rp_xl_block_desc* desc, const rp_xl_block_weights* w, const void* R, void* out,
                        const rp_xl_block_tape* tape, void* workspace, int64_t workspace_bytes, int32_t* flag,
                        void* stream) {
  return rp::xl_block_forward(*desc, *w, R, out, *tape, workspace, workspace_bytes, flag, RP_S(stream));
}
int rp_xl_block_backward(const rp_xl_block_desc* desc, const rp_xl_block_weights* w, const void* R,
                         const rp_xl_block_tape* tape, const float* g_out, float* g_x, const rp_xl_block_grads* grads,
                         void* workspace, int64_t workspace_bytes, void* stream) {
  return rp::xl_block_backward(*desc, *w, R, *tape, g_out, g_x, *grads, workspace, workspace_bytes, RP_S(stream));
}
int64_t rp_block_workspace_bytes(const rp_block_desc* desc) { return rp::block_workspace_bytes(*desc); }
int rp_block_forward(const rp_block_desc* desc, const rp_block_weights* w, const void* x, void* out,
                     const rp_block_tape* tape, void* workspace, int64_t workspace_bytes, int32_t* flag,
                     void* stream) {
  return rp::block_forward(*desc, *w, x, out, *tape, workspace, workspace_bytes, flag, RP_S(stream));
}
int rp_block_backward(const rp_block_desc* desc, const rp_block_weights* w, const void* x, const rp_block_tape* tape,
                      const float* g_out, float* g_x, const rp_block_grads* grads, void* workspace,
                      int64_t workspace_bytes, void* stream) {
  return rp::block_backward(*desc, *w, x, *tape, g_out, g_x, *grads, workspace, workspace_bytes, RP_S(stream));
}
int64_t rp_head_workspace_bytes(const rp_head_desc* desc) { return rp::head_workspace_bytes(*desc); }
int rp_head_forward(const rp_head_desc* desc, const void* x, const void* tied, const int64_t* targets, float* lse,
                    float* loss, double* loss64, void* workspace, int64_t workspace_bytes, int32_t* flag,
                    void* stream) {
  return rp::head_forward(*desc, x, tied, targets, lse, loss, loss64, workspace, workspace_bytes, flag, RP_S(stream));
}
int rp_head_backward(const rp_head_desc* desc, const void* x, const void* tied, const int64_t* targets,
                     const float* lse, float* g_x, float* vo, float vo_alpha, int32_t vo_accumulate,
                     void* workspace, int64_t workspace_bytes, void* stream) {
  return rp::head_backward(*desc, x, tied, targets, lse, g_x, vo, vo_alpha, vo_accumulate, workspace, workspace_bytes,
                           RP_S(stream));
}

}  // extern "C"
