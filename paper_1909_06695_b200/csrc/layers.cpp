// Native layer composition: one C-ABI call runs a whole transformer block
// forward or backward, or the tied head, issuing its GEMMs and row kernels
// back-to-back on the caller's stream.  This is the reference's layer
// protocol seam (`forward(params, x, rng, train)` / `backward(params, tape,
// grad_out)`, reference layers.py:28-37, 168-253, 299-322) with the Python
// per-op dispatch removed from the hot loop.
//
// Scratch comes from a caller-owned device workspace (rp_*_workspace_bytes);
// in tf32x3 mode every GEMM operand is split into (hi, lo) halves inside it.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "rp_internal.h"

namespace rp {
namespace {

inline int64_t pad8(int64_t n) { return (n + 7) / 8 * 8; }

#define RP_TRY0(x)                \
  do {                            \
    if (int _e = (x)) return _e;  \
  } while (0)
inline int64_t al256(int64_t n) { return (n + 255) / 256 * 256; }
inline int esize(int dt) { return dt == RP_BF16 ? 2 : 4; }

struct Bump {
  char* base;
  int64_t cap, off = 0;
  void* take(int64_t bytes) {
    void* p = base + off;
    off += al256(bytes);
    return p;
  }
};

// Row-major matrix view (optionally batched).
struct Mat {
  const void* p;
  int64_t rows, cols, ld;
  int64_t batch = 1, bstride = 0;
};

inline Mat mat(const void* p, int64_t rows, int64_t cols, int64_t ld) { return Mat{p, rows, cols, ld, 1, 0}; }
inline Mat bmat(const void* p, int64_t b, int64_t rows, int64_t cols, int64_t ld, int64_t bs) {
  return Mat{p, rows, cols, ld, b, bs};
}

struct Ctx {
  int dtype;  // compute dtype of activations / weights
  cudaStream_t st;
  int max_ctas = 0;
  char* split_base = nullptr;  // tf32x3 split scratch
  int64_t split_cap = 0;
  float* splitk = nullptr;  // split-K partials
  int64_t splitk_cap = 0;   // bytes
};

// Deterministic split-K for weight-gradient shaped GEMMs (few output tiles,
// long K): pick S minimising waves(S) * tile_time(K/S) + partial traffic.
int choose_splits(int64_t M, int64_t N, int64_t K, int bn, int64_t cap_bytes, int64_t batch) {
  batch = std::max<int64_t>(batch, 1);
  const int64_t tiles = ((M + 127) / 128) * ((N + bn - 1) / bn) * batch;
  if (tiles >= 148 || K < 1024 || cap_bytes <= 0) return 1;
  const double R = 1.1e15 / 148.0, BW = 5.5e12;
  int best = 1;
  double best_t = 2.0 * 128 * bn * (double)K / R;
  const int smax = (int)std::min<int64_t>({64, K / 512, cap_bytes / (M * N * 4 * batch)});
  for (int S = 2; S <= smax; ++S) {
    const double waves = std::ceil((double)(tiles * S) / 148.0);
    const double t = waves * 2.0 * 128 * bn * ((double)K / S) / R + (double)S * M * N * batch * 8.0 / BW;
    if (t < best_t * 0.97) {
      best_t = t;
      best = S;
    }
  }
  return best;
}

struct Epi {
  int kind = RP_EPI_STORE;
  float alpha = 1.f;
  const float* bias = nullptr;
  const void* resid = nullptr;
  int64_t ld_resid = 0, stride_resid = 0;
  int drop = 0;
  uint64_t seed = 0, thr = 0, pos0 = 0;
  float scale = 1.f;
  const int64_t* targets = nullptr;
  const float* lse = nullptr;
  float* partial = nullptr;
  float* target_logit = nullptr;
  float ce_scale = 0.f;
  int tile_n = 0;  // N tile override (0: the library default)
  int64_t k_lo_off = 0;  // banded A: row m of op(A) is zero for k < m + k_lo_off (with k_lo = 1)
  int k_lo = 0;
};

int split_into(Ctx& c, Bump& b, const Mat& m, const void** hi, const void** lo, int64_t* ld, int64_t* bs) {
  const int64_t ldd = (m.cols + 3) / 4 * 4;
  const int64_t n = m.batch * m.rows * ldd;
  float* h = static_cast<float*>(b.take(n * 4));
  float* l = static_cast<float*>(b.take(n * 4));
  if (b.off > b.cap) return set_error(RP_ERR_INVALID, "tf32x3 split scratch too small");
  if (m.batch <= 1 || m.bstride == m.rows * m.ld) {  // batch rows evenly pitched: one launch
    if (int e = tf32_split(static_cast<const float*>(m.p), h, l, m.batch * m.rows, m.cols, m.ld, ldd, c.st)) return e;
  } else {
    for (int64_t i = 0; i < m.batch; ++i) {
      const float* src = static_cast<const float*>(m.p) + i * m.bstride;
      if (int e = tf32_split(src, h + i * m.rows * ldd, l + i * m.rows * ldd, m.rows, m.cols, m.ld, ldd, c.st))
        return e;
    }
  }
  *hi = h;
  *lo = l;
  *ld = ldd;
  *bs = m.rows * ldd;
  return RP_OK;
}

// C = epi(alpha * opA(A) opB(B)).  A: [M,K] (a_mn: stored [K,M]); B: stored [N,K] (b_mn: [K,N]).
int mm(Ctx& c, const Mat& A, bool a_mn, const Mat& B, bool b_mn, const Mat& C, int out_dtype, const Epi& e = Epi()) {
  rp_gemm_args g;
  std::memset(&g, 0, sizeof(g));
  g.math = c.dtype == RP_BF16 ? RP_MATH_BF16 : RP_MATH_TF32X3;
  g.out_dtype = out_dtype;
  g.max_ctas = c.max_ctas;
  g.a_mn_major = a_mn;
  g.b_mn_major = b_mn;
  g.M = a_mn ? A.cols : A.rows;
  g.K = a_mn ? A.rows : A.cols;
  g.N = b_mn ? B.cols : B.rows;
  g.batch = std::max(A.batch, B.batch);
  g.A = A.p;
  g.lda = A.ld;
  g.stride_a = A.batch > 1 ? A.bstride : 0;
  g.B = B.p;
  g.ldb = B.ld;
  g.stride_b = B.batch > 1 ? B.bstride : 0;
  Bump sb{c.split_base, c.split_cap};
  if (g.math == RP_MATH_TF32X3) {
    int64_t ld, bs;
    const void *hi, *lo;
    if (int r = split_into(c, sb, A, &hi, &lo, &ld, &bs)) return r;
    g.A = hi;
    g.A_lo = lo;
    g.lda = ld;
    g.stride_a = A.batch > 1 ? bs : 0;
    if (int r = split_into(c, sb, B, &hi, &lo, &ld, &bs)) return r;
    g.B = hi;
    g.B_lo = lo;
    g.ldb = ld;
    g.stride_b = B.batch > 1 ? bs : 0;
  }
  g.C = const_cast<void*>(C.p);
  g.ldc = C.ld;
  g.stride_c = C.bstride;
  g.k_lo_sign = e.k_lo;
  g.k_lo_off = e.k_lo_off;
  int splits = 1;
  // batched split-K needs the batch's output rows contiguous (one [batch*M, N] reduce)
  const bool rows_fold = g.batch == 1 || g.stride_c == g.M * g.ldc;
  if (out_dtype == RP_F32 && e.kind == RP_EPI_STORE && rows_fold && g.k_lo_sign <= 0 && c.splitk)
    splits = choose_splits(g.M, g.N, g.K, 256, c.splitk_cap, g.batch);
  if (splits > 1) {
    g.k_splits = splits;
    g.C = c.splitk;
    g.ldc = g.N;
    g.stride_c = g.M * g.N;
  }
  g.epilogue = e.kind;
  g.alpha = e.alpha;
  g.bias = e.bias;
  g.residual = e.resid;
  g.ld_residual = e.ld_resid;
  g.stride_residual = e.stride_resid;
  g.drop_enabled = e.drop;
  g.drop_seed = e.seed;
  g.drop_threshold = e.thr;
  g.drop_pos0 = e.pos0;
  g.drop_scale = e.scale;
  g.targets = e.targets;
  g.lse = e.lse;
  g.partial = e.partial;
  g.target_logit = e.target_logit;
  g.ce_scale = e.ce_scale;
  g.tile_n = e.tile_n;
  RP_TRY0(gemm(g, c.st));
  if (splits > 1) return splitk_reduce(c.splitk, splits, g.batch * g.M, g.N, static_cast<float*>(const_cast<void*>(C.p)), C.ld,
                                       c.st);
  return RP_OK;
}

int64_t split_bytes(int dtype, int64_t max_elems) {
  // two operands x (hi, lo), rows padded to 4 floats
  return dtype == RP_BF16 ? 0 : 4 * al256((max_elems + 4096) * 4) + 4096;
}

#define RP_TRY(x)                 \
  do {                            \
    if (int _e = (x)) return _e;  \
  } while (0)

// A second stream (per device, per host thread) onto which the block backward
// forks the independent GEMM of each pair that shares an input; the fork and
// join are event edges, so the pair overlaps (and CUDA-graph capture works).
struct SideStream {
  int device = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

SideStream& side_for(cudaStream_t main) {
  // one side stream per (device, main stream): concurrent callers on
  // different streams must not serialise on a shared side stream
  static thread_local std::vector<std::pair<cudaStream_t, SideStream>> pool;
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& e : pool)
    if (e.first == main && e.second.device == dev) return e.second;
  SideStream ss;
  int prio = 0;
  cudaStreamGetPriority(main, &prio);
  cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, prio);
  cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming);
  ss.device = dev;
  pool.emplace_back(main, ss);
  return pool.back().second;
}

bool fork_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RP_FORK");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

}  // namespace

int gemm_choose_splits(int64_t M, int64_t N, int64_t K, int64_t cap_bytes, int64_t batch) {
  return choose_splits(M, N, K, 256, cap_bytes, batch);
}

// ---------------------------------------------------------------------------
// block

constexpr int64_t kBlockSplitK = 296LL * 128 * 256 * 4;  // split-K partials of the dW GEMMs

int64_t block_workspace_bytes(const rp_block_desc& d) {
  const int64_t N = d.B * d.T, Tp = pad8(d.T), e = esize(d.dtype);
  const int64_t nbp = std::max<int64_t>({colsum_blocks(N), ln_bwd_blocks(N), mask_grad_blocks(N, d.d)});
  int64_t b = 0;
  b += al256(d.B * d.T * Tp * 4);              // scores / g_p
  b += al256(d.B * d.T * Tp * e);              // g_s
  b += al256(N * d.d * e) * 3;                 // g_h2, g_proj, g_ctx
  b += al256(N * d.f * e);                     // g_z1
  b += al256(N * 3 * d.d * e);                 // g_qkv
  b += al256(N * d.d * 4) * 3;                 // g_m, g_x1, g_a
  b += al256(nbp * std::max(d.f, 3 * d.d) * 4) * 3;  // partials
  b += al256(nbp * d.d * 4) * 3;                      // b2 / ln2 partials (finished together at the end)
  b += al256(kBlockSplitK) * 2;  // main + side stream partials
  b += split_bytes(d.dtype, std::max({N * d.f, d.B * d.T * Tp, N * 3 * d.d, d.d * d.f}));
  return b + 4096;
}

int block_forward(const rp_block_desc& d, const rp_block_weights& w, const void* x, void* out, const rp_block_tape& tp,
                  void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st) {
  if (ws_bytes < block_workspace_bytes(d)) return set_error(RP_ERR_INVALID, "block workspace too small");
  const int64_t B = d.B, T = d.T, D = d.d, F = d.f, N = B * T, Tp = pad8(T);
  const int dt = d.dtype, e = esize(dt);
  Bump bp{static_cast<char*>(ws), ws_bytes};
  float* scores = static_cast<float*>(bp.take(B * T * Tp * 4));
  Ctx c{dt, st};
  c.max_ctas = d.max_ctas;
  c.split_base = bp.base + bp.off;
  c.split_cap = ws_bytes - bp.off;
  const char* qkv = static_cast<const char*>(tp.qkv);
  RP_TRY(layernorm_fwd(dt, x, w.ln1_g, w.ln1_b, tp.a, tp.mean1, tp.rstd1, N, D, flag, st));
  RP_TRY(mm(c, mat(tp.a, N, D, D), false, mat(w.wqkv, D, 3 * D, 3 * D), true, mat(tp.qkv, N, 3 * D, 3 * D), dt));
  Epi es;
  es.alpha = 1.f / std::sqrt(static_cast<float>(D));
  RP_TRY(mm(c, bmat(qkv, B, T, D, 3 * D, T * 3 * D), false, bmat(qkv + D * e, B, T, D, 3 * D, T * 3 * D), false,
            bmat(scores, B, T, T, Tp, T * Tp), RP_F32, es));
  RP_TRY(softmax_causal(dt, scores, tp.probs, N, T, Tp, st));
  RP_TRY(mm(c, bmat(tp.probs, B, T, T, Tp, T * Tp), false, bmat(qkv + 2 * D * e, B, T, D, 3 * D, T * 3 * D), true,
            bmat(tp.ctx, B, T, D, D, T * D), dt));
  Epi e0;
  e0.kind = RP_EPI_BIAS_DROPOUT_RESIDUAL;
  e0.resid = x;
  e0.ld_resid = D;
  e0.drop = d.drop_enabled;
  e0.seed = d.drop_seed;
  e0.thr = d.drop_threshold;
  e0.scale = d.drop_scale;
  e0.pos0 = 0;
  RP_TRY(mm(c, mat(tp.ctx, N, D, D), false, mat(w.wo, D, D, D), true, mat(tp.x1, N, D, D), dt, e0));
  RP_TRY(layernorm_fwd(dt, tp.x1, w.ln2_g, w.ln2_b, tp.m, tp.mean2, tp.rstd2, N, D, flag, st));
  Epi e1;
  e1.bias = w.b1;
  if (d.activation == 1) {
    // GELU: z1 = m w1 + b1 kept for the backward, h1 = gelu(z1) by the vector kernel
    if (!tp.z1) return set_error(RP_ERR_INVALID, "block_forward: GELU needs tape.z1");
    e1.kind = RP_EPI_BIAS_DROPOUT_RESIDUAL;  // bias only: no residual, no dropout
    RP_TRY(mm(c, mat(tp.m, N, D, D), false, mat(w.w1, D, F, F), true, mat(tp.z1, N, F, F), dt, e1));
    RP_TRY(gelu_fwd(dt, tp.z1, tp.h1, N * F, st));
  } else {
    e1.kind = RP_EPI_BIAS_RELU;
    RP_TRY(mm(c, mat(tp.m, N, D, D), false, mat(w.w1, D, F, F), true, mat(tp.h1, N, F, F), dt, e1));
  }
  Epi e2 = e0;
  e2.bias = w.b2;
  e2.resid = tp.x1;
  e2.pos0 = static_cast<uint64_t>((d.drop_rows_total > 0 ? d.drop_rows_total : N) * D);
  RP_TRY(mm(c, mat(tp.h1, N, F, F), false, mat(w.w2, F, D, D), true, mat(out, N, D, D), dt, e2));
  return RP_OK;
}

int block_backward(const rp_block_desc& d, const rp_block_weights& w, const void* x, const rp_block_tape& tp,
                   const float* g_out, float* g_x, const rp_block_grads& G, void* ws, int64_t ws_bytes,
                   cudaStream_t st) {
  if (ws_bytes < block_workspace_bytes(d)) return set_error(RP_ERR_INVALID, "block workspace too small");
  const int64_t B = d.B, T = d.T, D = d.d, F = d.f, N = B * T, Tp = pad8(T);
  const int dt = d.dtype, e = esize(dt);
  const int nbc = colsum_blocks(N), nbl = ln_bwd_blocks(N);
  const int64_t nbp = std::max<int64_t>({(int64_t)nbc, (int64_t)nbl, (int64_t)mask_grad_blocks(N, D)});
  Bump bp{static_cast<char*>(ws), ws_bytes};
  float* g_p = static_cast<float*>(bp.take(B * T * Tp * 4));
  void* g_s = bp.take(B * T * Tp * e);
  void* g_h2 = bp.take(N * D * e);
  void* g_proj = bp.take(N * D * e);
  void* g_ctx = bp.take(N * D * e);
  void* g_z1 = bp.take(N * F * e);
  char* g_qkv = static_cast<char*>(bp.take(N * 3 * D * e));
  float* g_m = static_cast<float*>(bp.take(N * D * 4));
  float* g_x1 = static_cast<float*>(bp.take(N * D * 4));
  float* g_a = static_cast<float*>(bp.take(N * D * 4));
  const int64_t pw = std::max(F, 3 * D);
  float* part = static_cast<float*>(bp.take(nbp * pw * 4));
  float* pg = static_cast<float*>(bp.take(nbp * pw * 4));
  float* pb = static_cast<float*>(bp.take(nbp * pw * 4));
  float* part_b2 = static_cast<float*>(bp.take(nbp * D * 4));
  float* pg2 = static_cast<float*>(bp.take(nbp * D * 4));
  float* pb2 = static_cast<float*>(bp.take(nbp * D * 4));
  Ctx c{dt, st};
  c.max_ctas = d.max_ctas;
  c.splitk = static_cast<float*>(bp.take(kBlockSplitK));
  c.splitk_cap = kBlockSplitK;
  float* splitk_side = static_cast<float*>(bp.take(kBlockSplitK));
  c.split_base = bp.base + bp.off;
  c.split_cap = ws_bytes - bp.off;
  // side context for the second GEMM of each independent pair (bf16 only:
  // the tf32x3 check mode shares one operand-split scratch, so it stays serial)
  const bool fork = dt == RP_BF16 && fork_enabled();
  SideStream* ss = fork ? &side_for(st) : nullptr;
  Ctx cs = c;
  Ctx cf = c;  // first GEMM of a forked pair
  if (fork) {
    cs.st = ss->s;
    cs.splitk = splitk_side;
    static int budget = -1;
    if (budget < 0) {
      const char* e = getenv("RP_FORK_CTAS");
      budget = e ? atoi(e) : 0;
    }
    if (budget > 0) {
      cs.max_ctas = budget;
      cf.max_ctas = 148 - budget;
    }
  }
  auto pair = [&](auto&& first, auto&& second) -> int {
    if (!fork) {
      RP_TRY(first(c));
      return second(c);
    }
    if (cudaEventRecord(ss->fork, st) != cudaSuccess || cudaStreamWaitEvent(ss->s, ss->fork, 0) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "block_backward: fork failed");
    RP_TRY(second(cs));
    RP_TRY(first(cf));
    if (cudaEventRecord(ss->join, ss->s) != cudaSuccess || cudaStreamWaitEvent(st, ss->join, 0) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "block_backward: join failed");
    return RP_OK;
  };
  const char* qkv = static_cast<const char*>(tp.qkv);
  const float inv = 1.f / std::sqrt(static_cast<float>(D));
  // feed-forward branch (layers.py:209-232)
  // The bias / LayerNorm column sums only feed the optimizer: their partials
  // get separate buffers and one batched finish at the end, off the chain of
  // dependent kernels that carries g_x.
  RP_TRY(mask_grad(dt, g_out, g_h2, N, D, d.drop_seed,
                   static_cast<uint64_t>((d.drop_rows_total > 0 ? d.drop_rows_total : N) * D), d.drop_threshold,
                   d.drop_scale,
                   d.drop_enabled, part_b2, st));
  Epi er;
  er.kind = d.activation == 1 ? RP_EPI_GELU_GRAD : RP_EPI_RELU_GRAD;
  er.resid = d.activation == 1 ? tp.z1 : tp.h1;
  er.ld_resid = F;
  if (d.activation == 1 && !tp.z1) return set_error(RP_ERR_INVALID, "block_backward: GELU needs tape.z1");
  RP_TRY(pair([&](Ctx& x) { return mm(x, mat(g_h2, N, D, D), false, mat(w.w2, F, D, D), false, mat(g_z1, N, F, F), dt, er); },
              [&](Ctx& x) { return mm(x, mat(tp.h1, N, F, F), true, mat(g_h2, N, D, D), true, mat(G.w2, F, D, D), RP_F32); }));
  // b1 partial sums ride with dW1 on the side stream (both only read g_z1)
  RP_TRY(pair([&](Ctx& x) { return mm(x, mat(g_z1, N, F, F), false, mat(w.w1, D, F, F), false, mat(g_m, N, D, D), RP_F32); },
              [&](Ctx& x) {
                RP_TRY(colsum_partial(dt, g_z1, N, F, F, part, x.st));
                return mm(x, mat(tp.m, N, D, D), true, mat(g_z1, N, F, F), true, mat(G.w1, D, F, F), RP_F32);
              }));
  RP_TRY(layernorm_bwd(dt, g_m, tp.x1, tp.mean2, tp.rstd2, w.ln2_g, g_out, g_x1, g_proj, d.drop_seed,
                       d.drop_threshold, d.drop_scale, d.drop_enabled, pg2, pb2, N, D, st));
  // attention branch (layers.py:234-247)
  RP_TRY(pair([&](Ctx& x) { return mm(x, mat(g_proj, N, D, D), false, mat(w.wo, D, D, D), false, mat(g_ctx, N, D, D), dt); },
              [&](Ctx& x) { return mm(x, mat(tp.ctx, N, D, D), true, mat(g_proj, N, D, D), true, mat(G.wo, D, D, D), RP_F32); }));
  const Mat q = bmat(qkv, B, T, D, 3 * D, T * 3 * D);
  const Mat k = bmat(qkv + D * e, B, T, D, 3 * D, T * 3 * D);
  const Mat v = bmat(qkv + 2 * D * e, B, T, D, 3 * D, T * 3 * D);
  const Mat P = bmat(tp.probs, B, T, T, Tp, T * Tp);
  const Mat gctx = bmat(g_ctx, B, T, D, D, T * D);
  RP_TRY(pair([&](Ctx& x) { return mm(x, gctx, false, v, false, bmat(g_p, B, T, T, Tp, T * Tp), RP_F32); },
              [&](Ctx& x) { return mm(x, P, true, gctx, true, bmat(g_qkv + 2 * D * e, B, T, D, 3 * D, T * 3 * D), dt); }));
  RP_TRY(softmax_bwd(dt, g_p, tp.probs, g_s, inv, N, T, Tp, st));
  const Mat gs = bmat(g_s, B, T, T, Tp, T * Tp);
  RP_TRY(pair([&](Ctx& x) { return mm(x, gs, false, k, true, bmat(g_qkv, B, T, D, 3 * D, T * 3 * D), dt); },
              [&](Ctx& x) { return mm(x, gs, true, q, true, bmat(g_qkv + D * e, B, T, D, 3 * D, T * 3 * D), dt); }));
  RP_TRY(pair([&](Ctx& x) { return mm(x, mat(g_qkv, N, 3 * D, 3 * D), false, mat(w.wqkv, D, 3 * D, 3 * D), false, mat(g_a, N, D, D), RP_F32); },
              [&](Ctx& x) { return mm(x, mat(tp.a, N, D, D), true, mat(g_qkv, N, 3 * D, 3 * D), true, mat(G.wqkv, D, 3 * D, 3 * D), RP_F32); }));
  RP_TRY(layernorm_bwd(dt, g_a, x, tp.mean1, tp.rstd1, w.ln1_g, g_x1, g_x, nullptr, 0, 0, 1.f, 0, pg, pb, N, D, st));
  const ColsumJob jobs[6] = {{part_b2, mask_grad_blocks(N, D), D, G.b2}, {part, nbc, F, G.b1},
                             {pg2, nbl, D, G.ln2_g}, {pb2, nbl, D, G.ln2_b},
                             {pg, nbl, D, G.ln1_g}, {pb, nbl, D, G.ln1_b}};
  return colsum_finish_multi(jobs, 6, st);
}

// ---------------------------------------------------------------------------
// tied head

constexpr int64_t kHeadSplitK = 16;  // max split-K factor of g_x = dz @ tied

int64_t head_workspace_bytes(const rp_head_desc& h) {
  const int bn = gemm_tile_n(h.rows, h.vocab, 1);
  const int64_t nt = (h.vocab + bn - 1) / bn;
  const int64_t e = esize(h.dtype);
  int64_t b = al256(h.rows * nt * 4 * 4) + al256(h.rows * 4) * 2 + al256(h.rows * pad8(h.vocab) * e);
  b += al256(kHeadSplitK * h.rows * h.d * 4);
  b += split_bytes(h.dtype, std::max({h.rows * pad8(h.vocab), h.vocab * h.d, h.rows * h.d}));
  return b + 4096;
}

int head_forward(const rp_head_desc& h, const void* x, const void* tied, const int64_t* targets, float* lse,
                 float* loss, double* loss64, void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st) {
  if (ws_bytes < head_workspace_bytes(h)) return set_error(RP_ERR_INVALID, "head workspace too small");
  const int bn = gemm_tile_n(h.rows, h.vocab, 1);
  const int64_t nt = (h.vocab + bn - 1) / bn, N = h.rows, D = h.d, V = h.vocab;
  Bump bp{static_cast<char*>(ws), ws_bytes};
  float* partial = static_cast<float*>(bp.take(N * nt * 4 * 4));  // (max, sum) per row, tile and column half
  float* zy = static_cast<float*>(bp.take(N * 4));
  float* rows = static_cast<float*>(bp.take(N * 4));
  bp.take(N * pad8(V) * esize(h.dtype));  // dz (backward)
  bp.take(kHeadSplitK * N * D * 4);        // split-K partials (backward)
  Ctx c{h.dtype, st};
  c.split_base = bp.base + bp.off;
  c.split_cap = ws_bytes - bp.off;
  Epi e;
  e.kind = RP_EPI_LSE_PARTIAL;
  e.targets = targets;
  e.partial = partial;
  e.target_logit = zy;
  RP_TRY(mm(c, mat(x, N, D, D), false, mat(tied, V, D, D), false, Mat{nullptr, N, V, 0}, RP_F32, e));
  return ce_finish(partial, (int)(2 * nt), zy, targets, V, N, lse, rows, loss, loss64, flag, st);
}

int head_backward(const rp_head_desc& h, const void* x, const void* tied, const int64_t* targets, const float* lse,
                  float* g_x, float* vo, float vo_alpha, int vo_accumulate, void* ws, int64_t ws_bytes,
                  cudaStream_t st) {
  if (ws_bytes < head_workspace_bytes(h)) return set_error(RP_ERR_INVALID, "head workspace too small");
  const int bn = gemm_tile_n(h.rows, h.vocab, 1);
  const int64_t nt = (h.vocab + bn - 1) / bn, N = h.rows, D = h.d, V = h.vocab, Vp = pad8(V);
  Bump bp{static_cast<char*>(ws), ws_bytes};
  bp.take(N * nt * 2 * 4);
  bp.take(N * 4);
  bp.take(N * 4);
  void* dz = bp.take(N * Vp * esize(h.dtype));
  Ctx c{h.dtype, st};
  c.splitk = static_cast<float*>(bp.take(kHeadSplitK * N * D * 4));
  c.splitk_cap = kHeadSplitK * N * D * 4;
  c.split_base = bp.base + bp.off;
  c.split_cap = ws_bytes - bp.off;
  Epi e;
  e.kind = RP_EPI_CE_GRAD;
  e.targets = targets;
  e.lse = lse;
  e.ce_scale = 1.f / static_cast<float>(h.rows_total > 0 ? h.rows_total : N);
  RP_TRY(mm(c, mat(x, N, D, D), false, mat(tied, V, D, D), false, mat(dz, N, V, Vp), h.dtype, e));
  RP_TRY(mm(c, mat(dz, N, V, Vp), false, mat(tied, V, D, D), true, mat(g_x, N, D, D), RP_F32));
  if (vo) {
    Epi ev;
    ev.alpha = vo_alpha;
    if (vo_accumulate) {  // vo += alpha * dz^T x   (residual epilogue reading vo in place)
      ev.kind = RP_EPI_BIAS_DROPOUT_RESIDUAL;
      ev.resid = vo;
      ev.ld_resid = D;
    }
    RP_TRY(mm(c, mat(dz, N, V, Vp), true, mat(x, N, D, D), true, mat(vo, V, D, D), RP_F32, ev));
  }
  return RP_OK;
}


// ---------------------------------------------------------------------------
// Transformer-XL block (the same op sequence as paper_1909_06695_b200/xl.py,
// so results are bitwise identical; the restatement is oracle/xl.py)

namespace {

struct XlDims {
  int64_t B, T, M, Kl, D, F, H, dh, N, HB, ldk;
};

XlDims xl_dims(const rp_xl_block_desc& d) {
  XlDims x;
  x.B = d.B;
  x.T = d.T;
  x.M = d.M;
  x.Kl = d.M + d.T;
  x.D = d.d;
  x.F = d.f;
  x.H = d.H;
  x.dh = d.d / d.H;
  x.N = d.B * d.T;
  x.HB = d.H * d.B;
  x.ldk = d.ldk;
  return x;
}

int check_xl(const rp_xl_block_desc& d) {
  if (d.H <= 0 || d.d % d.H || d.B <= 0 || d.T <= 0 || d.M < 0 || d.mem_len < 0 || d.mem_len > d.M)
    return set_error(RP_ERR_DIMENSION, "xl_block: bad shape");
  if (d.ldk < d.M + d.T || d.ldk % 8) return set_error(RP_ERR_DIMENSION, "xl_block: ldk must be pad8(M+T)");
  if (d.dtype == RP_BF16 && (d.d % 8 || d.f % 8 || (d.d / d.H) % 8))
    return set_error(RP_ERR_DIMENSION,
                     "xl_block: the composite takes dense bf16 rows (d, d_ff, head dim multiples of 8); "
                     "pitched rows go through the op-level entry points");
  if (d.dtype != RP_BF16 && (d.fused & (15 | RP_XL_FUSED_KV)))
    return set_error(RP_ERR_INVALID, "xl_block: fused kernels are bf16 only");
  if ((d.fused & RP_XL_FUSED_KV) && !(d.fused & RP_XL_FUSED_DQ))
    return set_error(RP_ERR_INVALID, "xl_block: RP_XL_FUSED_KV needs RP_XL_FUSED_DQ");
  return RP_OK;
}

}  // namespace

int64_t xl_block_workspace_bytes(const rp_xl_block_desc& d) {
  const XlDims x = xl_dims(d);
  const int64_t e = esize(d.dtype);
  const int64_t nbc = colsum_blocks(x.N), nbm = mask_grad_blocks(x.N, x.D);
  const int64_t nbl = ln_bwd_blocks(x.N) + (x.M ? ln_bwd_blocks(x.B * x.M) : 0);
  int64_t b = 0;
  // forward: r, ctx_h, ac, bd (unfused scores)
  const int64_t fwd = al256(x.Kl * x.D * e) + al256(x.HB * x.T * x.dh * e) + 2 * al256(x.HB * x.T * x.ldk * 4);
  // backward
  int64_t bwd = al256(std::max(nbc, nbm) * std::max(x.F, 3 * x.D) * 4) + al256(nbm * x.D * 4);
  bwd += al256(x.N * x.D * e) * 3;          // g_h2, g_proj, g_ctx
  bwd += al256(x.N * x.F * e);              // g_z1
  bwd += al256(x.N * x.D * 4) * 2;          // g_m, g_x1
  bwd += al256(nbl * x.D * 4) * 2 + al256(ln_bwd_blocks(x.N) * x.D * 4) * 2;  // LN partials
  bwd += al256(x.H * x.N * x.dh * e);       // g_ctx_h
  bwd += 2 * al256(x.HB * x.T * x.ldk * e); // g_ac, g_bd
  bwd += al256(x.HB * x.T * x.ldk * 4);     // g_p (unfused)
  bwd += 2 * al256(x.H * x.N * x.dh * 4);   // g_qu, g_qv
  bwd += 2 * al256(x.HB * x.Kl * x.dh * e) + al256(x.H * x.Kl * x.dh * 4);  // g_vh, g_kh (compute dtype), g_rh
  bwd += al256(xl_bias_grad_workspace_bytes((int)x.H, (int)x.dh));
  if (d.fused & RP_XL_FUSED_DQ) bwd += al256(xl_dq_bias_part_bytes((int)x.H, x.B, x.T));
  if (d.fused & RP_XL_FUSED_KV) bwd += al256(x.HB * x.T * 4);  // D rows
  bwd += al256(x.Kl * x.D * e) + al256(x.B * x.Kl * 3 * x.D * e);  // g_r, g_qkv
  bwd += al256(x.B * x.Kl * x.D * 4);  // g_a
  bwd += al256(kBlockSplitK) * 2;  // main + side stream partials
  b = std::max(fwd, bwd);
  // tf32x3 split scratch: the largest operand of any contraction of the block,
  // rows padded to 4 floats (split_into)
  auto pd = [](int64_t rows, int64_t cols) { return rows * ((cols + 3) / 4 * 4); };
  b += split_bytes(d.dtype, std::max({pd(x.HB * x.T, x.ldk), pd(x.B * x.Kl, 3 * x.D), pd(x.N, x.F), pd(x.D, x.F),
                                      pd(x.F, x.D), pd(x.D, 3 * x.D), pd(x.HB * x.Kl, x.dh), pd(x.H * x.N, x.dh),
                                      pd(x.Kl, x.D), pd(x.B * x.Kl, x.D)}));
  return b + 4096;
}

int xl_block_forward(const rp_xl_block_desc& d, const rp_xl_block_weights& w, const void* R, void* out,
                     const rp_xl_block_tape& tp, void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st) {
  RP_TRY(check_xl(d));
  if (ws_bytes < xl_block_workspace_bytes(d)) return set_error(RP_ERR_INVALID, "xl_block workspace too small");
  const XlDims x = xl_dims(d);
  const int dt = d.dtype, e = esize(dt);
  const float scale = 1.f / std::sqrt(static_cast<float>(x.dh));
  Bump bp{static_cast<char*>(ws), ws_bytes};
  void* r = bp.take(x.Kl * x.D * e);
  void* ctx_h = bp.take(x.HB * x.T * x.dh * e);
  float* ac = static_cast<float*>(bp.take(x.HB * x.T * x.ldk * 4));
  float* bd = static_cast<float*>(bp.take(x.HB * x.T * x.ldk * 4));
  Ctx c{dt, st};
  c.max_ctas = d.max_ctas;
  c.split_base = bp.base + bp.off;
  c.split_cap = ws_bytes - bp.off;
  const int64_t BK = x.B * x.Kl;
  // the relative-encoding projection (independent of the block input) on the
  // side stream beside LN1 and the QKV projection (bf16; joined before the scores)
  const bool fork = dt == RP_BF16 && fork_enabled();
  SideStream* ss = fork ? &side_for(st) : nullptr;
  Ctx cs = c;
  if (fork) {
    cs.st = ss->s;
    if (cudaEventRecord(ss->fork, st) != cudaSuccess || cudaStreamWaitEvent(ss->s, ss->fork, 0) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "xl_block_forward: fork failed");
  }
  RP_TRY(mm(cs, mat(R, x.Kl, x.D, x.D), false, mat(w.wr, x.D, x.D, x.D), true, mat(r, x.Kl, x.D, x.D), dt));
  RP_TRY(xl_split_heads(dt, r, x.D, dt, tp.rh, x.Kl, (int)x.H, (int)x.dh, cs.st));
  RP_TRY(layernorm_fwd(dt, tp.xa, w.ln1_g, w.ln1_b, tp.a, tp.mean1, tp.rstd1, BK, x.D, flag, st));
  RP_TRY(mm(c, mat(tp.a, BK, x.D, x.D), false, mat(w.wqkv, x.D, 3 * x.D, 3 * x.D), true,
            mat(tp.qkv, BK, 3 * x.D, 3 * x.D), dt));
  RP_TRY(xl_split_qkv(dt, tp.qkv, w.r_w_bias, w.r_r_bias, tp.qu, tp.qv, tp.kh, tp.vh, x.B, x.T, x.M, (int)x.H,
                      (int)x.dh, st));
  if (fork && (cudaEventRecord(ss->join, ss->s) != cudaSuccess || cudaStreamWaitEvent(st, ss->join, 0) != cudaSuccess))
    return set_error(RP_ERR_CUDA, "xl_block_forward: join failed");
  bool pv_done = false;
  if (d.fused & RP_XL_FUSED_PV) {
    RP_TRY(xl_attn_fwd_pv(tp.qu, tp.qv, tp.kh, tp.vh, tp.rh, tp.probs, x.ldk, tp.ctx, x.B, x.T, x.M, (int)x.H,
                          (int)x.dh, d.mem_len, scale, st));
    pv_done = true;
  } else if (d.fused & RP_XL_FUSED_FWD) {
    RP_TRY(xl_attn_fwd(tp.qu, tp.qv, tp.kh, tp.rh, tp.probs, x.ldk, x.B, x.T, x.M, (int)x.H, (int)x.dh, d.mem_len,
                       scale, st));
  } else {
    Epi es;
    es.tile_n = d.score_tile;
    RP_TRY(mm(c, bmat(tp.qu, x.HB, x.T, x.dh, x.dh, x.T * x.dh), false, bmat(tp.kh, x.HB, x.Kl, x.dh, x.dh, x.Kl * x.dh),
              false, bmat(ac, x.HB, x.T, x.Kl, x.ldk, x.T * x.ldk), RP_F32, es));
    RP_TRY(mm(c, bmat(tp.qv, x.H, x.N, x.dh, x.dh, x.N * x.dh), false, bmat(tp.rh, x.H, x.Kl, x.dh, x.dh, x.Kl * x.dh),
              false, bmat(bd, x.H, x.N, x.Kl, x.ldk, x.N * x.ldk), RP_F32, es));
    RP_TRY(xl_softmax_fwd(dt, ac, bd, x.ldk, tp.probs, x.ldk, x.HB * x.T, x.T, x.M, d.mem_len, scale, st));
  }
  if (!pv_done) {
    RP_TRY(mm(c, bmat(tp.probs, x.HB, x.T, x.Kl, x.ldk, x.T * x.ldk), false,
              bmat(tp.vh, x.HB, x.Kl, x.dh, x.dh, x.Kl * x.dh), true, bmat(ctx_h, x.HB, x.T, x.dh, x.dh, x.T * x.dh),
              dt));
    RP_TRY(xl_merge_heads(dt, ctx_h, dt, tp.ctx, x.D, x.N, (int)x.H, (int)x.dh, st));
  }
  const int64_t n = (d.drop_rows_total > 0 ? d.drop_rows_total : x.N) * x.D;
  const void* xcur = static_cast<const char*>(tp.xa) + x.B * x.M * x.D * e;
  Epi e0;
  e0.kind = RP_EPI_BIAS_DROPOUT_RESIDUAL;
  e0.resid = xcur;
  e0.ld_resid = x.D;
  e0.drop = d.drop_enabled;
  e0.seed = d.drop_seed;
  e0.thr = d.drop_threshold;
  e0.scale = d.drop_scale;
  e0.pos0 = 0;
  RP_TRY(mm(c, mat(tp.ctx, x.N, x.D, x.D), false, mat(w.wo, x.D, x.D, x.D), true, mat(tp.x1, x.N, x.D, x.D), dt, e0));
  RP_TRY(layernorm_fwd(dt, tp.x1, w.ln2_g, w.ln2_b, tp.m, tp.mean2, tp.rstd2, x.N, x.D, flag, st));
  Epi e1;
  e1.bias = w.b1;
  if (d.activation == 1) {
    if (!tp.z1) return set_error(RP_ERR_INVALID, "xl_block_forward: GELU needs tape.z1");
    e1.kind = RP_EPI_BIAS_DROPOUT_RESIDUAL;
    RP_TRY(mm(c, mat(tp.m, x.N, x.D, x.D), false, mat(w.w1, x.D, x.F, x.F), true, mat(tp.z1, x.N, x.F, x.F), dt, e1));
    RP_TRY(gelu_fwd(dt, tp.z1, tp.h1, x.N * x.F, st));
  } else {
    e1.kind = RP_EPI_BIAS_RELU;
    RP_TRY(mm(c, mat(tp.m, x.N, x.D, x.D), false, mat(w.w1, x.D, x.F, x.F), true, mat(tp.h1, x.N, x.F, x.F), dt, e1));
  }
  Epi e2 = e0;
  e2.bias = w.b2;
  e2.resid = tp.x1;
  e2.pos0 = static_cast<uint64_t>(n);
  return mm(c, mat(tp.h1, x.N, x.F, x.F), false, mat(w.w2, x.F, x.D, x.D), true, mat(out, x.N, x.D, x.D), dt, e2);
}

int xl_block_backward(const rp_xl_block_desc& d, const rp_xl_block_weights& w, const void* R,
                      const rp_xl_block_tape& tp, const float* g_out, float* g_x, const rp_xl_block_grads& G,
                      void* ws, int64_t ws_bytes, cudaStream_t st) {
  RP_TRY(check_xl(d));
  if (ws_bytes < xl_block_workspace_bytes(d)) return set_error(RP_ERR_INVALID, "xl_block workspace too small");
  const XlDims x = xl_dims(d);
  const int dt = d.dtype, e = esize(dt);
  const float scale = 1.f / std::sqrt(static_cast<float>(x.dh));
  const int64_t N = x.N, D = x.D, F = x.F, BM = x.B * x.M, BK = x.B * x.Kl;
  const int64_t n = (d.drop_rows_total > 0 ? d.drop_rows_total : N) * D;
  const int nbc = colsum_blocks(N), nbm = mask_grad_blocks(N, D);
  const int nbl_cur = ln_bwd_blocks(N), nbl_mem = x.M ? ln_bwd_blocks(BM) : 0;
  Bump bp{static_cast<char*>(ws), ws_bytes};
  float* part = static_cast<float*>(bp.take((int64_t)std::max(nbc, nbm) * std::max(F, 3 * D) * 4));
  float* pm = static_cast<float*>(bp.take((int64_t)nbm * D * 4));
  void* g_h2 = bp.take(N * D * e);
  void* g_proj = bp.take(N * D * e);
  void* g_ctx = bp.take(N * D * e);
  void* g_z1 = bp.take(N * F * e);
  float* g_m = static_cast<float*>(bp.take(N * D * 4));
  float* g_x1 = static_cast<float*>(bp.take(N * D * 4));
  float* pg = static_cast<float*>(bp.take((int64_t)(nbl_cur + nbl_mem) * D * 4));
  float* pb = static_cast<float*>(bp.take((int64_t)(nbl_cur + nbl_mem) * D * 4));
  float* pg2 = static_cast<float*>(bp.take((int64_t)nbl_cur * D * 4));
  float* pb2 = static_cast<float*>(bp.take((int64_t)nbl_cur * D * 4));
  void* g_ctx_h = bp.take(x.H * N * x.dh * e);
  void* g_ac = bp.take(x.HB * x.T * x.ldk * e);
  void* g_bd = bp.take(x.HB * x.T * x.ldk * e);
  float* g_p = static_cast<float*>(bp.take(x.HB * x.T * x.ldk * 4));
  float* g_qu = static_cast<float*>(bp.take(x.H * N * x.dh * 4));
  float* g_qv = static_cast<float*>(bp.take(x.H * N * x.dh * 4));
  void* g_vh = bp.take(x.HB * x.Kl * x.dh * e);  // compute dtype: rounded as g_qkv holds them
  void* g_kh = bp.take(x.HB * x.Kl * x.dh * e);
  float* g_rh = static_cast<float*>(bp.take(x.H * x.Kl * x.dh * 4));
  float* bias_ws = static_cast<float*>(bp.take(xl_bias_grad_workspace_bytes((int)x.H, (int)x.dh)));
  float* dq_bias = (d.fused & RP_XL_FUSED_DQ) ? static_cast<float*>(bp.take(xl_dq_bias_part_bytes((int)x.H, x.B, x.T)))
                                              : nullptr;
  const bool kv = (d.fused & RP_XL_FUSED_KV) != 0;
  // the persistent bwd_dq and bwd_kv write straight into the merged g_qkv
  // rows (no fp32 dQu / dQv, no xl_merge_grads pass)
  const bool merged = kv && xl_dq_persistent();
  float* d_rows = kv ? static_cast<float*>(bp.take(x.HB * x.T * 4)) : nullptr;
  void* g_r = bp.take(x.Kl * D * e);
  void* g_qkv = bp.take(BK * 3 * D * e);
  float* g_a = static_cast<float*>(bp.take(BK * D * 4));
  Ctx c{dt, st};
  c.max_ctas = d.max_ctas;
  c.splitk = static_cast<float*>(bp.take(kBlockSplitK));
  c.splitk_cap = kBlockSplitK;
  float* splitk_side = static_cast<float*>(bp.take(kBlockSplitK));
  c.split_base = bp.base + bp.off;
  c.split_cap = ws_bytes - bp.off;
  const int64_t ld_part = std::max(F, 3 * D);
  // weight-gradient GEMMs on a side stream beside their input-gradient twins
  // (bf16; the block backward's pairing, bitwise the serial order)
  const bool fork = dt == RP_BF16 && fork_enabled();
  SideStream* ss = fork ? &side_for(st) : nullptr;
  Ctx cs = c;
  if (fork) {
    cs.st = ss->s;
    cs.splitk = splitk_side;
  }
  auto pair = [&](auto&& first, auto&& second) -> int {
    if (!fork) {
      RP_TRY(first(c));
      return second(c);
    }
    if (cudaEventRecord(ss->fork, st) != cudaSuccess || cudaStreamWaitEvent(ss->s, ss->fork, 0) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "xl_block_backward: fork failed");
    RP_TRY(second(cs));
    RP_TRY(first(c));
    if (cudaEventRecord(ss->join, ss->s) != cudaSuccess || cudaStreamWaitEvent(st, ss->join, 0) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "xl_block_backward: join failed");
    return RP_OK;
  };
  // feed-forward + LN2 (as the reference block)
  RP_TRY(mask_grad(dt, g_out, g_h2, N, D, d.drop_seed, static_cast<uint64_t>(n), d.drop_threshold, d.drop_scale,
                   d.drop_enabled, pm, st));
  Epi er;
  er.kind = d.activation == 1 ? RP_EPI_GELU_GRAD : RP_EPI_RELU_GRAD;
  er.resid = d.activation == 1 ? tp.z1 : tp.h1;
  er.ld_resid = F;
  RP_TRY(pair([&](Ctx& x) { return mm(x, mat(g_h2, N, D, D), false, mat(w.w2, F, D, D), false, mat(g_z1, N, F, F), dt, er); },
              [&](Ctx& x) { return mm(x, mat(tp.h1, N, F, F), true, mat(g_h2, N, D, D), true, mat(G.w2, F, D, D), RP_F32); }));
  (void)ld_part;
  // b1 partial sums ride with dW1 on the side stream (both only read g_z1)
  RP_TRY(pair([&](Ctx& x) { return mm(x, mat(g_z1, N, F, F), false, mat(w.w1, D, F, F), false, mat(g_m, N, D, D), RP_F32); },
              [&](Ctx& x) {
                RP_TRY(colsum_partial(dt, g_z1, N, F, F, part, x.st));
                return mm(x, mat(tp.m, N, D, D), true, mat(g_z1, N, F, F), true, mat(G.w1, D, F, F), RP_F32);
              }));
  RP_TRY(layernorm_bwd(dt, g_m, tp.x1, tp.mean2, tp.rstd2, w.ln2_g, g_out, g_x1, g_proj, d.drop_seed,
                       d.drop_threshold, d.drop_scale, d.drop_enabled, pg2, pb2, N, D, st));
  // relative-position attention
  RP_TRY(pair(
      [&](Ctx& cx) {
        RP_TRY(mm(cx, mat(g_proj, N, D, D), false, mat(w.wo, D, D, D), false, mat(g_ctx, N, D, D), dt));
        return xl_split_heads(dt, g_ctx, D, dt, g_ctx_h, N, (int)x.H, (int)x.dh, cx.st);  // beside dWo too
      },
      [&](Ctx& cx) { return mm(cx, mat(tp.ctx, N, D, D), true, mat(g_proj, N, D, D), true, mat(G.wo, D, D, D), RP_F32); }));
  bool dq_done = false;
  if (d.fused & RP_XL_FUSED_DQ) {
    RP_TRY(xl_attn_bwd_dq(g_ctx_h, tp.vh, tp.kh, tp.rh, tp.probs, kv ? nullptr : g_ac, g_bd, x.ldk, g_ctx, tp.ctx,
                          g_qu, g_qv, x.B, x.T, x.M, (int)x.H, (int)x.dh, d.mem_len, scale, st, dq_bias, d_rows,
                          merged ? g_qkv : nullptr));
    dq_done = true;
  } else if (d.fused & RP_XL_FUSED_BWD) {
    RP_TRY(xl_attn_bwd(g_ctx_h, tp.vh, tp.probs, g_ac, g_bd, x.ldk, g_ctx, tp.ctx, x.B, x.T, x.M, (int)x.H, (int)x.dh,
                       d.mem_len, scale, st));
  } else {
    Epi es;
    es.tile_n = d.score_tile;
    RP_TRY(mm(c, bmat(g_ctx_h, x.HB, x.T, x.dh, x.dh, x.T * x.dh), false,
              bmat(tp.vh, x.HB, x.Kl, x.dh, x.dh, x.Kl * x.dh), false, bmat(g_p, x.HB, x.T, x.Kl, x.ldk, x.T * x.ldk),
              RP_F32, es));
    RP_TRY(xl_softmax_bwd(dt, g_p, x.ldk, tp.probs, x.ldk, g_ac, g_bd, x.HB * x.T, x.T, x.M, d.mem_len, scale, st));
  }
  // P^T and dAC^T are banded (key j sees queries i >= j - M): with
  // RP_XL_BANDED the key tiles start their query loop at the first live block
  Epi eband;
  eband.k_lo = (d.fused & RP_XL_BANDED) ? 1 : 0;
  eband.k_lo_off = -x.M;
  // the production path: the key-major dK / dV kernel on this stream, the
  // relative-encoding chain (dR GEMM over dBD, head merge, dWr) on the side
  // stream -- they share no operand
  const bool rel_side = kv && dq_done && dq_bias;
  if (rel_side) {
    RP_TRY(pair(
        [&](Ctx& cx) {
          return xl_attn_bwd_kv(g_ctx_h, tp.vh, tp.qu, tp.probs, x.ldk, d_rows, g_kh, g_vh, x.B, x.T, x.M, (int)x.H,
                                (int)x.dh, d.mem_len, scale, cx.st, merged ? g_qkv : nullptr);
        },
        [&](Ctx& cx) {
          RP_TRY(mm(cx, bmat(g_bd, x.H, N, x.Kl, x.ldk, N * x.ldk), true, bmat(tp.qv, x.H, N, x.dh, x.dh, N * x.dh),
                    true, bmat(g_rh, x.H, x.Kl, x.dh, x.dh, x.Kl * x.dh), RP_F32));
          RP_TRY(xl_merge_heads(RP_F32, g_rh, dt, g_r, D, x.Kl, (int)x.H, (int)x.dh, cx.st));
          return mm(cx, mat(R, x.Kl, D, D), true, mat(g_r, x.Kl, D, D), true, mat(G.wr, D, D, D), RP_F32);
        }));
  } else if (kv)  // dV = P^T dO and dK = dS^T (q+u) in one key-major kernel (no dAC)
    RP_TRY(xl_attn_bwd_kv(g_ctx_h, tp.vh, tp.qu, tp.probs, x.ldk, d_rows, g_kh, g_vh, x.B, x.T, x.M, (int)x.H,
                          (int)x.dh, d.mem_len, scale, st, merged ? g_qkv : nullptr));
  else
    RP_TRY(mm(c, bmat(tp.probs, x.HB, x.T, x.Kl, x.ldk, x.T * x.ldk), true,
              bmat(g_ctx_h, x.HB, x.T, x.dh, x.dh, x.T * x.dh), true, bmat(g_vh, x.HB, x.Kl, x.dh, x.dh, x.Kl * x.dh), dt,
              eband));
  const Mat gac = bmat(g_ac, x.HB, x.T, x.Kl, x.ldk, x.T * x.ldk);
  const Mat gbd = bmat(g_bd, x.H, N, x.Kl, x.ldk, N * x.ldk);
  if (!dq_done)
    RP_TRY(mm(c, gac, false, bmat(tp.kh, x.HB, x.Kl, x.dh, x.dh, x.Kl * x.dh), true,
              bmat(g_qu, x.HB, x.T, x.dh, x.dh, x.T * x.dh), RP_F32));
  if (!kv)
    RP_TRY(mm(c, gac, true, bmat(tp.qu, x.HB, x.T, x.dh, x.dh, x.T * x.dh), true,
              bmat(g_kh, x.HB, x.Kl, x.dh, x.dh, x.Kl * x.dh), dt, eband));
  if (!dq_done)
    RP_TRY(mm(c, gbd, false, bmat(tp.rh, x.H, x.Kl, x.dh, x.dh, x.Kl * x.dh), true,
              bmat(g_qv, x.H, N, x.dh, x.dh, N * x.dh), RP_F32));
  if (!rel_side) {
    RP_TRY(mm(c, gbd, true, bmat(tp.qv, x.H, N, x.dh, x.dh, N * x.dh), true,
              bmat(g_rh, x.H, x.Kl, x.dh, x.dh, x.Kl * x.dh), RP_F32));
    if (!dq_bias)  // else: the fused backward's column sums, finished with the others below
      RP_TRY(xl_bias_grad(g_qu, g_qv, bias_ws, G.r_w_bias, G.r_r_bias, (int)x.H, N, (int)x.dh, st));
    RP_TRY(xl_merge_heads(RP_F32, g_rh, dt, g_r, D, x.Kl, (int)x.H, (int)x.dh, st));
    RP_TRY(mm(c, mat(R, x.Kl, D, D), true, mat(g_r, x.Kl, D, D), true, mat(G.wr, D, D, D), RP_F32));
  }
  if (!merged) RP_TRY(xl_merge_grads(dt, g_qu, g_qv, g_kh, g_vh, g_qkv, x.B, x.T, x.M, (int)x.H, (int)x.dh, st));
  RP_TRY(pair(
      [&](Ctx& x) { return mm(x, mat(g_qkv, BK, 3 * D, 3 * D), false, mat(w.wqkv, D, 3 * D, 3 * D), false, mat(g_a, BK, D, D), RP_F32); },
      [&](Ctx& x) { return mm(x, mat(tp.a, BK, D, D), true, mat(g_qkv, BK, 3 * D, 3 * D), true, mat(G.wqkv, D, 3 * D, 3 * D), RP_F32); }));
  // LN1 over both row blocks: memory rows add to the gain / bias sums only
  // the memory rows take no gradient (stop-gradient): only their gain / bias
  // sums, no dx -- on the side stream beside the current rows' LN1 backward
  RP_TRY(pair(
      [&](Ctx& x) {
        return layernorm_bwd(dt, g_a + BM * D, static_cast<const char*>(tp.xa) + BM * D * e, tp.mean1 + BM,
                             tp.rstd1 + BM, w.ln1_g, g_x1, g_x, nullptr, 0, 0, 1.f, 0, pg, pb, N, D, x.st);
      },
      [&](Ctx& x) {
        return BM ? layernorm_bwd(dt, g_a, tp.xa, tp.mean1, tp.rstd1, w.ln1_g, nullptr, nullptr, nullptr, 0, 0, 1.f,
                                  0, pg + (int64_t)nbl_cur * D, pb + (int64_t)nbl_cur * D, BM, D, x.st)
                  : (int)RP_OK;
      }));
  const int nq = (int)(x.B * (x.T / 128));  // the fused backward's [B*nqt, H*64] bias partials
  const ColsumJob jobs[8] = {{pm, nbm, D, G.b2}, {part, nbc, F, G.b1}, {pg2, nbl_cur, D, G.ln2_g},
                             {pb2, nbl_cur, D, G.ln2_b}, {pg, nbl_cur + nbl_mem, D, G.ln1_g},
                             {pb, nbl_cur + nbl_mem, D, G.ln1_b},
                             {dq_bias, nq, D, G.r_w_bias}, {dq_bias + (int64_t)nq * D, nq, D, G.r_r_bias}};
  return colsum_finish_multi(jobs, dq_bias ? 8 : 6, st);
}

}  // namespace rp
