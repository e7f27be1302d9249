// Token embedding gather/scatter (reference layers.py:114-136) and the
// cross-entropy finish of the tied head (layers.py:287-296, 310-316).
//
// The input-side tied gradient is a scatter-add over token ids
// (np.add.at, layers.py:135).  It is made deterministic without float
// atomics: one CTA bitonic-sorts (token, position) keys in shared memory, then
// runs of equal tokens are summed in position order (chunked, so Zipf-head
// tokens with hundreds of occurrences do not serialise) and beta * sum is
// added into the packet's mixed embedding gradient (engine.py:54-69) whose
// output-side half the head GEMM already wrote.
#include <algorithm>

#include "common.cuh"
#include "rp_internal.h"

namespace rp {

// out[r, :] = (V[tok[r], :] + pos[r % T, :]) * mask(r*d + j)
template <typename T>
__global__ void embed_fwd_kernel(const int64_t* __restrict__ tok, const T* __restrict__ V, const T* __restrict__ pos,
                                 T* __restrict__ out, int64_t rows, int Tn, int d, int64_t vocab, uint64_t seed,
                                 uint64_t thr, float scale, int drop_on, int32_t* flag, int64_t ld) {
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const int64_t id = tok[r];
  const bool ok = id >= 0 && id < vocab;
  if (!ok) {
    if (threadIdx.x == 0 && flag) atomicOr(flag, RP_FLAG_DIMENSION);
  }
  const int t = (int)(r % Tn);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float v = (ok ? to_f(V[id * ld + j]) : 0.f) + to_f(pos[(int64_t)t * ld + j]);
    if (drop_on) v = dropout_keep(seed, (uint64_t)r * d + j, thr) ? v * scale : 0.f;
    out[r * ld + j] = from_f<T>(v);
  }
}

// grad_pos[t, j] = sum_b g[b*T + t, j] * mask ; rows t >= T are zero.
__global__ void embed_pos_grad_kernel(const float* __restrict__ g, float* __restrict__ gpos, int B, int Tn, int Tmax,
                                      int d, uint64_t seed, uint64_t thr, float scale, int drop_on, int64_t ldp) {
  const int t = blockIdx.x;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float s = 0.f;
    if (t < Tn) {
      for (int b = 0; b < B; ++b) {
        const int64_t r = (int64_t)b * Tn + t;
        float v = g[r * d + j];
        if (drop_on) v = dropout_keep(seed, (uint64_t)r * d + j, thr) ? v * scale : 0.f;
        s += v;
      }
    }
    gpos[(int64_t)t * ldp + j] = s;
  }
}

// Sort of (token << 32 | position) keys, in two launches spread over the
// SMs (the keys are unique, so any correct sort gives the same order):
//  1) each CTA bitonic-sorts one chunk of kSortChunk keys in shared memory
//     (padding ~0 sorts last and is never below a real key);
//  2) each key's global rank = its index in its own chunk + the number of
//     keys below it in every other chunk (binary search), and it is stored
//     at that rank.
constexpr int kSortChunk = 1024;

// Ids outside [0, vocab) (the forward raised RP_FLAG_DIMENSION for them) get
// the sentinel token kBadTok: they sort after every valid id and the
// scatter skips them, so a bad id never addresses the tied gradient.
constexpr uint32_t kBadTok = 0xffffffffu;

__global__ void __launch_bounds__(kSortChunk) token_chunk_sort_kernel(const int64_t* __restrict__ tok, int n,
                                                                      int64_t vocab, uint64_t* __restrict__ chunks) {
  __shared__ uint64_t keys[kSortChunk];
  const int i = threadIdx.x, gi = blockIdx.x * kSortChunk + i;
  uint64_t key = ~0ull;
  if (gi < n) {
    const int64_t id = tok[gi];
    const uint32_t tv = (id >= 0 && id < vocab) ? static_cast<uint32_t>(id) : kBadTok;
    key = (static_cast<uint64_t>(tv) << 32) | static_cast<uint32_t>(gi);
  }
  keys[i] = key;
  __syncthreads();
  for (int k = 2; k <= kSortChunk; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int ixj = i ^ j;
      if (ixj > i) {
        const bool up = (i & k) == 0;
        const uint64_t a = keys[i], b = keys[ixj];
        if ((a > b) == up) {
          keys[i] = b;
          keys[ixj] = a;
        }
      }
      __syncthreads();
    }
  }
  chunks[gi] = keys[i];
}

__global__ void token_rank_kernel(const uint64_t* __restrict__ chunks, int n, int nchunk,
                                  uint64_t* __restrict__ sorted) {
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= n) return;  // chunk-sorted padding sits at indices >= n
  const uint64_t key = chunks[gi];
  const int mine = gi / kSortChunk;
  int rank = gi - mine * kSortChunk;
  for (int c = 0; c < nchunk; ++c) {
    if (c == mine) continue;
    const uint64_t* ch = chunks + (int64_t)c * kSortChunk;
    int lo = 0, hi = kSortChunk;  // first index with ch[idx] >= key
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ch[mid] < key) lo = mid + 1; else hi = mid;
    }
    rank += lo;
  }
  sorted[rank] = key;
}

// Deterministic scatter-sum of masked gradient rows into the tied gradient,
// in two passes so hot (Zipf-head) tokens do not serialise on one warp:
//  1) chunk c of kChunk sorted positions: per column, sum each run of equal
//     tokens inside the chunk in position order -> partial[first position];
//  2) per run start (segment of equal tokens): add the chunk partials of the
//     segment in chunk order, emb[tok] += beta * total.
constexpr int kChunk = 32;

__global__ void embed_chunk_partial_kernel(const uint64_t* __restrict__ sorted, int n, const float* __restrict__ g,
                                           int d, uint64_t seed, uint64_t thr, float scale, int drop_on,
                                           float* __restrict__ partial) {
  __shared__ uint32_t tok_s[kChunk];
  __shared__ uint32_t row_s[kChunk];
  const int c0 = blockIdx.x * kChunk;
  const int len = min(kChunk, n - c0);
  if (threadIdx.x < len) {
    tok_s[threadIdx.x] = static_cast<uint32_t>(sorted[c0 + threadIdx.x] >> 32);
    row_s[threadIdx.x] = static_cast<uint32_t>(sorted[c0 + threadIdx.x] & 0xffffffffu);
  }
  __syncthreads();
  for (int j = blockIdx.y * blockDim.x + threadIdx.x; j < d; j += gridDim.y * blockDim.x) {
    float acc = 0.f;
    int start = 0;
    for (int q = 0; q < len; ++q) {
      const int64_t r = row_s[q];
      float v = g[r * d + j];
      if (drop_on) v = dropout_keep(seed, (uint64_t)r * d + j, thr) ? v * scale : 0.f;
      acc += v;
      if (q + 1 == len || tok_s[q + 1] != tok_s[q]) {
        partial[(int64_t)(c0 + start) * d + j] = acc;
        acc = 0.f;
        start = q + 1;
      }
    }
  }
}

__global__ void embed_segment_kernel(const uint64_t* __restrict__ sorted, int n, const float* __restrict__ partial,
                                     int d, float beta, float* __restrict__ emb, int64_t lde) {
  const int i = blockIdx.x;
  const uint32_t tokv = static_cast<uint32_t>(sorted[i] >> 32);
  if (tokv == kBadTok || (i > 0 && static_cast<uint32_t>(sorted[i - 1] >> 32) == tokv)) return;
  int end = i + 1;
  // segment end: first position with a different token (scan chunk starts)
  while (end < n && static_cast<uint32_t>(sorted[end] >> 32) == tokv) {
    const int next_chunk = (end / kChunk + 1) * kChunk;
    if (next_chunk < n && static_cast<uint32_t>(sorted[next_chunk - 1] >> 32) == tokv) {
      end = next_chunk;
    } else {
      ++end;
    }
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float total = partial[(int64_t)i * d + j];
    for (int c = (i / kChunk + 1) * kChunk; c < end; c += kChunk) total += partial[(int64_t)c * d + j];
    emb[(int64_t)tokv * lde + j] += beta * total;
  }
}

// ---------------------------------------------------------------------------
// cross-entropy finish: lse per row from the head GEMM's (max, sumexp)
// partials, per-row loss lse - z_y, then a fixed-order mean.
// one warp per row: lanes stride over the row's n-tile partials (coalesced)
__global__ void ce_rows_kernel(const float* __restrict__ partial, int ntiles, const float* __restrict__ zy,
                               const int64_t* __restrict__ tgt, int64_t vocab, int64_t rows, float* __restrict__ lse,
                               float* __restrict__ loss_rows, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (m >= rows) return;
  const float2* p = reinterpret_cast<const float2*>(partial + m * ntiles * 2);
  float mx = -INFINITY;
  for (int t = lane; t < ntiles; t += 32) mx = fmaxf(mx, p[t].x);
  mx = warp_max(mx);
  float s = 0.f;
  for (int t = lane; t < ntiles; t += 32) {
    const float2 v = p[t];
    s += v.y * __expf(v.x - mx);
  }
  s = warp_sum(s);
  if (lane == 0) {
    const float l = mx + logf(s);
    lse[m] = l;
    loss_rows[m] = l - zy[m];
    const int64_t y = tgt[m];
    if (flag) {
      if (y < 0 || y >= vocab) atomicOr(flag, RP_FLAG_DIMENSION);
      if (!isfinite(l)) atomicOr(flag, RP_FLAG_NONFINITE);
    }
  }
}

__global__ void __launch_bounds__(1024) mean_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ out,
                                                    double* __restrict__ out64) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double mean = n ? red[0] / (double)n : 0.0;
    if (out) *out = (float)mean;
    if (out64) *out64 = mean;
  }
}

// ---------------------------------------------------------------------------
#define RP_DT(DT, ...)              \
  if ((DT) == RP_BF16) {            \
    using T = __nv_bfloat16;        \
    __VA_ARGS__;                    \
  } else {                          \
    using T = float;                \
    __VA_ARGS__;                    \
  }

int embed_fwd(int dtype, const int64_t* tok, const void* V, const void* pos, void* out, int64_t B, int64_t Tn,
              int64_t d, int64_t vocab, uint64_t seed, uint64_t thr, float scale, int drop_on, int32_t* flag,
              cudaStream_t st, int64_t ld) {
  const int64_t rows = B * Tn;
  if (rows == 0) return RP_OK;
  if (ld <= 0) ld = d;
  const int threads = (int)std::min<int64_t>(256, ((d + 31) / 32) * 32);
  RP_DT(dtype, embed_fwd_kernel<T><<<(unsigned)rows, threads, 0, st>>>(tok, (const T*)V, (const T*)pos, (T*)out,
                                                                       rows, (int)Tn, (int)d, vocab, seed, thr,
                                                                       scale, drop_on, flag, ld));
  return check_launch("embed_fwd");
}

// [sorted keys, padded to 256 B][row partials n*d fp32; the chunk-sorted keys
// of the token sort live here first (consumed before the partials are written)]
int64_t embed_bwd_workspace_bytes(int64_t n_tokens, int64_t d) {
  const int64_t chunks = (n_tokens + kSortChunk - 1) / kSortChunk * kSortChunk * 8;
  return ((n_tokens * 8 + 255) / 256) * 256 + std::max<int64_t>(n_tokens * d * 4, chunks);
}

int embed_bwd(const float* g, const int64_t* tok, int64_t B, int64_t Tn, int64_t Tmax, int64_t d, int64_t vocab,
              uint64_t seed,
              uint64_t thr, float scale, int drop_on, float* gpos, float* emb, float beta, void* workspace,
              cudaStream_t st, int64_t ld_out) {
  if (ld_out <= 0) ld_out = d;
  uint64_t* work = static_cast<uint64_t*>(workspace);
  float* partial = reinterpret_cast<float*>(static_cast<char*>(workspace) + ((B * Tn * 8 + 255) / 256) * 256);
  const int64_t n = B * Tn;
  const int threads = (int)std::min<int64_t>(256, ((d + 31) / 32) * 32);
  if (gpos) {
    embed_pos_grad_kernel<<<(unsigned)Tmax, threads, 0, st>>>(g, gpos, (int)B, (int)Tn, (int)Tmax, (int)d, seed, thr,
                                                              scale, drop_on, ld_out);
    if (int e = check_launch("embed_pos_grad")) return e;
  }
  if (!emb || n == 0) return RP_OK;
  if (n > INT32_MAX) return set_error(RP_ERR_DIMENSION, "embed_bwd: %lld tokens", (long long)n);
  if (vocab <= 0 || vocab >= (int64_t)kBadTok) return set_error(RP_ERR_DIMENSION, "embed_bwd: vocab %lld", (long long)vocab);
  const int nsort = (int)((n + kSortChunk - 1) / kSortChunk);
  uint64_t* chunks = reinterpret_cast<uint64_t*>(partial);
  token_chunk_sort_kernel<<<(unsigned)nsort, kSortChunk, 0, st>>>(tok, (int)n, vocab, chunks);
  if (int e = check_launch("token_chunk_sort")) return e;
  token_rank_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(chunks, (int)n, nsort, work);
  if (int e = check_launch("token_rank")) return e;
  const int nchunk = (int)((n + kChunk - 1) / kChunk);
  const int tpb = (int)std::min<int64_t>(256, ((d + 31) / 32) * 32);
  dim3 grid(nchunk, (unsigned)std::max<int64_t>(1, (d + tpb - 1) / tpb));
  embed_chunk_partial_kernel<<<grid, tpb, 0, st>>>(work, (int)n, g, (int)d, seed, thr, scale, drop_on, partial);
  if (int e = check_launch("embed_chunk_partial")) return e;
  embed_segment_kernel<<<(unsigned)n, tpb, 0, st>>>(work, (int)n, partial, (int)d, beta, emb, ld_out);
  return check_launch("embed_segment");
}

int ce_finish(const float* partial, int ntiles, const float* zy, const int64_t* tgt, int64_t vocab, int64_t rows,
              float* lse, float* loss_rows, float* loss, double* loss64, int32_t* flag, cudaStream_t st) {
  if (rows == 0) return RP_OK;
  ce_rows_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(partial, ntiles, zy, tgt, vocab, rows, lse,
                                                                       loss_rows, flag);
  if (int e = check_launch("ce_rows")) return e;
  mean_kernel<<<1, 1024, 0, st>>>(loss_rows, rows, loss, loss64);
  return check_launch("ce_mean");
}

}  // namespace rp
