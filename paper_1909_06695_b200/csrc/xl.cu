// Transformer-XL attention glue (restated in oracle/xl.py
// from Dai et al. 2019 -- the reference has no XL path, so parity is pinned
// by the fp64 restatement's reduction and finite-difference tests).
//
// The contractions (AC = (q+u) k^T, BD = (q+v) r^T, P v and their backward
// GEMMs) run on the tcgen05 GEMM over head-major operands; these kernels do
// the HBM-bound remainder:
//   * head split of the fused QKV rows of [mem; x] with the u / v biases,
//   * the relative-shift softmax (reads AC and the unshifted BD rows,
//     applies the causal + memory-validity mask) and its backward, which
//     writes dAC and the un-shifted dBD rows for the two backward GEMMs,
//   * head merges, the fused dQ/dK/dV merge into the [mem; x] row layout,
//   * deterministic per-head column sums for the u / v gradients.
//
// Row layout of the concatenated block input ("xa"): the B*M memory rows
// first (row b*M + j), then the B*T current rows (row B*M + b*T + i); key j
// of batch b is memory row j (j < M) or current row j - M.
// Head-major layouts: qu, qv [H, B, T, dh]; kh, vh [H, B, Kl, dh] with
// Kl = M + T; r_h [H, Kl, dh]; score rows (h, b, i) of length Kl (ld >= Kl).
#include <algorithm>

#include "common.cuh"
#include "rp_internal.h"

namespace rp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

inline int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 64); }

__device__ __forceinline__ int64_t key_row(int64_t b, int64_t j, int64_t B, int64_t T, int64_t M) {
  return j < M ? b * M + j : B * M + b * T + (j - M);
}

template <typename T>
__global__ void split_qkv_kernel(const T* __restrict__ qkv, const float* __restrict__ u, const float* __restrict__ v,
                                 T* __restrict__ qu, T* __restrict__ qv, T* __restrict__ kh, T* __restrict__ vh,
                                 int64_t B, int64_t Tn, int64_t M, int H, int dh) {
  const int64_t Kl = M + Tn;
  const int64_t d = (int64_t)H * dh;
  const int64_t total = (int64_t)H * B * Kl * dh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % dh);
    int64_t r = e / dh;
    const int64_t j = r % Kl;
    r /= Kl;
    const int64_t b = r % B;
    const int h = (int)(r / B);
    const T* src = qkv + key_row(b, j, B, Tn, M) * 3 * d + (int64_t)h * dh + c;
    kh[e] = src[d];
    vh[e] = src[2 * d];
    if (j >= M) {
      const float q = to_f(src[0]);
      const int64_t o = (((int64_t)h * B + b) * Tn + (j - M)) * dh + c;
      qu[o] = from_f<T>(q + u[h * dh + c]);
      qv[o] = from_f<T>(q + v[h * dh + c]);
    }
  }
}

template <typename S, typename D>
__global__ void split_heads_kernel(const S* __restrict__ src, int64_t ld, D* __restrict__ dst, int64_t rows, int H,
                                   int dh) {
  const int64_t total = rows * H * dh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % dh);
    const int64_t r = (e / dh) % rows;
    const int h = (int)(e / (dh * rows));
    dst[e] = from_f<D>(to_f(src[r * ld + (int64_t)h * dh + c]));
  }
}

template <typename S, typename D>
__global__ void merge_heads_kernel(const S* __restrict__ src, D* __restrict__ dst, int64_t ld, int64_t rows, int H,
                                   int dh) {
  const int64_t d = (int64_t)H * dh;
  const int64_t total = rows * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int col = (int)(e % d);
    const int h = col / dh, c = col % dh;
    dst[r * ld + col] = from_f<D>(to_f(src[((int64_t)h * rows + r) * dh + c]));
  }
}

// g_qkv rows in the xa layout: q columns = dQu + dQv (zero on memory rows),
// k / v columns from the head-major key gradients.
template <typename T>
__global__ void merge_grads_kernel(const float* __restrict__ gqu, const float* __restrict__ gqv,
                                   const float* __restrict__ gkh, const float* __restrict__ gvh, T* __restrict__ gqkv,
                                   int64_t B, int64_t Tn, int64_t M, int H, int dh) {
  const int64_t Kl = M + Tn;
  const int64_t d = (int64_t)H * dh;
  const int64_t total = B * Kl * 3 * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / (3 * d);
    const int col = (int)(e % (3 * d));
    const int part = col / (int)d;
    const int h = (col % (int)d) / dh, c = col % dh;
    int64_t b, j;
    if (row < B * M) {
      b = row / M;
      j = row % M;
    } else {
      b = (row - B * M) / Tn;
      j = M + (row - B * M) % Tn;
    }
    float g;
    if (part == 0) {
      if (j < M) {
        g = 0.f;
      } else {
        const int64_t o = (((int64_t)h * B + b) * Tn + (j - M)) * dh + c;
        g = gqu[o] + gqv[o];
      }
    } else {
      const int64_t o = (((int64_t)h * B + b) * Kl + j) * dh + c;
      g = part == 1 ? gkh[o] : gvh[o];
    }
    gqkv[e] = from_f<T>(g);
  }
}

// One warp per score row (h, b, i): s_j = (AC[j] + BD[T-1-i+j]) * scale for
// M - mem_len <= j <= M + i, softmax, P written up to ldp (zeros elsewhere).
template <typename T, int NPL>
__global__ void __launch_bounds__(kThreads) softmax_fwd_kernel(const float* __restrict__ ac,
                                                                const float* __restrict__ bd, int64_t lds,
                                                                T* __restrict__ p, int64_t ldp, int64_t rows, int Tn,
                                                                int M, int mem_len, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int i = (int)(row % Tn);
  const int lo = M - mem_len, hi = M + i, off = Tn - 1 - i;
  const float* a = ac + row * lds;
  const float* r = bd + row * lds + off;
  float s[NPL];
  float mx = -INFINITY;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    s[q] = (j >= lo && j <= hi) ? (a[j] + r[j]) * scale : -INFINITY;
    mx = fmaxf(mx, s[q]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    s[q] = (j >= lo && j <= hi) ? __expf(s[q] - mx) : 0.f;
    sum += s[q];
  }
  const float inv = 1.f / warp_sum(sum);
  T* pr = p + row * ldp;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    if (j < ldp) pr[j] = from_f<T>(s[q] * inv);
  }
}

// dS = P (dP - <dP, P>) * scale; writes dAC = dS and the un-shifted
// dBD[p] = dS[p - (T-1-i)] (zero where no key maps to p).
template <typename T, int NPL>
__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(const float* __restrict__ gp, int64_t lds,
                                                                const T* __restrict__ p, int64_t ldp,
                                                                T* __restrict__ gac, T* __restrict__ gbd,
                                                                int64_t rows, int Tn, int M, int mem_len,
                                                                float scale) {
  extern __shared__ float sh_gs[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kWarps + warp;
  if (row >= rows) return;
  float* gs_row = sh_gs + warp * (32 * NPL);
  const int i = (int)(row % Tn);
  const int lo = M - mem_len, hi = M + i, off = Tn - 1 - i;
  const float* g = gp + row * lds;
  const T* pr = p + row * ldp;
  float pv[NPL], gv[NPL];
  float dot = 0.f;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    const bool ok = j >= lo && j <= hi;
    pv[q] = ok ? to_f(pr[j]) : 0.f;
    gv[q] = ok ? g[j] : 0.f;
    dot += pv[q] * gv[q];
  }
  dot = warp_sum(dot);
  T* ga = gac + row * ldp;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    const float v = pv[q] * (gv[q] - dot) * scale;
    gs_row[j] = v;
    if (j < ldp) ga[j] = from_f<T>(v);
  }
  __syncwarp();
  T* gb = gbd + row * ldp;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int pcol = lane + 32 * q;
    const int j = pcol - off;
    if (pcol < ldp) gb[pcol] = from_f<T>((j >= 0 && j < 32 * NPL) ? gs_row[j] : 0.f);
  }
}

// Per-head column sums of two [H, R, dh] fp32 arrays, deterministic:
// stage 1 writes part[src][h][chunk][c], stage 2 sums chunks in order.
constexpr int kBiasChunks = 64;

__global__ void bias_partial_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ part,
                                    int H, int64_t R, int dh) {
  __shared__ float red[kThreads];
  const int chunk = blockIdx.x, h = blockIdx.y, which = blockIdx.z;
  const float* src = (which ? b : a) + (int64_t)h * R * dh;
  const int groups = kThreads / dh;
  const int c = threadIdx.x % dh, gi = threadIdx.x / dh;
  const int64_t per = (R + kBiasChunks - 1) / kBiasChunks;
  const int64_t r0 = chunk * per;
  const int64_t r1 = (r0 + per < R) ? r0 + per : R;
  float acc = 0.f;
  if (gi < groups)
    for (int64_t r = r0 + gi; r < r1; r += groups) acc += src[r * dh + c];
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < dh) {
    float s = 0.f;
    for (int k = 0; k < groups; ++k) s += red[k * dh + threadIdx.x];
    part[(((int64_t)which * H + h) * kBiasChunks + chunk) * dh + threadIdx.x] = s;
  }
}

__global__ void bias_finish_kernel(const float* __restrict__ part, float* __restrict__ out_a,
                                   float* __restrict__ out_b, int H, int dh) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * H * dh) return;
  const int which = e / (H * dh), h = (e / dh) % H, c = e % dh;
  const float* p = part + (((int64_t)which * H + h) * kBiasChunks) * dh + c;
  float s = 0.f;
  for (int k = 0; k < kBiasChunks; ++k) s += p[(int64_t)k * dh];
  (which ? out_b : out_a)[h * dh + c] = s;
}

inline int npl_for(int64_t n) {
  if (n <= 64) return 2;
  if (n <= 128) return 4;
  if (n <= 256) return 8;
  if (n <= 512) return 16;
  if (n <= 1024) return 32;
  if (n <= 2048) return 64;
  return -1;
}

}  // namespace

#define XL_DTYPE(DT, ...)          \
  if ((DT) == RP_BF16) {           \
    using T = __nv_bfloat16;       \
    __VA_ARGS__;                   \
  } else {                         \
    using T = float;               \
    __VA_ARGS__;                   \
  }

#define XL_NPL(NPL_VAL, ...)                                             \
  switch (NPL_VAL) {                                                     \
    case 2: { constexpr int NPL = 2; __VA_ARGS__; break; }               \
    case 4: { constexpr int NPL = 4; __VA_ARGS__; break; }               \
    case 8: { constexpr int NPL = 8; __VA_ARGS__; break; }               \
    case 16: { constexpr int NPL = 16; __VA_ARGS__; break; }             \
    case 32: { constexpr int NPL = 32; __VA_ARGS__; break; }             \
    case 64: { constexpr int NPL = 64; __VA_ARGS__; break; }             \
    default: return set_error(RP_ERR_DIMENSION, "XL key length too large"); \
  }

int xl_split_qkv(int dtype, const void* qkv, const float* u, const float* v, void* qu, void* qv, void* kh, void* vh,
                 int64_t B, int64_t Tn, int64_t M, int H, int dh, cudaStream_t st) {
  const int64_t n = (int64_t)H * B * (M + Tn) * dh;
  if (n == 0) return RP_OK;
  XL_DTYPE(dtype, split_qkv_kernel<T><<<blocks_for(n), kThreads, 0, st>>>(
                      (const T*)qkv, u, v, (T*)qu, (T*)qv, (T*)kh, (T*)vh, B, Tn, M, H, dh));
  return check_launch("xl_split_qkv");
}

int xl_split_heads(int src_dtype, const void* src, int64_t ld, int dst_dtype, void* dst, int64_t rows, int H, int dh,
                   cudaStream_t st) {
  const int64_t n = rows * H * dh;
  if (n == 0) return RP_OK;
  const int g = blocks_for(n);
  if (src_dtype == RP_BF16 && dst_dtype == RP_BF16)
    split_heads_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, ld, (__nv_bfloat16*)dst, rows, H, dh);
  else if (src_dtype == RP_F32 && dst_dtype == RP_BF16)
    split_heads_kernel<<<g, kThreads, 0, st>>>((const float*)src, ld, (__nv_bfloat16*)dst, rows, H, dh);
  else if (src_dtype == RP_BF16 && dst_dtype == RP_F32)
    split_heads_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, ld, (float*)dst, rows, H, dh);
  else
    split_heads_kernel<<<g, kThreads, 0, st>>>((const float*)src, ld, (float*)dst, rows, H, dh);
  return check_launch("xl_split_heads");
}

int xl_merge_heads(int src_dtype, const void* src, int dst_dtype, void* dst, int64_t ld, int64_t rows, int H, int dh,
                   cudaStream_t st) {
  const int64_t n = rows * H * dh;
  if (n == 0) return RP_OK;
  const int g = blocks_for(n);
  if (src_dtype == RP_BF16 && dst_dtype == RP_BF16)
    merge_heads_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, ld, rows, H, dh);
  else if (src_dtype == RP_F32 && dst_dtype == RP_BF16)
    merge_heads_kernel<<<g, kThreads, 0, st>>>((const float*)src, (__nv_bfloat16*)dst, ld, rows, H, dh);
  else if (src_dtype == RP_BF16 && dst_dtype == RP_F32)
    merge_heads_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, (float*)dst, ld, rows, H, dh);
  else
    merge_heads_kernel<<<g, kThreads, 0, st>>>((const float*)src, (float*)dst, ld, rows, H, dh);
  return check_launch("xl_merge_heads");
}

int xl_merge_grads(int dtype, const float* gqu, const float* gqv, const float* gkh, const float* gvh, void* gqkv,
                   int64_t B, int64_t Tn, int64_t M, int H, int dh, cudaStream_t st) {
  const int64_t n = B * (M + Tn) * 3 * (int64_t)H * dh;
  if (n == 0) return RP_OK;
  XL_DTYPE(dtype, merge_grads_kernel<T><<<blocks_for(n), kThreads, 0, st>>>(gqu, gqv, gkh, gvh, (T*)gqkv, B, Tn, M,
                                                                           H, dh));
  return check_launch("xl_merge_grads");
}

int xl_softmax_fwd(int dtype, const float* ac, const float* bd, int64_t lds, void* p, int64_t ldp, int64_t rows,
                   int64_t Tn, int64_t M, int64_t mem_len, float scale, cudaStream_t st) {
  if (rows == 0) return RP_OK;
  if (mem_len < 0 || mem_len > M || ldp < M + Tn || lds < M + Tn)
    return set_error(RP_ERR_DIMENSION, "xl_softmax_fwd: bad memory length or leading dimension");
  const int npl = npl_for(ldp);
  const int g = (int)((rows + kWarps - 1) / kWarps);
  XL_DTYPE(dtype, XL_NPL(npl, softmax_fwd_kernel<T, NPL><<<g, kThreads, 0, st>>>(
                                  ac, bd, lds, (T*)p, ldp, rows, (int)Tn, (int)M, (int)mem_len, scale)));
  return check_launch("xl_softmax_fwd");
}

int xl_softmax_bwd(int dtype, const float* gp, int64_t lds, const void* p, int64_t ldp, void* gac, void* gbd,
                   int64_t rows, int64_t Tn, int64_t M, int64_t mem_len, float scale, cudaStream_t st) {
  if (rows == 0) return RP_OK;
  if (mem_len < 0 || mem_len > M || ldp < M + Tn || lds < M + Tn)
    return set_error(RP_ERR_DIMENSION, "xl_softmax_bwd: bad memory length or leading dimension");
  const int npl = npl_for(ldp);
  const int g = (int)((rows + kWarps - 1) / kWarps);
  XL_DTYPE(dtype, XL_NPL(npl, {
    const size_t smem = sizeof(float) * kWarps * 32 * NPL;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(softmax_bwd_kernel<T, NPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    softmax_bwd_kernel<T, NPL><<<g, kThreads, smem, st>>>(gp, lds, (const T*)p, ldp, (T*)gac, (T*)gbd, rows,
                                                          (int)Tn, (int)M, (int)mem_len, scale);
  }));
  return check_launch("xl_softmax_bwd");
}

int64_t xl_bias_grad_workspace_bytes(int H, int dh) { return (int64_t)2 * H * kBiasChunks * dh * sizeof(float); }

int xl_bias_grad(const float* gqu, const float* gqv, float* part, float* gu, float* gv, int H, int64_t R, int dh,
                 cudaStream_t st) {
  if (dh > kThreads || kThreads % dh) return set_error(RP_ERR_DIMENSION, "xl_bias_grad: head dim must divide 256");
  bias_partial_kernel<<<dim3(kBiasChunks, H, 2), kThreads, 0, st>>>(gqu, gqv, part, H, R, dh);
  bias_finish_kernel<<<(2 * H * dh + kThreads - 1) / kThreads, kThreads, 0, st>>>(part, gu, gv, H, dh);
  return check_launch("xl_bias_grad");
}

}  // namespace rp
