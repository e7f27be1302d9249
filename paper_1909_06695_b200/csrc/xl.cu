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

// 8 consecutive elements as fp32 (16 B of bf16 / 32 B of fp32); every head
// dimension is a multiple of 8, so each vector stays inside one head row and
// both sides of a head permute are 16-byte aligned and coalesced.
template <typename T> struct V8;
template <> struct V8<__nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
      v[2 * k] = f.x;
      v[2 * k + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
      w[k] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct V8<float> {
  static __device__ __forceinline__ void ld(const float* p, float (&v)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void st(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

#define XL_GRID_LOOP(e, total) \
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (total); e += (int64_t)gridDim.x * blockDim.x)

// unit e = ((h*B + b)*Kl + j)*C + c8, C = dh/8
template <typename T>
__global__ void split_qkv_kernel(const T* __restrict__ qkv, const float* __restrict__ u, const float* __restrict__ v,
                                 T* __restrict__ qu, T* __restrict__ qv, T* __restrict__ kh, T* __restrict__ vh,
                                 int B, int Tn, int M, int H, int dh) {
  const int Kl = M + Tn, C = dh / 8, d = H * dh;
  const int64_t total = (int64_t)H * B * Kl * C;
  XL_GRID_LOOP(e, total) {
    const int c = (int)(e % C) * 8;
    const int64_t hbj = e / C;
    const int j = (int)(hbj % Kl);
    const int hb = (int)(hbj / Kl);
    const int b = hb % B, h = hb / B;
    const T* src = qkv + key_row(b, j, B, Tn, M) * 3 * d + h * dh + c;
    float x[8];
    V8<T>::ld(src + d, x);
    V8<T>::st(kh + hbj * dh + c, x);
    V8<T>::ld(src + 2 * d, x);
    V8<T>::st(vh + hbj * dh + c, x);
    if (j >= M) {
      V8<T>::ld(src, x);
      float y[8];
      const float* uu = u + h * dh + c;
      const float* vv = v + h * dh + c;
#pragma unroll
      for (int k = 0; k < 8; ++k) y[k] = x[k] + uu[k];
      const int64_t o = ((int64_t)hb * Tn + (j - M)) * dh + c;
      V8<T>::st(qu + o, y);
#pragma unroll
      for (int k = 0; k < 8; ++k) y[k] = x[k] + vv[k];
      V8<T>::st(qv + o, y);
    }
  }
}

// dst[h, r, c] = src[r*ld + h*dh + c]; unit e = (h*rows + r)*C + c8
template <typename S, typename D>
__global__ void split_heads_kernel(const S* __restrict__ src, int64_t ld, D* __restrict__ dst, int64_t rows, int H,
                                   int dh) {
  const int C = dh / 8;
  XL_GRID_LOOP(e, rows * H * C) {
    const int c = (int)(e % C) * 8;
    const int64_t hr = e / C;
    const int64_t r = hr % rows;
    const int h = (int)(hr / rows);
    float x[8];
    V8<S>::ld(src + r * ld + h * dh + c, x);
    V8<D>::st(dst + hr * dh + c, x);
  }
}

// dst[r*ld + h*dh + c] = src[h, r, c]; unit e = (r*H + h)*C + c8 (row-major writes)
template <typename S, typename D>
__global__ void merge_heads_kernel(const S* __restrict__ src, D* __restrict__ dst, int64_t ld, int64_t rows, int H,
                                   int dh) {
  const int C = dh / 8;
  XL_GRID_LOOP(e, rows * H * C) {
    const int c = (int)(e % C) * 8;
    const int64_t rh = e / C;
    const int h = (int)(rh % H);
    const int64_t r = rh / H;
    float x[8];
    V8<S>::ld(src + ((int64_t)h * rows + r) * dh + c, x);
    V8<D>::st(dst + r * ld + h * dh + c, x);
  }
}

// Row-block forms of the head split / merge kernels for any head dim and
// row pitches (d or the head dim not a multiple of 8, e.g. BASELINE
// configs[3]: d 410 = 10 heads x 41; bf16 rows are padded to 16-byte pitches,
// so row r starts at r * ld).  One CTA per row (grid-stride over rows): the
// row's coordinates are decoded once, the threads sweep its columns with
// 32-bit index math, and the row-major side is read / written coalesced.
constexpr int kRowBlk = 128;

inline int row_grid(int64_t rows) { return (int)std::min<int64_t>(rows, 148 * 32); }

__device__ __forceinline__ void key_coords(int64_t row, int B, int Tn, int M, int& b, int& j) {
  const int64_t BM = (int64_t)B * M;
  if (row < BM) {
    b = (int)(row / M);
    j = (int)(row - (int64_t)b * M);
  } else {
    const int64_t r = row - BM;
    b = (int)(r / Tn);
    j = M + (int)(r - (int64_t)b * Tn);
  }
}

// qkv row (b, j) in the xa layout -> kh, vh [H, B, Kl, ldh]; current rows also
// -> qu = q + u, qv = q + v [H, B, T, ldh]
template <typename T>
__global__ void __launch_bounds__(kRowBlk) split_qkv_rows_kernel(
    const T* __restrict__ qkv, const float* __restrict__ u, const float* __restrict__ v, T* __restrict__ qu,
    T* __restrict__ qv, T* __restrict__ kh, T* __restrict__ vh, int B, int Tn, int M, int H, int dh, int64_t ldq,
    int64_t ldh) {
  const int Kl = M + Tn, d = H * dh;
  const int64_t rows = (int64_t)B * Kl;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    int b, j;
    key_coords(row, B, Tn, M, b, j);
    const T* src = qkv + row * ldq;
    for (int col = threadIdx.x; col < d; col += kRowBlk) {
      const int h = col / dh, c = col - h * dh;
      const int64_t hb = (int64_t)h * B + b;
      kh[(hb * Kl + j) * ldh + c] = src[d + col];
      vh[(hb * Kl + j) * ldh + c] = src[2 * d + col];
      if (j >= M) {
        const float x = to_f(src[col]);
        const int64_t o = (hb * Tn + (j - M)) * ldh + c;
        qu[o] = from_f<T>(x + u[col]);
        qv[o] = from_f<T>(x + v[col]);
      }
    }
  }
}

// dst[h, r, c] (pitch ldh) = src[r*ld + h*dh + c]
template <typename S, typename D>
__global__ void __launch_bounds__(kRowBlk) split_heads_rows_kernel(const S* __restrict__ src, int64_t ld,
                                                                    D* __restrict__ dst, int64_t rows, int H, int dh,
                                                                    int64_t ldh) {
  const int d = H * dh;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    for (int col = threadIdx.x; col < d; col += kRowBlk) {
      const int h = col / dh, c = col - h * dh;
      dst[((int64_t)h * rows + r) * ldh + c] = from_f<D>(to_f(src[r * ld + col]));
    }
  }
}

// dst[r*ld + h*dh + c] = src[h, r, c] (pitch ldh)
template <typename S, typename D>
__global__ void __launch_bounds__(kRowBlk) merge_heads_rows_kernel(const S* __restrict__ src, D* __restrict__ dst,
                                                                    int64_t ld, int64_t rows, int H, int dh,
                                                                    int64_t ldh) {
  const int d = H * dh;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    for (int col = threadIdx.x; col < d; col += kRowBlk) {
      const int h = col / dh, c = col - h * dh;
      dst[r * ld + col] = from_f<D>(to_f(src[((int64_t)h * rows + r) * ldh + c]));
    }
  }
}

// g_qkv row (b, j) (pitch ldq) from the head-major fp32 gradients (pitch ldg)
template <typename T>
__global__ void __launch_bounds__(kRowBlk) merge_grads_rows_kernel(
    const float* __restrict__ gqu, const float* __restrict__ gqv, const T* __restrict__ gkh,
    const T* __restrict__ gvh, T* __restrict__ gqkv, int B, int Tn, int M, int H, int dh, int64_t ldq,
    int64_t ldg, int64_t ldkv) {
  const int Kl = M + Tn, d = H * dh;
  const int64_t rows = (int64_t)B * Kl;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    int b, j;
    key_coords(row, B, Tn, M, b, j);
    T* dst = gqkv + row * ldq;
    for (int col = threadIdx.x; col < d; col += kRowBlk) {
      const int h = col / dh, c = col - h * dh;
      const int64_t hb = (int64_t)h * B + b;
      float q = 0.f;
      if (j >= M) {
        const int64_t o = (hb * Tn + (j - M)) * ldg + c;
        q = gqu[o] + gqv[o];
      }
      const int64_t ok = (hb * Kl + j) * ldkv + c;
      dst[col] = from_f<T>(q);
      dst[d + col] = gkh[ok];
      dst[2 * d + col] = gvh[ok];
    }
  }
}

// g_qkv rows in the xa layout: q columns = dQu + dQv (zero on memory rows),
// k / v columns from the head-major key gradients.  unit = 8 columns of a row.
template <typename T>
__global__ void merge_grads_kernel(const float* __restrict__ gqu, const float* __restrict__ gqv,
                                   const T* __restrict__ gkh, const T* __restrict__ gvh, T* __restrict__ gqkv,
                                   int B, int Tn, int M, int H, int dh) {
  const int Kl = M + Tn, d = H * dh, C3 = 3 * d / 8;
  const int64_t BM = (int64_t)B * M;
  XL_GRID_LOOP(e, (int64_t)B * Kl * C3) {
    const int64_t row = e / C3;
    const int col = (int)(e % C3) * 8;
    const int part = col / d;
    const int h = (col % d) / dh, c = col % dh;
    int b, j;
    if (row < BM) {
      b = (int)(row / M);
      j = (int)(row % M);
    } else {
      b = (int)((row - BM) / Tn);
      j = M + (int)((row - BM) % Tn);
    }
    float g[8];
    if (part == 0) {
      if (j < M) {
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] = 0.f;
      } else {
        const int64_t o = (((int64_t)h * B + b) * Tn + (j - M)) * dh + c;
        float g2[8];
        V8<float>::ld(gqu + o, g);
        V8<float>::ld(gqv + o, g2);
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] += g2[k];
      }
    } else {
      const int64_t o = (((int64_t)h * B + b) * Kl + j) * dh + c;
      V8<T>::ld((part == 1 ? gkh : gvh) + o, g);
    }
    V8<T>::st(gqkv + row * 3 * d + col, g);
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

// 4-wide row access for the backward softmax
template <typename T> struct V4x;
template <> struct V4x<__nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float (&v)[4]) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[4]) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
    *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
};
template <> struct V4x<float> {
  static __device__ __forceinline__ void ld(const float* p, float (&v)[4]) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  static __device__ __forceinline__ void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

// dS = P (dP - <dP, P>) * scale; writes dAC = dS and the un-shifted
// dBD[p] = dS[p - (T-1-i)] (zero where no key maps to p).  Lane owns 4
// consecutive columns per 128-column group (NG groups); dS is staged in
// shared memory for the shifted write.
template <typename T, int NG>
__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(const float* __restrict__ gp, int64_t lds,
                                                                const T* __restrict__ p, int64_t ldp,
                                                                T* __restrict__ gac, T* __restrict__ gbd,
                                                                int64_t rows, int Tn, int M, int mem_len,
                                                                float scale) {
  extern __shared__ float sh_gs[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kWarps + warp;
  if (row >= rows) return;
  // one padding float per 32: the stride-4 lane pattern of both the stores
  // and the shifted reads then hits 32 distinct banks
  float* gs_row = sh_gs + warp * (132 * NG);
  const int i = (int)(row % Tn);
  const int lo = M - mem_len, hi = M + i, off = Tn - 1 - i;
  const float* g = gp + row * lds;
  const T* pr = p + row * ldp;
  float pv[NG][4], gv[NG][4];
  float dot = 0.f;
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int j0 = 4 * lane + 128 * q;
    if (j0 < ldp) {
      V4x<T>::ld(pr + j0, pv[q]);
      V4x<float>::ld(g + j0, gv[q]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) pv[q][k] = gv[q][k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      if (j < lo || j > hi) pv[q][k] = gv[q][k] = 0.f;
      dot += pv[q][k] * gv[q][k];
    }
  }
  dot = warp_sum(dot);
  T* ga = gac + row * ldp;
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int j0 = 4 * lane + 128 * q;
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = pv[q][k] * (gv[q][k] - dot) * scale;
#pragma unroll
    for (int k = 0; k < 4; ++k) gs_row[j0 + k + ((j0 + k) >> 5)] = o[k];
    if (j0 < ldp) V4x<T>::st(ga + j0, o);
  }
  __syncwarp();
  T* gb = gbd + row * ldp;
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int p0 = 4 * lane + 128 * q;
    if (p0 >= ldp) continue;
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = p0 + k - off;
      o[k] = (j >= 0 && j < 128 * NG) ? gs_row[j + (j >> 5)] : 0.f;
    }
    V4x<T>::st(gb + p0, o);
  }
}

// Per-head column sums of two [H, R, dh] fp32 arrays, deterministic:
// stage 1 writes part[src][h][chunk][c], stage 2 sums chunks in order.
constexpr int kBiasChunks = 64;

__global__ void bias_partial_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ part,
                                    int H, int64_t R, int dh, int64_t ldg) {
  __shared__ float red[kThreads];
  const int chunk = blockIdx.x, h = blockIdx.y, which = blockIdx.z;
  const float* src = (which ? b : a) + (int64_t)h * R * ldg;
  const int groups = kThreads / dh;
  const int c = threadIdx.x % dh, gi = threadIdx.x / dh;
  const int64_t per = (R + kBiasChunks - 1) / kBiasChunks;
  const int64_t r0 = chunk * per;
  const int64_t r1 = (r0 + per < R) ? r0 + per : R;
  float acc = 0.f;
  if (gi < groups)
    for (int64_t r = r0 + gi; r < r1; r += groups) acc += src[r * ldg + c];
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

inline int blocks8(int64_t units) { return blocks_for(units); }

int xl_split_qkv(int dtype, const void* qkv, const float* u, const float* v, void* qu, void* qv, void* kh, void* vh,
                 int64_t B, int64_t Tn, int64_t M, int H, int dh, cudaStream_t st, int64_t ldq, int64_t ldh) {
  if (ldq <= 0) ldq = 3 * (int64_t)H * dh;
  if (ldh <= 0) ldh = dh;
  if (dh % 8 || ldq != 3 * (int64_t)H * dh || ldh != dh) {
    const int64_t rows = B * (M + Tn);
    if (rows == 0) return RP_OK;
    XL_DTYPE(dtype, split_qkv_rows_kernel<T><<<row_grid(rows), kRowBlk, 0, st>>>(
                        (const T*)qkv, u, v, (T*)qu, (T*)qv, (T*)kh, (T*)vh, (int)B, (int)Tn, (int)M, H, dh, ldq, ldh));
    return check_launch("xl_split_qkv");
  }
  const int64_t n = (int64_t)H * B * (M + Tn) * (dh / 8);
  if (n == 0) return RP_OK;
  XL_DTYPE(dtype, split_qkv_kernel<T><<<blocks8(n), kThreads, 0, st>>>(
                      (const T*)qkv, u, v, (T*)qu, (T*)qv, (T*)kh, (T*)vh, (int)B, (int)Tn, (int)M, H, dh));
  return check_launch("xl_split_qkv");
}

#define XL_PAIR(SD, DD, LAUNCH)                        \
  if ((SD) == RP_BF16 && (DD) == RP_BF16) {              \
    using S = __nv_bfloat16;                             \
    using D = __nv_bfloat16;                             \
    LAUNCH;                                              \
  } else if ((SD) == RP_F32 && (DD) == RP_BF16) {        \
    using S = float;                                     \
    using D = __nv_bfloat16;                             \
    LAUNCH;                                              \
  } else if ((SD) == RP_BF16 && (DD) == RP_F32) {        \
    using S = __nv_bfloat16;                             \
    using D = float;                                     \
    LAUNCH;                                              \
  } else {                                               \
    using S = float;                                     \
    using D = float;                                     \
    LAUNCH;                                              \
  }

int xl_split_heads(int src_dtype, const void* src, int64_t ld, int dst_dtype, void* dst, int64_t rows, int H, int dh,
                   cudaStream_t st, int64_t ldh) {
  if (ldh <= 0) ldh = dh;
  if (dh % 8 || ld % 8 || ldh != dh) {
    if (rows == 0) return RP_OK;
    XL_PAIR(src_dtype, dst_dtype, (split_heads_rows_kernel<S, D><<<row_grid(rows), kRowBlk, 0, st>>>(
                                      (const S*)src, ld, (D*)dst, rows, H, dh, ldh)));
    return check_launch("xl_split_heads");
  }
  const int64_t n = rows * H * (dh / 8);
  if (n == 0) return RP_OK;
  const int g = blocks8(n);
  XL_PAIR(src_dtype, dst_dtype,
          (split_heads_kernel<S, D><<<g, kThreads, 0, st>>>((const S*)src, ld, (D*)dst, rows, H, dh)));
  return check_launch("xl_split_heads");
}

int xl_merge_heads(int src_dtype, const void* src, int dst_dtype, void* dst, int64_t ld, int64_t rows, int H, int dh,
                   cudaStream_t st, int64_t ldh) {
  if (ldh <= 0) ldh = dh;
  if (dh % 8 || ld % 8 || ldh != dh) {
    if (rows == 0) return RP_OK;
    XL_PAIR(src_dtype, dst_dtype, (merge_heads_rows_kernel<S, D><<<row_grid(rows), kRowBlk, 0, st>>>(
                                      (const S*)src, (D*)dst, ld, rows, H, dh, ldh)));
    return check_launch("xl_merge_heads");
  }
  const int64_t n = rows * H * (dh / 8);
  if (n == 0) return RP_OK;
  const int g = blocks8(n);
  XL_PAIR(src_dtype, dst_dtype,
          (merge_heads_kernel<S, D><<<g, kThreads, 0, st>>>((const S*)src, (D*)dst, ld, rows, H, dh)));
  return check_launch("xl_merge_heads");
}

int xl_merge_grads(int dtype, const float* gqu, const float* gqv, const void* gkh, const void* gvh, void* gqkv,
                   int64_t B, int64_t Tn, int64_t M, int H, int dh, cudaStream_t st, int64_t ldq, int64_t ldg,
                   int64_t ldkv) {
  if (ldq <= 0) ldq = 3 * (int64_t)H * dh;
  if (ldg <= 0) ldg = dh;
  if (ldkv <= 0) ldkv = dh;
  if (dh % 8 || ldq != 3 * (int64_t)H * dh || ldg != dh || ldkv != dh) {
    const int64_t rows = B * (M + Tn);
    if (rows == 0) return RP_OK;
    XL_DTYPE(dtype, merge_grads_rows_kernel<T><<<row_grid(rows), kRowBlk, 0, st>>>(
                        gqu, gqv, (const T*)gkh, (const T*)gvh, (T*)gqkv, (int)B, (int)Tn, (int)M, H, dh, ldq, ldg,
                        ldkv));
    return check_launch("xl_merge_grads");
  }
  const int64_t n = B * (M + Tn) * 3 * (int64_t)H * dh / 8;
  if (n == 0) return RP_OK;
  XL_DTYPE(dtype, merge_grads_kernel<T><<<blocks8(n), kThreads, 0, st>>>(gqu, gqv, (const T*)gkh, (const T*)gvh,
                                                                        (T*)gqkv, (int)B, (int)Tn, (int)M, H, dh));
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
  if (mem_len < 0 || mem_len > M || ldp < M + Tn || lds < M + Tn || ldp % 8 || lds % 4)
    return set_error(RP_ERR_DIMENSION, "xl_softmax_bwd: bad memory length or leading dimension");
  const int need = (int)((ldp + 127) / 128);
  const int ng = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 12 ? 12 : need <= 16 ? 16 : -1;
  const int g = (int)((rows + kWarps - 1) / kWarps);
#define XL_BWD(NGV)                                                                                   \
  case NGV: {                                                                                         \
    constexpr int NG = NGV;                                                                           \
    const size_t smem = sizeof(float) * kWarps * 132 * NG;                                            \
    XL_DTYPE(dtype, {                                                                                 \
      if (smem > 48 * 1024)                                                                           \
        cudaFuncSetAttribute(softmax_bwd_kernel<T, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)smem);                                                              \
      softmax_bwd_kernel<T, NG><<<g, kThreads, smem, st>>>(gp, lds, (const T*)p, ldp, (T*)gac, (T*)gbd, \
                                                           rows, (int)Tn, (int)M, (int)mem_len, scale); \
    });                                                                                               \
    break;                                                                                            \
  }
  switch (ng) {
    XL_BWD(1)
    XL_BWD(2)
    XL_BWD(4)
    XL_BWD(8)
    XL_BWD(12)
    XL_BWD(16)
    default:
      return set_error(RP_ERR_DIMENSION, "xl_softmax_bwd: key length not supported");
  }
#undef XL_BWD
  return check_launch("xl_softmax_bwd");
}

int64_t xl_bias_grad_workspace_bytes(int H, int dh) { return (int64_t)2 * H * kBiasChunks * dh * sizeof(float); }

int xl_bias_grad(const float* gqu, const float* gqv, float* part, float* gu, float* gv, int H, int64_t R, int dh,
                 cudaStream_t st, int64_t ldg) {
  if (ldg <= 0) ldg = dh;
  if (dh > kThreads) return set_error(RP_ERR_DIMENSION, "xl_bias_grad: head dim must be <= 256");
  bias_partial_kernel<<<dim3(kBiasChunks, H, 2), kThreads, 0, st>>>(gqu, gqv, part, H, R, dh, ldg);
  bias_finish_kernel<<<(2 * H * dh + kThreads - 1) / kThreads, kThreads, 0, st>>>(part, gu, gv, H, dh);
  return check_launch("xl_bias_grad");
}

}  // namespace rp
