// Row-wise HBM-bound kernels of the block: LayerNorm forward/backward
// (reference layers.py:62-79), causal softmax forward/backward
// (layers.py:180-183, 237), dropout-masked gradients (layers.py:209-216) and
// deterministic column reductions for the bias / gain / LN-bias gradients
// (layers.py:72-73, 220, 223).
//
// One warp owns one row; a row of d <= 32*NPL elements lives in registers, so
// every kernel reads its inputs once and writes its outputs once.  Column
// reductions never use float atomics: each CTA writes a partial row and a
// second pass sums partials in fixed order, so results are bitwise
// reproducible for a given shape.
#include <cstdlib>
#include <initializer_list>
#include <utility>
#include <algorithm>

#include "common.cuh"
#include "rp_internal.h"

namespace rp {

constexpr int kRowThreads = 256;  // 8 warps
constexpr int kRowWarps = kRowThreads / 32;
constexpr float kLnEps = 1e-5f;  // layers.py:25

__device__ __forceinline__ void flag_set(int32_t* flag, int bit) {
  if (flag) atomicOr(flag, bit);
}

// 4-wide vector load/store of T as fp32.
template <typename T> struct V4;
template <> struct V4<float> {
  static __device__ __forceinline__ void ld(const float* p, float (&v)[4]) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  static __device__ __forceinline__ void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct V4<__nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float (&v)[4]) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[4]) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  }
};

// VW-wide vector load/store of T as fp32 (VW = 4: 16 B of fp32 / 8 B of
// bf16; VW = 2: 8 B / 4 B -- even widths whose fp32 rows are only 8-byte
// aligned, e.g. BASELINE configs[3]'s d 410).
template <typename T, int VW> struct VecIO;
template <typename T> struct VecIO<T, 4> {
  static __device__ __forceinline__ void ld(const T* p, float (&v)[4]) { V4<T>::ld(p, v); }
  static __device__ __forceinline__ void st(T* p, const float (&v)[4]) { V4<T>::st(p, v); }
};
template <> struct VecIO<float, 2> {
  static __device__ __forceinline__ void ld(const float* p, float (&v)[2]) {
    const float2 f = *reinterpret_cast<const float2*>(p);
    v[0] = f.x; v[1] = f.y;
  }
  static __device__ __forceinline__ void st(float* p, const float (&v)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};
template <> struct VecIO<__nv_bfloat16, 2> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float (&v)[2]) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
    v[0] = a.x; v[1] = a.y;
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[2]) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v[0], v[1]);
  }
};

// ---------------------------------------------------------------------------
// Vectorised variants: lane owns VW consecutive columns per (32*VW)-column
// group, NG groups per row (a ragged last group is masked).  Rows of the
// compute-dtype tensors sit at their pitches (ldx / ldy / ldm: padded bf16
// rows), fp32 rows at d.

template <typename T, int NG, int VW = 4>
__global__ void __launch_bounds__(kRowThreads) ln_fwd_v4_kernel(const T* __restrict__ x, const float* __restrict__ g,
                                                                 const float* __restrict__ b, T* __restrict__ y,
                                                                 float* __restrict__ mean, float* __restrict__ rstd,
                                                                 int64_t rows, int d, int32_t* flag, int64_t ldx,
                                                                 int64_t ldy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  float v[NG][VW];
  float s = 0.f;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    if ((i * 32 + lane) * VW < d) {
      VecIO<T, VW>::ld(x + row * ldx + (i * 32 + lane) * VW, v[i]);
    } else {
#pragma unroll
      for (int q = 0; q < VW; ++q) v[i][q] = 0.f;
    }
#pragma unroll
    for (int q = 0; q < VW; ++q) {
      finite &= isfinite(v[i][q]);
      s += v[i][q];
    }
  }
  const float mu = warp_sum(s) / d;
  float qv = 0.f;
#pragma unroll
  for (int i = 0; i < NG; ++i)
    if ((i * 32 + lane) * VW < d) {
#pragma unroll
      for (int q = 0; q < VW; ++q) qv += (v[i][q] - mu) * (v[i][q] - mu);
    }
  const float rs = rsqrtf(warp_sum(qv) / d + kLnEps);
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const int j = (i * 32 + lane) * VW;
    if (j >= d) continue;
    float gg[VW], bb[VW], o[VW];
    VecIO<float, VW>::ld(g + j, gg);
    VecIO<float, VW>::ld(b + j, bb);
#pragma unroll
    for (int q = 0; q < VW; ++q) o[q] = (v[i][q] - mu) * rs * gg[q] + bb[q];
    VecIO<T, VW>::st(y + row * ldy + j, o);
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
  if (!__all_sync(0xffffffffu, finite) && lane == 0) flag_set(flag, RP_FLAG_NONFINITE);
}

template <typename T, int NG, int VW = 4>
__global__ void __launch_bounds__(kRowThreads) ln_bwd_v4_kernel(
    const float* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ g, const float* __restrict__ resid_grad,
    float* __restrict__ dx, T* __restrict__ dx_masked, uint64_t seed, uint64_t thr, float scale, int drop_on,
    float* __restrict__ part_g, float* __restrict__ part_b, int64_t rows, int d, int64_t ldx, int64_t ldm) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int GW = 32 * VW;  // columns per group
  // wide rows (NG > 4 groups of 128, d >= 1024): the gain and the residual
  // gradient are read where they are used instead of living in registers
  constexpr bool kLean = NG * VW > 16;
  __shared__ float red[kRowWarps][2][GW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc_g[NG][VW], acc_b[NG][VW], gv[kLean ? 1 : NG][VW];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    if constexpr (!kLean) {
      if ((i * 32 + lane) * VW < d) {
        VecIO<float, VW>::ld(g + (i * 32 + lane) * VW, gv[i]);
      } else {
#pragma unroll
        for (int q = 0; q < VW; ++q) gv[i][q] = 0.f;
      }
    }
#pragma unroll
    for (int q = 0; q < VW; ++q) acc_g[i][q] = acc_b[i][q] = 0.f;
  }
  auto gain = [&](int i, float (&o)[VW]) {
    if constexpr (kLean) {
      if ((i * 32 + lane) * VW < d) {
        VecIO<float, VW>::ld(g + (i * 32 + lane) * VW, o);
      } else {
#pragma unroll
        for (int q = 0; q < VW; ++q) o[q] = 0.f;
      }
    } else {
#pragma unroll
      for (int q = 0; q < VW; ++q) o[q] = gv[kLean ? 0 : i][q];
    }
  };
  const int64_t stride = (int64_t)gridDim.x * kRowWarps;
  for (int64_t row = (int64_t)blockIdx.x * kRowWarps + w; row < rows; row += stride) {
    const float mu = mean[row], rs = rstd[row];
    float xh[NG][VW], dyv[NG][VW], rv[kLean ? 1 : NG][VW];
    float s1 = 0.f, s2 = 0.f;
    // every load of the row is issued up front (the residual gradient too):
    // one DRAM round trip per row instead of two
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int j = (i * 32 + lane) * VW;
      if (j >= d) {  // ragged width: columns past d contribute nothing
#pragma unroll
        for (int q = 0; q < VW; ++q) {
          xh[i][q] = dyv[i][q] = 0.f;
          if constexpr (!kLean) rv[i][q] = 0.f;
        }
        continue;
      }
      VecIO<T, VW>::ld(x + row * ldx + j, xh[i]);
      VecIO<float, VW>::ld(dy + row * d + j, dyv[i]);
      if constexpr (!kLean) {
        if (resid_grad) {
          VecIO<float, VW>::ld(resid_grad + row * d + j, rv[i]);
        } else {
#pragma unroll
          for (int q = 0; q < VW; ++q) rv[i][q] = 0.f;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float gq[VW];
      gain(i, gq);
#pragma unroll
      for (int q = 0; q < VW; ++q) {
        xh[i][q] = (xh[i][q] - mu) * rs;
        const float t = dyv[i][q] * gq[q];
        s1 += t;
        s2 += t * xh[i][q];
        acc_g[i][q] += dyv[i][q] * xh[i][q];
        acc_b[i][q] += dyv[i][q];
      }
    }
    s1 = warp_sum(s1) / d;
    s2 = warp_sum(s2) / d;
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int j = (i * 32 + lane) * VW;
      if (j >= d) continue;
      float gq[VW], r4[VW];
      gain(i, gq);
      if constexpr (kLean) {
        if (resid_grad) {
          VecIO<float, VW>::ld(resid_grad + row * d + j, r4);
        } else {
#pragma unroll
          for (int q = 0; q < VW; ++q) r4[q] = 0.f;
        }
      } else {
#pragma unroll
        for (int q = 0; q < VW; ++q) r4[q] = rv[kLean ? 0 : i][q];
      }
      float o[VW];
#pragma unroll
      for (int q = 0; q < VW; ++q) o[q] = rs * (dyv[i][q] * gq[q] - s1 - xh[i][q] * s2) + r4[q];
      if (dx) VecIO<float, VW>::st(dx + row * d + j, o);  // NULL: only the gain / bias sums (XL memory rows)
      if (dx_masked) {
        if (drop_on) {
#pragma unroll
          for (int q = 0; q < VW; ++q)
            o[q] = dropout_keep_z(dropout_z(seed, (uint64_t)row * d + j) + (uint64_t)q * kGolden, thr) ? o[q] * scale : 0.f;
        }
        VecIO<T, VW>::st(dx_masked + row * ldm + j, o);
      }
    }
  }
  // per-CTA column partials, one group at a time (warp order fixed)
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    if (i) __syncthreads();
#pragma unroll
    for (int q = 0; q < VW; ++q) {
      red[w][0][lane * VW + q] = acc_g[i][q];
      red[w][1][lane * VW + q] = acc_b[i][q];
    }
    __syncthreads();
    if (threadIdx.x < 2 * GW) {
      const int which = threadIdx.x / GW, c = threadIdx.x % GW;
      float sacc = 0.f;
#pragma unroll
      for (int q = 0; q < kRowWarps; ++q) sacc += red[q][which][c];
      if (i * GW + c < d) (which ? part_b : part_g)[(int64_t)blockIdx.x * d + i * GW + c] = sacc;
    }
  }
}

// Split rows: P warps own one row, each NG groups (gain and residual
// gradient in registers).  The one-warp-per-row kernel at d 1024 needs ~175
// registers, so one CTA (8 warps) fits an SM and too few row loads are in
// flight; NG 4 keeps 128 registers (two CTAs per SM), NG 2 ~80 (three).  The
// row sums s1, s2 combine the P parts through shared memory (part order, the
// same in every warp of the row); column partials are summed over the CTA's
// same-part warps in warp order.
template <typename T, int NG, int P, int VW = 4>
__global__ void __launch_bounds__(kRowThreads, NG == 1 ? 4 : NG == 2 ? 3 : 2) ln_bwd_split_kernel(
    const float* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ g, const float* __restrict__ resid_grad,
    float* __restrict__ dx, T* __restrict__ dx_masked, uint64_t seed, uint64_t thr, float scale, int drop_on,
    float* __restrict__ part_g, float* __restrict__ part_b, int64_t rows, int d, int64_t ldx, int64_t ldm) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int GW = 32 * VW;
  constexpr int kRows = kRowWarps / P;  // rows per CTA iteration
  __shared__ float red[kRowWarps][2][GW];
  __shared__ float xs[2][kRowWarps][2];  // [iteration parity][warp][s1, s2]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int part = w % P, pair = w / P;
  const int c0 = part * NG * GW;
  float acc_g[NG][VW], acc_b[NG][VW], gv[NG][VW];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const int j = c0 + (i * 32 + lane) * VW;
    if (j < d) {
      VecIO<float, VW>::ld(g + j, gv[i]);
    } else {
#pragma unroll
      for (int q = 0; q < VW; ++q) gv[i][q] = 0.f;
    }
#pragma unroll
    for (int q = 0; q < VW; ++q) acc_g[i][q] = acc_b[i][q] = 0.f;
  }
  const int64_t stride = (int64_t)gridDim.x * kRows;
  int it = 0;
  for (int64_t row = (int64_t)blockIdx.x * kRows + pair; row < rows; row += stride, ++it) {
    const float mu = mean[row], rs = rstd[row];
    float xh[NG][VW], dyv[NG][VW], rv[NG][VW];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int j = c0 + (i * 32 + lane) * VW;
      if (j >= d) {
#pragma unroll
        for (int q = 0; q < VW; ++q) xh[i][q] = dyv[i][q] = rv[i][q] = 0.f;
        continue;
      }
      VecIO<T, VW>::ld(x + row * ldx + j, xh[i]);
      VecIO<float, VW>::ld(dy + row * d + j, dyv[i]);
      if (resid_grad) {
        VecIO<float, VW>::ld(resid_grad + row * d + j, rv[i]);
      } else {
#pragma unroll
        for (int q = 0; q < VW; ++q) rv[i][q] = 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < NG; ++i) {
#pragma unroll
      for (int q = 0; q < VW; ++q) {
        xh[i][q] = (xh[i][q] - mu) * rs;
        const float t = dyv[i][q] * gv[i][q];
        s1 += t;
        s2 += t * xh[i][q];
        acc_g[i][q] += dyv[i][q] * xh[i][q];
        acc_b[i][q] += dyv[i][q];
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      xs[it & 1][w][0] = s1;
      xs[it & 1][w][1] = s2;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(32 * P) : "memory");
    s1 = 0.f;
    s2 = 0.f;
#pragma unroll
    for (int k = 0; k < P; ++k) {  // part order, identical in every warp of the row
      s1 += xs[it & 1][P * pair + k][0];
      s2 += xs[it & 1][P * pair + k][1];
    }
    s1 /= d;
    s2 /= d;
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int j = c0 + (i * 32 + lane) * VW;
      if (j >= d) continue;
      float o[VW];
#pragma unroll
      for (int q = 0; q < VW; ++q) o[q] = rs * (dyv[i][q] * gv[i][q] - s1 - xh[i][q] * s2) + rv[i][q];
      if (dx) VecIO<float, VW>::st(dx + row * d + j, o);  // NULL: only the gain / bias sums (XL memory rows)
      if (dx_masked) {
        if (drop_on) {
#pragma unroll
          for (int q = 0; q < VW; ++q)
            o[q] = dropout_keep_z(dropout_z(seed, (uint64_t)row * d + j) + (uint64_t)q * kGolden, thr) ? o[q] * scale : 0.f;
        }
        VecIO<T, VW>::st(dx_masked + row * ldm + j, o);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < VW; ++q) {
      red[w][0][lane * VW + q] = acc_g[i][q];
      red[w][1][lane * VW + q] = acc_b[i][q];
    }
    __syncthreads();
    if (threadIdx.x < 2 * GW) {
      const int which = threadIdx.x / GW, c = threadIdx.x % GW;
#pragma unroll
      for (int pp = 0; pp < P; ++pp) {
        float sacc = 0.f;
#pragma unroll
        for (int q = 0; q < kRows; ++q) sacc += red[P * q + pp][which][c];
        const int col = (pp * NG + i) * GW + c;
        if (col < d) (which ? part_b : part_g)[(int64_t)blockIdx.x * d + col] = sacc;
      }
    }
  }
}

// out = g * mask (T) with per-CTA column partials of the masked fp32 values.
template <typename T, int NG, int VW = 4>
__global__ void __launch_bounds__(kRowThreads) mask_grad_v4_kernel(const float* __restrict__ g, T* __restrict__ out,
                                                                    int64_t rows, int d, uint64_t seed, uint64_t pos0,
                                                                    uint64_t thr, float scale, int drop_on,
                                                                    float* __restrict__ part, int64_t ldo) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ float red[kRowWarps][32 * VW * NG];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc[NG][VW];
#pragma unroll
  for (int i = 0; i < NG; ++i)
#pragma unroll
    for (int q = 0; q < VW; ++q) acc[i][q] = 0.f;
  const int64_t stride = (int64_t)gridDim.x * kRowWarps;
  for (int64_t row = (int64_t)blockIdx.x * kRowWarps + w; row < rows; row += stride) {
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const int j = (i * 32 + lane) * VW;
      if (j >= d) continue;
      float v[VW];
      VecIO<float, VW>::ld(g + row * d + j, v);
      if (drop_on) {
#pragma unroll
        for (int q = 0; q < VW; ++q)
          v[q] = dropout_keep_z(dropout_z(seed, pos0 + (uint64_t)row * d + j) + (uint64_t)q * kGolden, thr) ? v[q] * scale : 0.f;
      }
      VecIO<T, VW>::st(out + row * ldo + j, v);
#pragma unroll
      for (int q = 0; q < VW; ++q) acc[i][q] += v[q];
    }
  }
  if (!part) return;
#pragma unroll
  for (int i = 0; i < NG; ++i)
#pragma unroll
    for (int q = 0; q < VW; ++q) red[w][(i * 32 + lane) * VW + q] = acc[i][q];
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += kRowThreads) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < kRowWarps; ++q) s += red[q][j];
    part[(int64_t)blockIdx.x * d + j] = s;
  }
}

// ---------------------------------------------------------------------------
// LayerNorm forward: y = (x - mu) * rstd * g + b; saves (mu, rstd).
template <typename T, int NPL>
__global__ void __launch_bounds__(kRowThreads) ln_fwd_kernel(const T* __restrict__ x, const float* __restrict__ g,
                                                              const float* __restrict__ b, T* __restrict__ y,
                                                              float* __restrict__ mean, float* __restrict__ rstd,
                                                              int64_t rows, int d, int32_t* flag, int64_t ldx,
                                                              int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * ldx;
  float v[NPL];
  float s = 0.f;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    v[i] = (j < d) ? to_f(xr[j]) : 0.f;
    finite &= isfinite(v[i]);
    s += v[i];
  }
  s = warp_sum(s);
  const float mu = s / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    const float c = (j < d) ? v[i] - mu : 0.f;
    q += c * c;
  }
  q = warp_sum(q);
  const float rs = rsqrtf(q / d + kLnEps);
  T* yr = y + row * ldy;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < d) yr[j] = from_f<T>((v[i] - mu) * rs * g[j] + b[j]);
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
  if (!__all_sync(0xffffffffu, finite) && lane == 0) flag_set(flag, RP_FLAG_NONFINITE);
}

// LayerNorm backward (layers.py:70-79) fused with the residual add and the
// dropout mask of the branch feeding this LN:
//   dx = rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat)) + resid_grad
//   dx_masked = dx * mask(seed, row*d + j)            (optional, dtype T)
// Per-CTA column partials of dy*xhat (gain) and dy (bias).
template <typename T, int NPL>
__global__ void __launch_bounds__(kRowThreads) ln_bwd_kernel(
    const float* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ g, const float* __restrict__ resid_grad,
    float* __restrict__ dx, T* __restrict__ dx_masked, uint64_t seed, uint64_t thr, float scale, int drop_on,
    float* __restrict__ part_g, float* __restrict__ part_b, int64_t rows, int d, int64_t ldx, int64_t ldm) {
  __shared__ float red[kRowWarps][2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc_g[NPL], acc_b[NPL], gv[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    acc_g[i] = acc_b[i] = 0.f;
    const int j = lane + 32 * i;
    gv[i] = (j < d) ? g[j] : 0.f;
  }
  const int64_t stride = (int64_t)gridDim.x * kRowWarps;
  for (int64_t row = (int64_t)blockIdx.x * kRowWarps + w; row < rows; row += stride) {
    const float mu = mean[row], rs = rstd[row];
    float xh[NPL], dyv[NPL];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int j = lane + 32 * i;
      if (j < d) {
        xh[i] = (to_f(x[row * ldx + j]) - mu) * rs;
        dyv[i] = dy[row * d + j];
      } else {
        xh[i] = dyv[i] = 0.f;
      }
      const float dxh = dyv[i] * gv[i];
      s1 += dxh;
      s2 += dxh * xh[i];
      acc_g[i] += dyv[i] * xh[i];
      acc_b[i] += dyv[i];
    }
    s1 = warp_sum(s1) / d;
    s2 = warp_sum(s2) / d;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int j = lane + 32 * i;
      if (j < d) {
        float o = rs * (dyv[i] * gv[i] - s1 - xh[i] * s2);
        if (resid_grad) o += resid_grad[row * d + j];
        if (dx) dx[row * d + j] = o;
        if (dx_masked) {
          float mo = o;
          if (drop_on) mo = dropout_keep(seed, (uint64_t)row * d + j, thr) ? o * scale : 0.f;
          dx_masked[row * ldm + j] = from_f<T>(mo);
        }
      }
    }
  }
  // per-CTA column partials, 32 columns at a time (static shared memory stays
  // at 2 KB for any d; the warp summation order is fixed)
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    if (32 * i >= d) break;
    if (i) __syncthreads();
    red[w][0][lane] = acc_g[i];
    red[w][1][lane] = acc_b[i];
    __syncthreads();
    if (threadIdx.x < 64) {
      const int which = threadIdx.x >> 5, c = threadIdx.x & 31, j = 32 * i + c;
      float sacc = 0.f;
#pragma unroll
      for (int q = 0; q < kRowWarps; ++q) sacc += red[q][which][c];
      if (j < d) (which ? part_b : part_g)[(int64_t)blockIdx.x * d + j] = sacc;
    }
  }
}

// out[j] = sum_b partial[b, j]: 32 columns x 32 partial lanes per CTA, each
// lane sums a fixed strided subset, then lane sums combine in fixed order.
// s += part[b * cols + j] for b = b0, b0 + 32, ... < nblk, in that order,
// four loads in flight (the additions keep their order: bitwise the plain loop)
__device__ __forceinline__ float colsum_strided(const float* __restrict__ part, int b0, int nblk, int64_t cols,
                                                int64_t j) {
  float s = 0.f;
  int b = b0;
  for (; b + 96 < nblk; b += 128) {
    const float v0 = part[(int64_t)b * cols + j], v1 = part[(int64_t)(b + 32) * cols + j];
    const float v2 = part[(int64_t)(b + 64) * cols + j], v3 = part[(int64_t)(b + 96) * cols + j];
    s += v0;
    s += v1;
    s += v2;
    s += v3;
  }
  for (; b < nblk; b += 32) s += part[(int64_t)b * cols + j];
  return s;
}

__global__ void __launch_bounds__(1024) colsum_finish_kernel(const float* __restrict__ part, int nblk, int64_t cols,
                                                             float* __restrict__ out) {
  __shared__ float red[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + tx;
  const float s = j < cols ? colsum_strided(part, ty, nblk, cols, j) : 0.f;
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < cols) {
    float t = 0.f;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) t += red[q][tx];
    out[j] = t;
  }
}

// Several colsum finishes in one launch (same per-column order as
// colsum_finish_kernel, so results are bitwise identical): CTA x covers 32
// columns of the job whose column-block range contains x.
__global__ void __launch_bounds__(1024) colsum_finish_multi_kernel(ColsumJobs jobs) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ float red[32][33];
  int jb = 0;
  while (jb + 1 < jobs.n && (int)blockIdx.x >= jobs.first_block[jb + 1]) ++jb;
  const ColsumJob& J = jobs.job[jb];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = (int64_t)(blockIdx.x - jobs.first_block[jb]) * 32 + tx;
  const float s = j < J.cols ? colsum_strided(J.part, ty, J.nblk, J.cols, j) : 0.f;
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < J.cols) {
    float t = 0.f;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) t += red[q][tx];
    J.out[j] = t;
  }
}

// Column partial sums of a [rows, cols] matrix (row-major, ld).
template <typename T>
__global__ void colsum_partial_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                      float* __restrict__ part) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t j = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += to_f(x[r * ld + j]);
  part[(int64_t)blockIdx.x * cols + j] = s;
}

// Two adjacent columns per thread (a warp reads 128 contiguous bytes of a
// bf16 row), rows in groups of 4 loads in flight; the same row order per
// column as colsum_partial_kernel (bitwise equal sums).
template <typename T>
__global__ void colsum_partial2_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                       float* __restrict__ part) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t j = 2 * ((int64_t)blockIdx.y * blockDim.x + threadIdx.x);
  if (j >= cols) return;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float s0 = 0.f, s1 = 0.f;
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4) {
    float a[4], b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float v[2];
      VecIO<T, 2>::ld(x + (r + k) * ld + j, v);
      a[k] = v[0];
      b[k] = v[1];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s0 += a[k];
      s1 += b[k];
    }
  }
  for (; r < r1; ++r) {
    float v[2];
    VecIO<T, 2>::ld(x + r * ld + j, v);
    s0 += v[0];
    s1 += v[1];
  }
  part[(int64_t)blockIdx.x * cols + j] = s0;
  part[(int64_t)blockIdx.x * cols + j + 1] = s1;
}

// out = g * mask (T) with column partials of the masked fp32 values
// (the b2 gradient, layers.py:215-220).
template <typename T>
__global__ void mask_grad_kernel(const float* __restrict__ g, T* __restrict__ out, int64_t rows, int d,
                                 uint64_t seed, uint64_t pos0, uint64_t thr, float scale, int drop_on,
                                 float* __restrict__ part, int64_t ldo) {
  const int64_t j = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    float v = g[r * d + j];
    if (drop_on) v = dropout_keep(seed, pos0 + (uint64_t)r * d + j, thr) ? v * scale : 0.f;
    out[r * ldo + j] = from_f<T>(v);
    s += v;
  }
  if (part) part[(int64_t)blockIdx.x * d + j] = s;
}

// ---------------------------------------------------------------------------
// causal softmax over rows of length T (scores already scaled by 1/sqrt(d)).
template <typename T, int NPL>
__global__ void __launch_bounds__(kRowThreads) softmax_causal_kernel(const float* __restrict__ s, T* __restrict__ p,
                                                                      int64_t rows, int Tn, int64_t ld) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int i = (int)(row % Tn);  // query position
  const float* sr = s + row * ld;
  float v[NPL];
  float mx = -INFINITY;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    v[q] = (j <= i) ? sr[j] : -INFINITY;
    mx = fmaxf(mx, v[q]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    v[q] = (j <= i) ? __expf(v[q] - mx) : 0.f;
    sum += v[q];
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  T* pr = p + row * ld;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    if (j < Tn) pr[j] = from_f<T>(v[q] * inv);
  }
}

// g_s = (g_p - sum_j g_p*P) * P * scale   (layers.py:237, 1/sqrt(d) folded in)
template <typename T, int NPL>
__global__ void __launch_bounds__(kRowThreads) softmax_bwd_kernel(const float* __restrict__ gp, const T* __restrict__ p,
                                                                   T* __restrict__ gs, float scale, int64_t rows,
                                                                   int Tn, int64_t ld) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  float gv[NPL], pv[NPL];
  float dot = 0.f;
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    gv[q] = (j < Tn) ? gp[row * ld + j] : 0.f;
    pv[q] = (j < Tn) ? to_f(p[row * ld + j]) : 0.f;
    dot += gv[q] * pv[q];
  }
  dot = warp_sum(dot);
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int j = lane + 32 * q;
    if (j < Tn) gs[row * ld + j] = from_f<T>((gv[q] - dot) * pv[q] * scale);
  }
}

// ---------------------------------------------------------------------------
// host launchers
namespace {

inline int npl_for(int64_t n) {
  if (n <= 64) return 2;
  if (n <= 128) return 4;
  if (n <= 256) return 8;
  if (n <= 512) return 16;
  if (n <= 1024) return 32;
  if (n <= 2048) return 64;
  return -1;
}

// Programmatic dependent launch for the row kernels: a launch may begin
// while the previous kernel on the stream drains; every kernel below waits
// (griddepcontrol.wait) before touching global memory.  RP_ROW_PDL=0 turns
// it off (A/B).
inline bool row_pdl() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RP_ROW_PDL");
    const char* g = getenv("RP_NO_PDL");
    on = ((e && e[0] == '0') || (g && g[0] == '1')) ? 0 : 1;
  }
  return on == 1;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = row_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int row_blocks(int64_t rows) { return (int)((rows + kRowWarps - 1) / kRowWarps); }

}  // namespace

int ln_bwd_blocks(int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>(row_blocks(rows), 592)); }

#define RP_NPL_DISPATCH(NPL_VAL, ...)                                   \
  switch (NPL_VAL) {                                                    \
    case 2: { constexpr int NPL = 2; __VA_ARGS__; break; }              \
    case 4: { constexpr int NPL = 4; __VA_ARGS__; break; }              \
    case 8: { constexpr int NPL = 8; __VA_ARGS__; break; }              \
    case 16: { constexpr int NPL = 16; __VA_ARGS__; break; }            \
    case 32: { constexpr int NPL = 32; __VA_ARGS__; break; }            \
    case 64: { constexpr int NPL = 64; __VA_ARGS__; break; }            \
    default: return set_error(RP_ERR_DIMENSION, "row length too large"); \
  }

#define RP_DTYPE_DISPATCH(DT, ...)                     \
  if ((DT) == RP_BF16) {                               \
    using T = __nv_bfloat16;                           \
    __VA_ARGS__;                                       \
  } else {                                             \
    using T = float;                                   \
    __VA_ARGS__;                                       \
  }

#define RP_NG_DISPATCH(NGV, ...)                     \
  switch (NGV) {                                    \
    case 1: { constexpr int NG = 1; __VA_ARGS__; break; } \
    case 2: { constexpr int NG = 2; __VA_ARGS__; break; } \
    case 4: { constexpr int NG = 4; __VA_ARGS__; break; } \
    case 8: { constexpr int NG = 8; __VA_ARGS__; break; } \
    default: break;                                 \
  }

// Vector width and (32*VW)-column groups per row for the vector kernels:
// VW 4 for d % 4 == 0 up to 1024, VW 2 for even d up to 512 (fp32 rows of an
// even width are 8-byte aligned: d 410); every compute-dtype pitch must be a
// multiple of VW.  A ragged last group is masked.  ng 0 = the scalar kernels.
struct VecShape {
  int vw = 0, ng = 0;
};
inline VecShape vec_for(int64_t d, std::initializer_list<int64_t> pitches = {}) {
  VecShape v;
  if (d <= 0) return v;
  for (int vw : {4, 2}) {
    if (d % vw || d > 32 * vw * 8) continue;
    bool ok = true;
    for (int64_t ld : pitches) ok &= ld % vw == 0;
    if (!ok) continue;
    const int64_t ng = (d + 32 * vw - 1) / (32 * vw);
    v.vw = vw;
    v.ng = ng <= 1 ? 1 : ng <= 2 ? 2 : ng <= 4 ? 4 : 8;
    return v;
  }
  return v;
}
inline int ng_for(int64_t d) { return vec_for(d).vw == 4 ? vec_for(d).ng : 0; }

#define RP_VW_DISPATCH(VWV, ...)                              \
  if ((VWV) == 4) {                                           \
    constexpr int VW = 4;                                     \
    __VA_ARGS__;                                              \
  } else {                                                    \
    constexpr int VW = 2;                                     \
    __VA_ARGS__;                                              \
  }

int layernorm_fwd(int dtype, const void* x, const float* g, const float* b, void* y, float* mean, float* rstd,
                  int64_t rows, int64_t d, int32_t* flag, cudaStream_t st, int64_t ldx, int64_t ldy) {
  if (rows == 0) return RP_OK;
  if (ldx <= 0) ldx = d;
  if (ldy <= 0) ldy = d;
  const VecShape vs = vec_for(d, {ldx, ldy});
  if (vs.ng) {
    RP_DTYPE_DISPATCH(dtype, RP_VW_DISPATCH(vs.vw, RP_NG_DISPATCH(vs.ng, launch_pdl(
                                 ln_fwd_v4_kernel<T, NG, VW>, row_blocks(rows), kRowThreads, 0, st, (const T*)x, g, b,
                                 (T*)y, mean, rstd, rows, (int)d, flag, ldx, ldy))));
    return check_launch("layernorm_fwd");
  }
  const int npl = npl_for(d);
  RP_DTYPE_DISPATCH(dtype, RP_NPL_DISPATCH(npl, ln_fwd_kernel<T, NPL><<<row_blocks(rows), kRowThreads, 0, st>>>(
                                                    (const T*)x, g, b, (T*)y, mean, rstd,
                                                    rows, (int)d, flag, ldx, ldy)));
  return check_launch("layernorm_fwd");
}

int layernorm_bwd(int dtype, const float* dy, const void* x, const float* mean, const float* rstd, const float* g,
                  const float* resid_grad, float* dx, void* dx_masked, uint64_t seed, uint64_t thr, float scale,
                  int drop_on, float* part_g, float* part_b, int64_t rows, int64_t d, cudaStream_t st, int64_t ldx,
                  int64_t ldm) {
  if (rows == 0) return RP_OK;
  if (ldx <= 0) ldx = d;
  if (ldm <= 0) ldm = d;
  const int nb = ln_bwd_blocks(rows);
  // warps per row once a lane holds >= 16 elements of the row (RP_LN_SPLIT:
  // 1 = one warp per row).  Measured (tools/ln_bwd_bench.py): d 1024 two
  // warps 106 -> 64 us (four: 70); d 512 four warps 57 -> 47 us at 22528
  // rows, 29 -> 23 us at 8192; d 400 27 -> 23 us
  static const int split_env = getenv("RP_LN_SPLIT") ? atoi(getenv("RP_LN_SPLIT")) : -1;
  const VecShape vs = vec_for(d, {ldx, ldm});
  const int per_lane = vs.ng * vs.vw;  // row elements per lane with one warp per row
  int split = split_env >= 0 ? split_env : (per_lane == 32 ? 2 : per_lane == 16 ? 4 : 1);
  if (per_lane < 16) split = 1;
#define RP_LN_SPLIT_LAUNCH(NGV, PV)                                                                              \
  RP_DTYPE_DISPATCH(dtype, RP_VW_DISPATCH(vs.vw, launch_pdl(ln_bwd_split_kernel<T, NGV, PV, VW>, nb, kRowThreads, 0, \
                                                            st, dy, (const T*)x, mean, rstd, g, resid_grad, dx,     \
                                                            (T*)dx_masked, seed, thr, scale, drop_on, part_g,      \
                                                            part_b, rows, (int)d, ldx, ldm)));                      \
  return check_launch("layernorm_bwd")
  if (vs.ng == 8 && split == 2) { RP_LN_SPLIT_LAUNCH(4, 2); }
  if (vs.ng == 8 && split == 4) { RP_LN_SPLIT_LAUNCH(2, 4); }
  if (vs.ng == 4 && split == 2) { RP_LN_SPLIT_LAUNCH(2, 2); }
  if (vs.ng == 4 && split == 4) { RP_LN_SPLIT_LAUNCH(1, 4); }
#undef RP_LN_SPLIT_LAUNCH
  if (vs.ng) {
    RP_DTYPE_DISPATCH(dtype, RP_VW_DISPATCH(vs.vw, RP_NG_DISPATCH(vs.ng, launch_pdl(
                                 ln_bwd_v4_kernel<T, NG, VW>, nb, kRowThreads, 0, st, dy, (const T*)x, mean, rstd, g,
                                 resid_grad, dx, (T*)dx_masked, seed, thr, scale, drop_on, part_g, part_b, rows,
                                 (int)d, ldx, ldm))));
    return check_launch("layernorm_bwd");
  }
  const int npl = npl_for(d);
  RP_DTYPE_DISPATCH(dtype, RP_NPL_DISPATCH(npl, ln_bwd_kernel<T, NPL><<<nb, kRowThreads, 0, st>>>(
                                                    dy, (const T*)x, mean, rstd, g, resid_grad, dx,
                                                    (T*)dx_masked, seed, thr, scale, drop_on, part_g, part_b,
                                                    rows, (int)d, ldx, ldm)));
  return check_launch("layernorm_bwd");
}

int colsum_finish(const float* part, int nblk, int64_t cols, float* out, cudaStream_t st) {
  if (cols == 0) return RP_OK;
  colsum_finish_kernel<<<(int)((cols + 31) / 32), 1024, 0, st>>>(part, nblk, cols, out);
  return check_launch("colsum_finish");
}

int colsum_finish_multi(const ColsumJob* jobs, int n, cudaStream_t st) {
  if (n < 1 || n > kMaxColsumJobs) return set_error(RP_ERR_INVALID, "colsum_finish_multi: 1..%d jobs", kMaxColsumJobs);
  ColsumJobs J{};
  J.n = n;
  int blocks = 0;
  for (int i = 0; i < n; ++i) {
    J.job[i] = jobs[i];
    J.first_block[i] = blocks;
    blocks += (int)((jobs[i].cols + 31) / 32);
  }
  if (blocks == 0) return RP_OK;
  launch_pdl(colsum_finish_multi_kernel, blocks, 1024, 0, st, J);
  return check_launch("colsum_finish_multi");
}

int mask_grad_blocks_ld(int64_t rows, int64_t d, int64_t ldo) {
  if (ldo <= 0) ldo = d;
  return vec_for(d, {ldo}).ng ? ln_bwd_blocks(rows) : colsum_blocks(rows);
}
int mask_grad_blocks(int64_t rows, int64_t d) { return mask_grad_blocks_ld(rows, d, d); }

int colsum_blocks(int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, 128)); }

int colsum_partial(int dtype, const void* x, int64_t rows, int64_t cols, int64_t ld, float* part, cudaStream_t st) {
  if (cols == 0) return RP_OK;
  const int esz = dtype == RP_BF16 ? 2 : 4;
  if (cols % 2 == 0 && ld % 2 == 0 && (reinterpret_cast<uintptr_t>(x) % (2 * esz)) == 0) {
    dim3 grid(colsum_blocks(rows), (unsigned)((cols / 2 + 127) / 128));
    RP_DTYPE_DISPATCH(dtype, launch_pdl(colsum_partial2_kernel<T>, grid, 128, 0, st, (const T*)x, rows, cols, ld,
                                        part));
    return check_launch("colsum_partial");
  }
  dim3 grid(colsum_blocks(rows), (unsigned)((cols + 127) / 128));
  RP_DTYPE_DISPATCH(dtype, launch_pdl(colsum_partial_kernel<T>, grid, 128, 0, st, (const T*)x, rows, cols, ld, part));
  return check_launch("colsum_partial");
}

int mask_grad(int dtype, const float* g, void* out, int64_t rows, int64_t d, uint64_t seed, uint64_t pos0,
              uint64_t thr, float scale, int drop_on, float* part, cudaStream_t st, int64_t ldo) {
  if (d == 0) return RP_OK;
  if (ldo <= 0) ldo = d;
  const VecShape vs = vec_for(d, {ldo});
  if (vs.ng) {
    RP_DTYPE_DISPATCH(dtype, RP_VW_DISPATCH(vs.vw, RP_NG_DISPATCH(vs.ng, launch_pdl(
                                 mask_grad_v4_kernel<T, NG, VW>, ln_bwd_blocks(rows), kRowThreads, 0, st, g, (T*)out,
                                 rows, (int)d, seed, pos0, thr, scale, drop_on, part, ldo))));
    return check_launch("mask_grad");
  }
  // scalar fallback writes colsum_blocks(rows) partial rows; callers pass
  // rp_mask_grad_blocks(rows, d) to the finish
  dim3 grid(colsum_blocks(rows), (unsigned)((d + 127) / 128));
  RP_DTYPE_DISPATCH(dtype, mask_grad_kernel<T><<<grid, 128, 0, st>>>(g, (T*)out, rows, (int)d, seed, pos0, thr,
                                                                     scale, drop_on, part, ldo));
  return check_launch("mask_grad");
}

int softmax_causal(int dtype, const float* s, void* p, int64_t rows, int64_t Tn, int64_t ld, cudaStream_t st) {
  if (rows == 0) return RP_OK;
  const int npl = npl_for(Tn);
  RP_DTYPE_DISPATCH(dtype, RP_NPL_DISPATCH(npl, launch_pdl(softmax_causal_kernel<T, NPL>, row_blocks(rows), kRowThreads, 0, st, 
                                                    s, (T*)p, rows, (int)Tn, ld)));
  return check_launch("softmax_causal");
}

int softmax_bwd(int dtype, const float* gp, const void* p, void* gs, float scale, int64_t rows, int64_t Tn,
                int64_t ld, cudaStream_t st) {
  if (rows == 0) return RP_OK;
  const int npl = npl_for(Tn);
  RP_DTYPE_DISPATCH(dtype, RP_NPL_DISPATCH(npl, launch_pdl(softmax_bwd_kernel<T, NPL>, row_blocks(rows), kRowThreads, 0, st, 
                                                    gp, (const T*)p, (T*)gs, scale, rows, (int)Tn, ld)));
  return check_launch("softmax_bwd");
}

}  // namespace rp
