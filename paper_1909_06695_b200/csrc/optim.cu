// Fused optimizer updates over a module's flat parameter buffer
// (reference optim.py:52-126), device-side weight init with the reference's
// counter RNG (layers.py:107-112, 149-166, tensor.py:72-74), dtype casts and a
// deterministic squared-norm reduction (engine.py:72-80).
//
// Adam/SGD read the fp32 master weights, gradient and moments once, write
// weights and moments once, and in the same pass write the compute-dtype copy
// of the updated weights straight into the next snapshot-ring slot (the
// reference's separate deep copy, model.py:171-172, disappears).  Any
// non-finite updated weight raises the NONFINITE status bit (optim.py:47-49).
#include <algorithm>

#include "common.cuh"
#include "rp_internal.h"

namespace rp {

template <typename T>
__global__ void adam_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, T* __restrict__ copy, int64_t n, float lr, float b1, float b2,
                            float eps, float c1, float c2, int32_t* flag) {
  bool finite = true;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    float mi = m[i] * b1 + (1.f - b1) * gi;
    float vi = v[i] * b2 + (1.f - b2) * (gi * gi);
    m[i] = mi;
    v[i] = vi;
    const float wi = w[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    w[i] = wi;
    finite &= isfinite(wi);
    if (copy) copy[i] = from_f<T>(wi);
  }
  if (!finite && flag) atomicOr(flag, RP_FLAG_NONFINITE);
}

// 4-wide variant: n % 4 == 0 and every pointer 16-byte aligned (8 for a bf16 copy).
template <typename T>
__global__ void adam_v4_kernel(float4* __restrict__ w, const float4* __restrict__ g, float4* __restrict__ m,
                               float4* __restrict__ v, T* __restrict__ copy, int64_t n4, float lr, float b1, float b2,
                               float eps, float c1, float c2, int32_t* flag) {
  bool finite = true;
  const float ic1 = 1.f / c1, ic2 = 1.f / c2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 gi = g[i];
    float4 mi = m[i], vi = v[i], wi = w[i];
    float* mp = &mi.x;
    float* vp = &vi.x;
    float* wp = &wi.x;
    const float* gp = &gi.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mp[q] = mp[q] * b1 + (1.f - b1) * gp[q];
      vp[q] = vp[q] * b2 + (1.f - b2) * (gp[q] * gp[q]);
      wp[q] = wp[q] - lr * (mp[q] * ic1) / (sqrtf(vp[q] * ic2) + eps);
      finite &= isfinite(wp[q]);
    }
    m[i] = mi;
    v[i] = vi;
    w[i] = wi;
    if (copy) {
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 a = __floats2bfloat162_rn(wi.x, wi.y), b = __floats2bfloat162_rn(wi.z, wi.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&a);
        u.y = *reinterpret_cast<uint32_t*>(&b);
        reinterpret_cast<uint2*>(copy)[i] = u;
      } else {
        reinterpret_cast<float4*>(copy)[i] = wi;
      }
    }
  }
  if (!finite && flag) atomicOr(flag, RP_FLAG_NONFINITE);
}

template <typename T>
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, T* __restrict__ copy, int64_t n,
                           float lr, int32_t* flag) {
  bool finite = true;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float wi = w[i] - lr * g[i];
    w[i] = wi;
    finite &= isfinite(wi);
    if (copy) copy[i] = from_f<T>(wi);
  }
  if (!finite && flag) atomicOr(flag, RP_FLAG_NONFINITE);
}

// Mixed tied gradient (reference engine.py:54-69): out = a*vo + b*vi.
__global__ void axpby_kernel(const float* __restrict__ x, float a, const float* __restrict__ y, float b,
                             float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (x ? a * x[i] : 0.f) + (y ? b * y[i] : 0.f);
}

// out[i] = ((bits53(seed, pos0 + i) * 2^-53) * 2 - 1) * scale, evaluated in
// fp64 exactly as the reference's uniform_signed, then rounded to fp32.
__global__ void init_uniform_kernel(float* __restrict__ out, int64_t n, uint64_t seed, uint64_t pos0, double scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)rng_bits53(seed, pos0 + (uint64_t)i) * (1.0 / 9007199254740992.0);
    out[i] = (float)((u * 2.0 - 1.0) * scale);
  }
}

template <typename Tin, typename Tout>
__global__ void cast_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = from_f<Tout>(to_f(in[i]));
}

__global__ void sq_norm_partial_kernel(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = x[i];
    s += t * t;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int n, double* __restrict__ out, int accumulate) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = accumulate ? *out + s : s;
  }
}

namespace {
inline int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }
}  // namespace

int adam_step(float* w, const float* g, float* m, float* v, void* copy, int copy_dtype, int64_t n, float lr, float b1,
              float b2, float eps, float c1, float c2, int32_t* flag, cudaStream_t st) {
  if (n == 0) return RP_OK;
  auto al = [](const void* p, int a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; };
  if (n % 4 == 0 && al(w, 16) && al(g, 16) && al(m, 16) && al(v, 16) &&
      (!copy || al(copy, copy_dtype == RP_BF16 ? 8 : 16))) {
    const int64_t n4 = n / 4;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, 148 * 16));
    if (copy_dtype == RP_BF16)
      adam_v4_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((float4*)w, (const float4*)g, (float4*)m, (float4*)v,
                                                          (__nv_bfloat16*)copy, n4, lr, b1, b2, eps, c1, c2, flag);
    else
      adam_v4_kernel<float><<<grid, 256, 0, st>>>((float4*)w, (const float4*)g, (float4*)m, (float4*)v,
                                                  (float*)copy, n4, lr, b1, b2, eps, c1, c2, flag);
    return check_launch("adam");
  }
  if (copy_dtype == RP_BF16)
    adam_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(w, g, m, v, (__nv_bfloat16*)copy, n, lr, b1, b2, eps, c1,
                                                             c2, flag);
  else
    adam_kernel<float><<<grid_for(n), 256, 0, st>>>(w, g, m, v, (float*)copy, n, lr, b1, b2, eps, c1, c2, flag);
  return check_launch("adam");
}

int sgd_step(float* w, const float* g, void* copy, int copy_dtype, int64_t n, float lr, int32_t* flag,
             cudaStream_t st) {
  if (n == 0) return RP_OK;
  if (copy_dtype == RP_BF16)
    sgd_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(w, g, (__nv_bfloat16*)copy, n, lr, flag);
  else
    sgd_kernel<float><<<grid_for(n), 256, 0, st>>>(w, g, (float*)copy, n, lr, flag);
  return check_launch("sgd");
}

// y += alpha * x (float4 where aligned): accumulation of a micro-batched
// slot's per-row-block weight gradients, in row-block order
__global__ void axpy_kernel(float* __restrict__ y, const float* __restrict__ x, float alpha, int64_t n, int vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t n4 = n / 4;
    for (int64_t q = i; q < n4; q += stride) {
      float4 a = reinterpret_cast<float4*>(y)[q];
      const float4 b = reinterpret_cast<const float4*>(x)[q];
      a.x = fmaf(alpha, b.x, a.x);
      a.y = fmaf(alpha, b.y, a.y);
      a.z = fmaf(alpha, b.z, a.z);
      a.w = fmaf(alpha, b.w, a.w);
      reinterpret_cast<float4*>(y)[q] = a;
    }
    for (int64_t q = n4 * 4 + i; q < n; q += stride) y[q] = fmaf(alpha, x[q], y[q]);
  } else {
    for (; i < n; i += stride) y[i] = fmaf(alpha, x[i], y[i]);
  }
}

// GELU, exact erf form: 8 bf16 (16 bytes) or 4 fp32 per thread per step --
// one read and one write of the pre-activation, at the HBM roofline
__device__ __forceinline__ float gelu_f(float z) { return 0.5f * z * (1.f + erff(z * 0.70710678118654752f)); }

__global__ void gelu_bf16_kernel(const uint4* __restrict__ z, uint4* __restrict__ y, int64_t n8) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    const uint4 u = z[i];
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      __nv_bfloat162 o = __floats2bfloat162_rn(gelu_f(f.x), gelu_f(f.y));
      w[e] = *reinterpret_cast<uint32_t*>(&o);
    }
    y[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename T>
__global__ void gelu_tail_kernel(const T* __restrict__ z, T* __restrict__ y, int64_t n0, int64_t n) {
  for (int64_t i = n0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Io<T>::st(y + i, gelu_f(Io<T>::ld(z + i)));
}

int gelu_fwd(int dtype, const void* z, void* y, int64_t n, cudaStream_t st) {
  if (n == 0) return RP_OK;
  if (dtype == RP_BF16 && ((reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
    const int64_t n8 = n / 8;
    if (n8) gelu_bf16_kernel<<<grid_for(n8), 256, 0, st>>>((const uint4*)z, (uint4*)y, n8);
    if (n8 * 8 < n)
      gelu_tail_kernel<__nv_bfloat16><<<1, 256, 0, st>>>((const __nv_bfloat16*)z, (__nv_bfloat16*)y, n8 * 8, n);
  } else if (dtype == RP_BF16) {
    gelu_tail_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)z, (__nv_bfloat16*)y, 0, n);
  } else {
    gelu_tail_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)z, (float*)y, 0, n);
  }
  return check_launch("gelu_fwd");
}

int axpy(float* y, const float* x, float alpha, int64_t n, cudaStream_t st) {
  if (n == 0) return RP_OK;
  const int vec = ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  axpy_kernel<<<grid_for(vec ? (n + 3) / 4 : n), 256, 0, st>>>(y, x, alpha, n, vec);
  return check_launch("axpy");
}

int embedding_gradient(int64_t t, int64_t K, const float* vo, const float* vi, float* out, int64_t n,
                       int convention, cudaStream_t st) {
  if (n == 0) return RP_OK;
  if (convention != 0 && convention != 1) return set_error(RP_ERR_INVALID, "unknown tied_grad convention");
  const bool padded = t - K + 1 < 0;  // the input-side half does not exist yet: a zero packet
  if (padded && vi) return set_error(RP_ERR_SCHEDULE, "stale embedding gradient before step K-1");
  if (!padded && !vi) return set_error(RP_ERR_SCHEDULE, "missing stale embedding gradient");
  const float c = padded ? 0.f : (convention == 0 ? 0.5f : 1.f);
  axpby_kernel<<<grid_for(n), 256, 0, st>>>(padded ? nullptr : vo, c, vi, c, out, n);
  return check_launch("embedding_gradient");
}

int init_uniform(float* out, int64_t n, uint64_t seed, uint64_t pos0, double scale, cudaStream_t st) {
  if (n == 0) return RP_OK;
  init_uniform_kernel<<<grid_for(n), 256, 0, st>>>(out, n, seed, pos0, scale);
  return check_launch("init_uniform");
}

int cast(const void* in, int in_dtype, void* out, int out_dtype, int64_t n, cudaStream_t st) {
  if (n == 0) return RP_OK;
  if (in_dtype == RP_F32 && out_dtype == RP_BF16)
    cast_kernel<float, __nv_bfloat16><<<grid_for(n), 256, 0, st>>>((const float*)in, (__nv_bfloat16*)out, n);
  else if (in_dtype == RP_BF16 && out_dtype == RP_F32)
    cast_kernel<__nv_bfloat16, float><<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)in, (float*)out, n);
  else if (in_dtype == RP_F32 && out_dtype == RP_F32)
    cast_kernel<float, float><<<grid_for(n), 256, 0, st>>>((const float*)in, (float*)out, n);
  else
    cast_kernel<__nv_bfloat16, __nv_bfloat16>
        <<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)in, (__nv_bfloat16*)out, n);
  return check_launch("cast");
}

int sq_norm(const float* x, int64_t n, double* part /* >= 296 */, double* out, int accumulate, cudaStream_t st) {
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 296));
  sq_norm_partial_kernel<<<nb, 256, 0, st>>>(x, n, part);
  if (int e = check_launch("sq_norm")) return e;
  sum_partials_kernel<<<1, 32, 0, st>>>(part, nb, out, accumulate);
  return check_launch("sq_norm_sum");
}

}  // namespace rp
