// Row gather / scatter / augment kernels for the adaptive tied softmax head
// (BASELINE configs[3]; restated in oracle/adaptive.py --
// the reference has no adaptive softmax).  The contractions themselves run on
// the tcgen05 head GEMM (log-sum-exp and softmax-gradient epilogues); these
// kernels only move rows:
//   * rows_copy:    dst[r, :cols] = src[r, :cols] (dtype conversion allowed),
//                   optionally dst[r, cols] = value(r) and zeros up to ld_dst
//                   -- builds [h | 1] and [V_head ; W_c | b_c] so the cluster
//                   bias rides in the GEMM as one extra K column;
//   * rows_gather:  dst[r] = src[idx[r]]      (rows of a tail cluster);
//   * rows_scatter_add: dst[idx[r]] += src[r] (fp32; a row appears in one
//                   cluster only, so there are no write conflicts and the
//                   result is deterministic).
#include <algorithm>

#include "common.cuh"
#include "rp_internal.h"

namespace rp {
namespace {

constexpr int kThreads = 256;

template <typename S, typename D>
__global__ void rows_copy_kernel(const S* __restrict__ src, int64_t ld_src, int64_t rows, int cols,
                                 const float* __restrict__ val, float val_const, int aug, D* __restrict__ dst,
                                 int64_t ld_dst) {
  const int64_t total = rows * ld_dst;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ld_dst;
    const int c = (int)(e - r * ld_dst);
    float v;
    if (c < cols)
      v = to_f(src[r * ld_src + c]);
    else if (aug && c == cols)
      v = val ? val[r] : val_const;
    else
      v = 0.f;
    dst[e] = from_f<D>(v);
  }
}

template <typename T>
__global__ void rows_gather_kernel(const T* __restrict__ src, int64_t ld_src, const int64_t* __restrict__ idx,
                                   int64_t n, int cols, T* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e - r * cols);
    dst[r * ld_dst + c] = src[idx[r] * ld_src + c];
  }
}

__global__ void rows_scatter_add_kernel(const float* __restrict__ src, int64_t ld_src, const int64_t* __restrict__ idx,
                                        int64_t n, int cols, float* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e - r * cols);
    dst[idx[r] * ld_dst + c] += src[r * ld_src + c];
  }
}

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 32); }

}  // namespace

int rows_copy(int src_dtype, const void* src, int64_t ld_src, int64_t rows, int64_t cols, const float* val,
              float val_const, int aug, int dst_dtype, void* dst, int64_t ld_dst, cudaStream_t st) {
  if (cols < 0 || ld_dst < cols + (aug ? 1 : 0) || ld_src < cols)
    return set_error(RP_ERR_DIMENSION, "rows_copy: bad leading dimensions");
  if (rows == 0 || ld_dst == 0) return RP_OK;
  const int g = grid_for(rows * ld_dst);
  const int c = (int)cols;
  if (src_dtype == RP_BF16 && dst_dtype == RP_BF16)
    rows_copy_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, ld_src, rows, c, val, val_const, aug,
                                             (__nv_bfloat16*)dst, ld_dst);
  else if (src_dtype == RP_F32 && dst_dtype == RP_BF16)
    rows_copy_kernel<<<g, kThreads, 0, st>>>((const float*)src, ld_src, rows, c, val, val_const, aug,
                                             (__nv_bfloat16*)dst, ld_dst);
  else if (src_dtype == RP_F32 && dst_dtype == RP_F32)
    rows_copy_kernel<<<g, kThreads, 0, st>>>((const float*)src, ld_src, rows, c, val, val_const, aug, (float*)dst,
                                             ld_dst);
  else
    rows_copy_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, ld_src, rows, c, val, val_const, aug,
                                             (float*)dst, ld_dst);
  return check_launch("rows_copy");
}

int rows_gather(int dtype, const void* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols, void* dst,
                int64_t ld_dst, cudaStream_t st) {
  if (n == 0 || cols == 0) return RP_OK;
  const int g = grid_for(n * cols);
  if (dtype == RP_BF16)
    rows_gather_kernel<<<g, kThreads, 0, st>>>((const __nv_bfloat16*)src, ld_src, idx, n, (int)cols,
                                               (__nv_bfloat16*)dst, ld_dst);
  else
    rows_gather_kernel<<<g, kThreads, 0, st>>>((const float*)src, ld_src, idx, n, (int)cols, (float*)dst, ld_dst);
  return check_launch("rows_gather");
}

int rows_scatter_add(const float* src, int64_t ld_src, const int64_t* idx, int64_t n, int64_t cols, float* dst,
                     int64_t ld_dst, cudaStream_t st) {
  if (n == 0 || cols == 0) return RP_OK;
  rows_scatter_add_kernel<<<grid_for(n * cols), kThreads, 0, st>>>(src, ld_src, idx, n, (int)cols, dst, ld_dst);
  return check_launch("rows_scatter_add");
}

}  // namespace rp
