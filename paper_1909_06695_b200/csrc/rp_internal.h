// Internal declarations shared by the ringpipe-b200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ringpipe_b200.h"

namespace rp {

// Records a formatted error message (thread-local) and returns `status`.
int set_error(int status, const char* fmt, ...);
// Returns RP_OK or RP_ERR_CUDA with the launch error recorded.
int check_launch(const char* what);

int gemm(const rp_gemm_args& a, cudaStream_t stream);
int gemm_tile_n(int64_t N);
int tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
               cudaStream_t stream);

}  // namespace rp
