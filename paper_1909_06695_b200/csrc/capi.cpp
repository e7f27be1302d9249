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

int rp_gemm_tile_n(int64_t N) { return rp::gemm_tile_n(N); }

int rp_tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
                  void* stream) {
  return rp::tf32_split(x, hi, lo, rows, cols, ld_src, ld_dst, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
