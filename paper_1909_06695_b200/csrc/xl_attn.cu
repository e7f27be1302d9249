// Fused Transformer-XL relative-position attention scores on tcgen05
// (the math is restated in oracle/xl.py, Dai et al. 2019
// section 3.3 -- the reference has no XL path).
//
// Forward (bf16, head dim 64): one CTA per (head*batch, 128-query tile)
// computes, per 128-key tile,
//     AC   = (q + u) k^T                 128 x 128   (TMEM cols   0..127)
//     BDb  = (q + v) R[p0 .. p0+255]^T   128 x 256   (TMEM cols 128..383)
// on the tensor cores from TMA-staged, 128B-swizzled operands, where the
// 256-row band of the relative encodings covers every distance the tile
// needs: BD[i, j] = BDb[r, 127 - r + jj] (r = i - i0, jj = j - j0).  The
// per-row shift is done through a per-warp shared-memory ring.  Softmax
// warps build s = (AC + BD) * scale under the causal + memory-validity mask
// (M - mem_len <= j <= M + i) and run two passes over the key tiles: online
// max / sum, then P = exp(s - max) / sum written once in bf16.  The fp32
// AC / BD score matrices of the unfused path (two GEMM outputs of
// H*B*T*Kl floats each, re-read by a softmax kernel) never reach HBM.
//
// Warp roles (384 threads): warp 0 TMA producer, warp 1 MMA issuer (one
// thread), warp 2 TMEM allocator, warps 4..11 softmax (warp w owns TMEM lane
// quarter w % 4 and half of each key tile's columns).
#include <algorithm>

#include "common.cuh"
#include "rp_internal.h"

#ifndef RP_TRY0
#define RP_TRY0(x)               \
  do {                           \
    if (int _e = (x)) return _e; \
  } while (0)
#endif

namespace rp {
namespace {

constexpr int kQT = 128;                  // query rows per CTA
constexpr int kKT = 128;                  // keys per step
constexpr int kBand = 256;                // relative-encoding rows per step
constexpr int kRowBytes = 128;            // dh = 64 bf16
constexpr int kQBytes = kQT * kRowBytes;  // 16 KB
constexpr int kKBytes = kKT * kRowBytes;  // 16 KB
constexpr int kRBytes = kBand * kRowBytes;  // 32 KB
constexpr int kStageBytes = kKBytes + kRBytes;
constexpr int kStages = 2;
constexpr int kRing = 66;                 // floats per staged band row: 2 chunks of 32, stride == 2 (mod 32)
constexpr int kRingWarp = 32 * kRing;
constexpr int kSoftWarps = 8;
constexpr int kThreadsFwd = 384;
constexpr int kTmemCols = 512;
constexpr int kSmemFwd = 1024 /*align*/ + 2 * kQBytes + kStages * kStageBytes + kSoftWarps * kRingWarp * 4 +
                         2 * kQT * 2 * 4 /*stats*/ + 128 /*barriers*/;

struct FwdParams {
  __nv_bfloat16* p;
  int64_t ldp;
  int B, T, M, Kl, lo, nqt;
  float c2;  // scale * log2(e)
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 32 TMEM columns of this thread's row -> staged ring slot (float2 stores:
// conflict-free with the == 2 (mod 32) row stride)
__device__ __forceinline__ void stage_band(float* ring_row, int slot, const uint32_t (&v)[32]) {
  float2* dst = reinterpret_cast<float2*>(ring_row + 32 * slot);
#pragma unroll
  for (int t = 0; t < 16; ++t) dst[t] = make_float2(__uint_as_float(v[2 * t]), __uint_as_float(v[2 * t + 1]));
}

__global__ void __launch_bounds__(kThreadsFwd, 1)
    xl_attn_fwd_kernel(const __grid_constant__ CUtensorMap mQu, const __grid_constant__ CUtensorMap mQv,
                       const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mR,
                       const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQu = smem;
  uint8_t* sQv = smem + kQBytes;
  uint8_t* stages = smem + 2 * kQBytes;
  float* ring = reinterpret_cast<float*>(stages + kStages * kStageBytes);
  float* stats = ring + kSoftWarps * kRingWarp;  // [half][row][max, sum]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stats + 2 * kQT * 2);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 3;
  uint64_t* s_full = bars + 5;
  uint64_t* s_empty = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hb = blockIdx.x / p.nqt, qt = blockIdx.x % p.nqt;
  const int h = hb / p.B;
  const int i0 = qt * kQT;
  const int imax = min(i0 + kQT, p.T) - 1;
  const int jt_lo = p.lo / kKT, jt_hi = min(p.M + imax, p.Kl - 1) / kKT;
  const int per_pass = jt_hi - jt_lo + 1;
  const int nsteps = 2 * per_pass;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQu);
    tma_prefetch(&mQv);
    tma_prefetch(&mK);
    tma_prefetch(&mR);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, kSoftWarps * 32);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_expect_tx(q_full, 2 * kQBytes);
      tma_load_3d(sQu, &mQu, q_full, 0, i0, hb);
      tma_load_3d(sQv, &mQv, q_full, 0, i0, hb);
      for (int n = 0; n < nsteps; ++n) {
        const int s = n & 1;
        mbar_wait(&kv_empty[s], ((n >> 1) & 1) ^ 1);
        const int j0 = (jt_lo + n % per_pass) * kKT;
        uint8_t* sk = stages + s * kStageBytes;
        mbar_expect_tx(&kv_full[s], kStageBytes);
        tma_load_3d(sk, &mK, &kv_full[s], 0, j0, hb);
        tma_load_3d(sk + kKBytes, &mR, &kv_full[s], 0, p.T - kQT - i0 + j0, h);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t id_ac = umma_idesc(false, false, false, kQT, kKT);
      const uint32_t id_bd = umma_idesc(false, false, false, kQT, kBand);
      const uint32_t qa = smem_u32(sQu), qb = smem_u32(sQv);
      mbar_wait(q_full, 0);
      for (int n = 0; n < nsteps; ++n) {
        const int s = n & 1;
        mbar_wait(&kv_full[s], (n >> 1) & 1);
        if (n > 0) mbar_wait(s_empty, (n - 1) & 1);
        tc_fence_after();
        const uint32_t kb = smem_u32(stages + s * kStageBytes), rb = kb + kKBytes;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(tmem_base, umma_desc(qa + 32 * k, 16, 1024), umma_desc(kb + 32 * k, 16, 1024), id_ac,
                        k > 0);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(tmem_base + kKT, umma_desc(qb + 32 * k, 16, 1024), umma_desc(rb + 32 * k, 16, 1024), id_bd,
                        k > 0);
        tc_commit(&kv_empty[s]);
        tc_commit(s_full);
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: row r = 32 q + lane, key columns [64 half, +64) ----------------
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const int i = i0 + r;
    const bool row_ok = i < p.T;
    const int jhi = p.M + i;
    float* myring = ring + (warp - 4) * kRingWarp + lane * kRing;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    const int cb0 = 96 - 32 * q + 64 * half;  // first band column this warp stages
    __nv_bfloat16* prow = p.p + ((int64_t)hb * p.T + i) * p.ldp;
    float m = -INFINITY, l = 0.f, inv = 0.f;
    for (int n = 0; n < nsteps; ++n) {
      const bool pass2 = n >= per_pass;
      if (n == per_pass) {
        // merge the two column halves' statistics of each row
        stats[(half * kQT + r) * 2] = m;
        stats[(half * kQT + r) * 2 + 1] = l;
        named_sync(1, kSoftWarps * 32);
        const float mo = stats[((1 - half) * kQT + r) * 2], lo_ = stats[((1 - half) * kQT + r) * 2 + 1];
        const float mm = fmaxf(m, mo);
        const float ll = (m == -INFINITY ? 0.f : l * ex2(m - mm)) + (mo == -INFINITY ? 0.f : lo_ * ex2(mo - mm));
        m = mm;
        inv = ll > 0.f ? 1.f / ll : 0.f;
        // columns of key tiles no query of this tile can see
        if (row_ok) {
          const uint4 z = make_uint4(0, 0, 0, 0);
          const int64_t a0 = half ? (int64_t)(jt_hi + 1) * kKT : 0;
          const int64_t a1 = half ? p.ldp : (int64_t)jt_lo * kKT;
          for (int64_t c = a0; c < a1; c += 8) *reinterpret_cast<uint4*>(prow + c) = z;
        }
      }
      const int j0 = (jt_lo + n % per_pass) * kKT + 64 * half;
      mbar_wait(s_full, n & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tl + kKT + cb0, v);
      stage_band(myring, 0, v);
      tmem_ld32(tl + kKT + cb0 + 32, v);
      stage_band(myring, 1, v);
      __syncwarp();
#pragma unroll 1
      for (int k = 0; k < 2; ++k) {
        uint32_t a[32];
        tmem_ld32(tl + 64 * half + 32 * k, a);
        if (k == 1) {
          tc_fence_before();
          mbar_arrive(s_empty);  // every TMEM read of this step is done
        }
        const int jb = j0 + 32 * k;
        const int off = 31 + 32 * k - lane;
        float s[32];
        float cm = -INFINITY;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int j = jb + t;
          const float bd = myring[(off + t) & 63];
          const float x = (__uint_as_float(a[t]) + bd) * p.c2;
          s[t] = (j >= p.lo && j <= jhi) ? x : -INFINITY;
          cm = fmaxf(cm, s[t]);
        }
        if (k == 0) {
          __syncwarp();  // slot 0 (band chunk 0) fully read
          tmem_ld32(tl + kKT + cb0 + 64, v);
          stage_band(myring, 0, v);
          __syncwarp();
        }
        if (!pass2) {
          const float mn = fmaxf(m, cm);
          if (mn != -INFINITY) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 32; ++t) acc += ex2(s[t] - mn);
            l = (m == -INFINITY ? 0.f : l * ex2(m - mn)) + acc;
            m = mn;
          }
        } else if (row_ok) {
          uint32_t w[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(ex2(s[2 * t] - m) * inv, ex2(s[2 * t + 1] - m) * inv);
            w[t] = *reinterpret_cast<uint32_t*>(&b2);
          }
          if (jb + 32 <= p.ldp) {
            uint4* dst = reinterpret_cast<uint4*>(prow + jb);
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
          } else {
            const __nv_bfloat16* wb = reinterpret_cast<const __nv_bfloat16*>(w);
            for (int t = 0; t < 32 && jb + t < p.ldp; ++t) prow[jb + t] = wb[t];
          }
        }
      }
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace

int xl_attn_fwd(const void* qu, const void* qv, const void* kh, const void* rh, void* probs, int64_t ldp, int64_t B,
                int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale, cudaStream_t st) {
  if (dh != 64) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: head dim must be 64 (got %d)", dh);
  const int64_t Kl = M + Tn, HB = (int64_t)H * B;
  if (ldp < Kl || ldp % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: ldp must be >= M+T and a multiple of 8");
  if (mem_len < 0 || mem_len > M) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: mem_len out of range");
  if ((reinterpret_cast<uintptr_t>(probs) & 15) != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: P not 16B aligned");
  CUtensorMap mqu, mqv, mk, mr;
  RP_TRY0(tma_map_bf16(&mqu, qu, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mqv, qv, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mk, kh, dh, Kl, dh, HB, Kl * dh, 64, kKT));
  RP_TRY0(tma_map_bf16(&mr, rh, dh, Kl, dh, H, Kl * dh, 64, kBand));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(xl_attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFwd);
    attr = true;
  }
  FwdParams p;
  p.p = static_cast<__nv_bfloat16*>(probs);
  p.ldp = ldp;
  p.B = (int)B;
  p.T = (int)Tn;
  p.M = (int)M;
  p.Kl = (int)Kl;
  p.lo = (int)(M - mem_len);
  p.nqt = (int)((Tn + kQT - 1) / kQT);
  p.c2 = scale * 1.4426950408889634f;
  const int64_t grid = HB * p.nqt;
  if (grid <= 0) return RP_OK;
  xl_attn_fwd_kernel<<<(unsigned)grid, kThreadsFwd, kSmemFwd, st>>>(mqu, mqv, mk, mr, p);
  return check_launch("xl_attn_fwd");
}

}  // namespace rp
