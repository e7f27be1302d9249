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
#include <cstdio>
#include <cstdlib>

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
constexpr int kKT = 128;                  // keys per backward step
constexpr int kRowBytes = 128;            // one 128B-swizzle atom: 64 bf16 of the head dim
constexpr int kStages = 2;
constexpr int kSoftWarps = 8;
// forward: 64 keys per step, so two steps' accumulators (AC 64 + band 192
// columns each) fit TMEM and the MMA of step n+1 overlaps the softmax of n
constexpr int kFKT = 64;                  // keys per forward step
constexpr int kFBand = kFKT + 128;        // relative-encoding rows per forward step (covers 127 + 64 distances)
// NA = head dim / 64 atoms: a tile of R rows is NA [R x 64] swizzle atoms
template <int NA>
struct FwdCfg {
  static constexpr int QBytes = kQT * kRowBytes * NA;
  static constexpr int KBytes = kFKT * kRowBytes * NA;
  static constexpr int RBytes = kFBand * kRowBytes * NA;
  static constexpr int StageBytes = KBytes + RBytes;
  static constexpr int Stages = NA == 1 ? 3 : 1;  // dh 128: one stage keeps Q + ring in smem
};
constexpr int kFBuf = 256;                // TMEM columns per accumulator buffer
constexpr int kRing = 66;                 // floats per staged band row: 2 chunks of 32, stride == 2 (mod 32)
constexpr int kRingWarp = 32 * kRing;
constexpr int kThreadsFwd = 384;
constexpr int kTmemCols = 512;
constexpr int kPStage = 32 * 64;  // per softmax warp: 32 rows x 32 bf16 of P, 64B-swizzled (TMA store)
template <int NA>
constexpr int smem_fwd() {
  return 1024 /*align*/ + 2 * FwdCfg<NA>::QBytes + FwdCfg<NA>::Stages * FwdCfg<NA>::StageBytes +
         kSoftWarps * kPStage + kSoftWarps * kRingWarp * 4 + 2 * kQT * 2 * 4 /*stats*/ + 128 /*barriers*/;
}

struct FwdParams {
  __nv_bfloat16* p;
  int64_t ldp;
  int B, T, M, Kl, lo, nqt;
  int heavy_first;  // CTA order: last (widest causal window) query tiles first
  float c2;  // scale * log2(e)
  int dbg;   // diagnostics (RP_XL_DBG): 1 = softmax warps only wait/arrive, 2 = no MMAs
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// CTA -> (head*batch, query tile).  Query tile qt sees keys up to M + 128 qt + 127,
// so the last tiles carry the most key tiles; heavy-first issues every
// head's last tile before any first tile (longest work first shortens the
// tail of the ~4.8 waves at C3).
__device__ __forceinline__ void cta_tile(int nqt, int heavy_first, int& hb, int& qt) {
  if (heavy_first) {
    const int nhb = gridDim.x / nqt;
    qt = nqt - 1 - (int)blockIdx.x / nhb;
    hb = (int)blockIdx.x % nhb;
  } else {
    hb = (int)blockIdx.x / nqt;
    qt = (int)blockIdx.x % nqt;
  }
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 32 TMEM columns of this thread's row -> staged ring slot (float2 stores:
// conflict-free with the == 2 (mod 32) row stride)
// Only the pairs the lane's shifted read [31 - lane, 63 - lane) touches are
// written (a predicated-off store moves no data): half the staging traffic.
__device__ __forceinline__ void stage_band(float* ring_row, int slot, const uint32_t (&v)[32], int lane) {
  float2* dst = reinterpret_cast<float2*>(ring_row + 32 * slot);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const bool used = slot == 0 ? (2 * t + 1 >= 31 - lane) : (2 * t <= 30 - lane);
    if (used) dst[t] = make_float2(__uint_as_float(v[2 * t]), __uint_as_float(v[2 * t + 1]));
  }
}

__device__ __forceinline__ void tma_store_3d_p(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// TMA-load NA swizzle atoms of a [rows x 64 NA] tile (atom a at + a * rows * 128 B)
template <int NA>
__device__ __forceinline__ void tma_atoms(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int rows, int r0,
                                          int b) {
#pragma unroll
  for (int a = 0; a < NA; ++a) tma_load_3d(dst + a * rows * kRowBytes, map, bar, 64 * a, r0, b);
}
// K-major SW128 descriptor of k-step k (16 elements) of an NA-atom tile of `rows` rows
template <int NA>
__device__ __forceinline__ uint64_t atom_desc(uint32_t base, int rows, int k) {
  return umma_desc(base + (k >> 2) * rows * kRowBytes + 32 * (k & 3), 16, 1024);
}

template <int NA>
__global__ void __launch_bounds__(kThreadsFwd, 1)
    xl_attn_fwd_kernel(const __grid_constant__ CUtensorMap mQu, const __grid_constant__ CUtensorMap mQv,
                       const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mR,
                       const __grid_constant__ CUtensorMap mP, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t* sQu = smem;
  using C = FwdCfg<NA>;
  uint8_t* sQv = smem + C::QBytes;
  uint8_t* stages = smem + 2 * C::QBytes;
  uint8_t* pstage = stages + C::Stages * C::StageBytes;  // 1024-aligned
  float* ring = reinterpret_cast<float*>(pstage + kSoftWarps * kPStage);
  float* stats = ring + kSoftWarps * kRingWarp;  // [half][row][max, sum]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stats + 2 * kQT * 2);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [kFStages]
  uint64_t* kv_empty = bars + 4;  // [kFStages]
  uint64_t* s_full = bars + 7;    // [2]
  uint64_t* s_empty = bars + 9;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int hb, qt;
  cta_tile(p.nqt, p.heavy_first, hb, qt);
  const int h = hb / p.B;
  const int i0 = qt * kQT;
  const int imax = min(i0 + kQT, p.T) - 1;
  const int jt_lo = p.lo / kFKT, jt_hi = min(p.M + imax, p.Kl - 1) / kFKT;
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
    for (int s = 0; s < C::Stages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], kSoftWarps * 32);
    }
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
      mbar_expect_tx(q_full, 2 * C::QBytes);
      tma_atoms<NA>(sQu, &mQu, q_full, kQT, i0, hb);
      tma_atoms<NA>(sQv, &mQv, q_full, kQT, i0, hb);
      int s = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nsteps; ++n) {
        mbar_wait(&kv_empty[s], ph ^ 1);
        const int j0 = (jt_lo + n % per_pass) * kFKT;
        uint8_t* sk = stages + s * C::StageBytes;
        mbar_expect_tx(&kv_full[s], C::StageBytes);
        tma_atoms<NA>(sk, &mK, &kv_full[s], kFKT, j0, hb);
        tma_atoms<NA>(sk + C::KBytes, &mR, &kv_full[s], kFBand, p.T - kQT - i0 + j0, h);
        if (++s == C::Stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t id_ac = umma_idesc(false, false, false, kQT, kFKT);
      const uint32_t id_bd = umma_idesc(false, false, false, kQT, kFBand);
      const uint32_t qa = smem_u32(sQu), qb = smem_u32(sQv);
      mbar_wait(q_full, 0);
      int s = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nsteps; ++n) {
        const int buf = n & 1;
        mbar_wait(&s_empty[buf], ((n >> 1) & 1) ^ 1);
        mbar_wait(&kv_full[s], ph);
        tc_fence_after();
        const uint32_t kb = smem_u32(stages + s * C::StageBytes), rb = kb + C::KBytes;
        const uint32_t d = tmem_base + buf * kFBuf;
        if (!(p.dbg & 2)) {
#pragma unroll
          for (int k = 0; k < 4 * NA; ++k)
            tc_mma<false>(d, atom_desc<NA>(qa, kQT, k), atom_desc<NA>(kb, kFKT, k), id_ac, k > 0);
#pragma unroll
          for (int k = 0; k < 4 * NA; ++k)
            tc_mma<false>(d + kFKT, atom_desc<NA>(qb, kQT, k), atom_desc<NA>(rb, kFBand, k), id_bd, k > 0);
        }
        tc_commit(&kv_empty[s]);
        tc_commit(&s_full[buf]);
        if (++s == C::Stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: row r = 32 q + lane, key columns [32 half, +32) of each step ----------------
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const int i = i0 + r;
    const bool row_ok = i < p.T;
    const int jhi = p.M + i;
    float* myring = ring + (warp - 4) * kRingWarp + lane * kRing;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    // band column of key jj for row r is 127 - r + jj: this warp's 32 keys
    // need band columns [cb0, cb0 + 63)
    const int cb0 = 96 - 32 * q + 32 * half;
    const int off = 31 - lane;
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
          const int64_t a0 = half ? (int64_t)(jt_hi + 1) * kFKT : 0;
          const int64_t a1 = half ? p.ldp : (int64_t)jt_lo * kFKT;
          for (int64_t c = a0; c < a1; c += 8) *reinterpret_cast<uint4*>(prow + c) = z;
        }
      }
      const int buf = n & 1;
      const int jb = (jt_lo + n % per_pass) * kFKT + 32 * half;
      mbar_wait(&s_full[buf], (n >> 1) & 1);
      tc_fence_after();
      if (p.dbg & 1) {
        tc_fence_before();
        mbar_arrive(&s_empty[buf]);
        continue;
      }
      const uint32_t tb = tl + buf * kFBuf;
      uint32_t v0[32], v1[32], a[32];
      tmem_ld32_async(tb + kFKT + cb0, v0);
      tmem_ld32_async(tb + kFKT + cb0 + 32, v1);
      tmem_ld32_async(tb + 32 * half, a);
      tmem_wait_ld(v0);
      tmem_wait_ld(v1);
      tmem_wait_ld(a);
      tc_fence_before();
      mbar_arrive(&s_empty[buf]);  // this step's TMEM buffer is free for step n + 2
      stage_band(myring, 0, v0, lane);
      stage_band(myring, 1, v1, lane);
      __syncwarp();
      float s[32];
      float cm = -INFINITY;
      if (jb >= p.lo && jb + 31 <= p.M + i0 + 32 * q) {
        // every key of this chunk is visible to every row of the warp
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          s[t] = (__uint_as_float(a[t]) + myring[off + t]) * p.c2;
          cm = fmaxf(cm, s[t]);
        }
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int j = jb + t;
          const float x = (__uint_as_float(a[t]) + myring[off + t]) * p.c2;
          s[t] = (j >= p.lo && j <= jhi) ? x : -INFINITY;
          cm = fmaxf(cm, s[t]);
        }
      }
      __syncwarp();  // ring reads done before the next step's staging
      if (!pass2) {
        const float mn = fmaxf(m, cm);
        if (mn != -INFINITY) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int t = 0; t < 32; ++t) acc[t & 3] += ex2(s[t] - mn);
          l = (m == -INFINITY ? 0.f : l * ex2(m - mn)) + ((acc[0] + acc[1]) + (acc[2] + acc[3]));
          m = mn;
        }
      } else {
        // the warp's 32 rows x 32 columns of P: staged 64B-swizzled, one TMA
        // bulk store (rows past T and columns past ldp are clipped by the map)
        uint32_t w[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(ex2(s[2 * t] - m) * inv, ex2(s[2 * t + 1] - m) * inv);
          w[t] = row_ok ? *reinterpret_cast<uint32_t*>(&b2) : 0u;
        }
        uint8_t* tile = pstage + (warp - 4) * kPStage;
        if (lane == 0) tma_store_wait_read();  // the previous chunk's store has read the tile
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(tile + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) =
              make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        // (a box starting past the tensor's end is skipped, not issued)
        if (lane == 0 && jb < p.ldp && i0 + 32 * q < p.T) tma_store_3d_p(&mP, tile, jb, i0 + 32 * q, hb);
      }
    }
  }
  if (warp >= 4 && lane == 0) tma_store_wait_all();  // P tiles written before the CTA retires
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// ---------------------------------------------------------------------------
// Backward of the scores + softmax: per (head*batch, 128-query tile), per
// 128-key tile
//     dP = g_ctx_h v^T                  128 x 128   (TMEM, double-buffered)
//     dS = P (dP - D) * scale,  D_i = g_ctx_i . ctx_i  (= sum_j P_ij dP_ij)
// written as dAC (row-aligned, = dS) and as the un-shifted dBD[i, p] =
// dS[i, p - (T-1-i)].  dBD is assembled in a 4-chunk shared-memory ring in
// "band" coordinates (row r of key tile n covers band columns
// 128 n + 127 - r + [0, 128)); after key tile n every row's band chunk n is
// complete and one TMA bulk store writes it (128 rows x 128 columns), which
// replaces the fp32 dP GEMM output and the separate softmax-backward pass
// of the unfused path.
constexpr int kThreadsBwd = 384;
template <int NA>
struct BwdCfg {
  static constexpr int GBytes = kQT * kRowBytes * NA;  // g_ctx tile
  static constexpr int VBytes = kKT * kRowBytes * NA;  // v tile
};
constexpr int kRingChunk = kQT * 128 * 2;   // 128 rows x 128 band columns bf16 = 32 KB
constexpr int kRingChunks = 4;
template <int NA>
constexpr int smem_bwd() {
  // dh 64: dAC leaves through per-warp TMA store tiles too (dh 128 has no smem to spare: per-row stores)
  return 1024 + BwdCfg<NA>::GBytes + kStages * BwdCfg<NA>::VBytes + kRingChunks * kRingChunk +
         (NA == 1 ? kSoftWarps * kPStage : 0) + 128;
}

struct BwdParams {
  const __nv_bfloat16* p;  // P [HB, T, ldp]
  __nv_bfloat16* gac;      // dAC [HB, T, ldp]
  __nv_bfloat16* gbd;      // dBD [HB, T, ldp] (for the zero margins)
  const __nv_bfloat16* gctx;  // merged g_ctx [B*T, d]
  const __nv_bfloat16* ctx;   // merged ctx [B*T, d]
  int64_t ldp;
  int B, T, M, Kl, lo, nqt, H, d;
  int heavy_first;
  float scale;
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

// zero bf16 [a, b) of a row (16-byte stores where aligned)
__device__ __forceinline__ void zero_row(__nv_bfloat16* row, int64_t a, int64_t b) {
  const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
  while (a < b && (a & 7)) row[a++] = z;
  for (; a + 8 <= b; a += 8) *reinterpret_cast<uint4*>(row + a) = make_uint4(0, 0, 0, 0);
  for (; a < b; ++a) row[a] = z;
}

template <int NA>
__global__ void __launch_bounds__(kThreadsBwd, 1)
    xl_attn_bwd_kernel(const __grid_constant__ CUtensorMap mG, const __grid_constant__ CUtensorMap mV,
                       const __grid_constant__ CUtensorMap mBD, const __grid_constant__ CUtensorMap mAC,
                       const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t* sG = smem;
  constexpr int kGBytes = BwdCfg<NA>::GBytes, kVBytes = BwdCfg<NA>::VBytes;
  uint8_t* stages = smem + kGBytes;
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(stages + kStages * kVBytes);
  uint8_t* astage = reinterpret_cast<uint8_t*>(ring) + kRingChunks * kRingChunk;  // dAC store tiles (NA == 1)
  uint64_t* bars = reinterpret_cast<uint64_t*>(astage + (NA == 1 ? kSoftWarps * kPStage : 0));
  uint64_t* g_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 3;
  uint64_t* acc_full = bars + 5;
  uint64_t* acc_empty = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int hb, qt;
  cta_tile(p.nqt, p.heavy_first, hb, qt);
  const int h = hb / p.B, b = hb % p.B;
  const int i0 = qt * kQT;
  const int imax = min(i0 + kQT, p.T) - 1;
  const int jt_lo = p.lo / kKT, jt_hi = min(p.M + imax, p.Kl - 1) / kKT;
  const int nt = jt_hi - jt_lo + 1;
  const int P0 = p.T - kQT - i0 + jt_lo * kKT;  // band column 0 in dBD coordinates

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mG);
    tma_prefetch(&mV);
    tma_prefetch(&mBD);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(g_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kSoftWarps * 32);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(g_full, kGBytes);
      tma_atoms<NA>(sG, &mG, g_full, kQT, i0, hb);
      for (int n = 0; n < nt; ++n) {
        const int s = n & 1;
        mbar_wait(&kv_empty[s], ((n >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], kVBytes);
        tma_atoms<NA>(stages + s * kVBytes, &mV, &kv_full[s], kKT, (jt_lo + n) * kKT, hb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(false, false, false, kQT, kKT);
      const uint32_t ga = smem_u32(sG);
      mbar_wait(g_full, 0);
      for (int n = 0; n < nt; ++n) {
        const int s = n & 1;
        mbar_wait(&acc_empty[s], ((n >> 1) & 1) ^ 1);
        mbar_wait(&kv_full[s], (n >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = smem_u32(stages + s * kVBytes);
#pragma unroll
        for (int k = 0; k < 4 * NA; ++k)
          tc_mma<false>(tmem_base + s * kKT, atom_desc<NA>(ga, kQT, k), atom_desc<NA>(vb, kKT, k), idesc, k > 0);
        tc_commit(&kv_empty[s]);
        tc_commit(&acc_full[s]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const int i = i0 + r;
    const bool row_ok = i < p.T;
    const int jhi = p.M + i;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    const int64_t rowoff = ((int64_t)hb * p.T + i) * p.ldp;
    const __nv_bfloat16* prow = p.p + rowoff;
    __nv_bfloat16* arow = p.gac + rowoff;
    __nv_bfloat16* brow = p.gbd + rowoff;
    __nv_bfloat16* myring = ring + r * 128;  // + chunk * 128*128 + column
    // D_i = g_ctx_i . ctx_i over this head's 64 columns
    float D = 0.f;
    if (row_ok) {
      const int64_t mo = ((int64_t)b * p.T + i) * p.d + h * (64 * NA);
      const uint4* g4 = reinterpret_cast<const uint4*>(p.gctx + mo);
      const uint4* c4 = reinterpret_cast<const uint4*>(p.ctx + mo);
#pragma unroll
      for (int c = 0; c < 8 * NA; ++c) {
        const uint4 gu = g4[c], cu = c4[c];
        const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w}, cw[4] = {cu.x, cu.y, cu.z, cu.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[e]));
          const float2 cf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cw[e]));
          D = fmaf(gf.x, cf.x, D);
          D = fmaf(gf.y, cf.y, D);
        }
      }
      // columns outside the key tiles this query tile sees: dAC = 0, and the
      // dBD margins outside the stored band chunks
      if (half == 0) {
        zero_row(arow, 0, (int64_t)jt_lo * kKT);
        zero_row(brow, 0, lmin(lmax(P0, 0), p.ldp));
      } else {
        zero_row(arow, lmin((int64_t)(jt_hi + 1) * kKT, p.ldp), p.ldp);
        zero_row(brow, lmin(lmax((int64_t)P0 + kKT * (nt + 1), 0), p.ldp), p.ldp);
      }
    }
    // band columns before this row's first key (chunk 0)
    const __nv_bfloat16 zb = __float2bfloat16_rn(0.f);
    if (half == 0)
      for (int c = 0; c < 127 - r; ++c) myring[c] = zb;
    for (int n = 0; n < nt; ++n) {
      const int s = n & 1;
      const int jt0 = (jt_lo + n) * kKT + 64 * half;
      uint4 pr[2][4];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          pr[k][c] = (row_ok && jt0 + 32 * k + 8 * c + 8 <= p.ldp) ? reinterpret_cast<const uint4*>(prow + jt0 + 32 * k)[c]
                                                                   : make_uint4(0, 0, 0, 0);
      mbar_wait(&acc_full[s], (n >> 1) & 1);
      tc_fence_after();
      uint32_t dp[2][32];
      tmem_ld32(tl + s * kKT + 64 * half, dp[0]);
      tmem_ld32(tl + s * kKT + 64 * half + 32, dp[1]);
      tc_fence_before();
      mbar_arrive(&acc_empty[s]);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int jb = jt0 + 32 * k;
        float ds[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t w[4] = {pr[k][c].x, pr[k][c].y, pr[k][c].z, pr[k][c].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 pf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
            const int t = 8 * c + 2 * e;
            ds[t] = pf.x * (__uint_as_float(dp[k][t]) - D) * p.scale;
            ds[t + 1] = pf.y * (__uint_as_float(dp[k][t + 1]) - D) * p.scale;
          }
        }
        uint32_t o[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          // P is zero outside the window, but dP there is not: mask explicitly
          const int j = jb + 2 * t;
          const float a0 = (j >= p.lo && j <= jhi) ? ds[2 * t] : 0.f;
          const float a1 = (j + 1 >= p.lo && j + 1 <= jhi) ? ds[2 * t + 1] : 0.f;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(a0, a1);
          o[t] = *reinterpret_cast<uint32_t*>(&b2);
        }
        if constexpr (NA == 1) {
          // the warp's 32 x 32 dAC chunk: 64B-swizzled tile, one TMA bulk store
          uint8_t* tile = astage + (warp - 4) * kPStage;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(tile + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) =
                row_ok ? make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]) : make_uint4(0, 0, 0, 0);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && jb < p.ldp && i0 + 32 * q < p.T) tma_store_3d_p(&mAC, tile, jb, i0 + 32 * q, hb);
        } else if (row_ok) {
          if (jb + 32 <= p.ldp) {
            uint4* dst = reinterpret_cast<uint4*>(arow + jb);
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[c] = make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
          } else {
            for (int t = 0; t < 32 && jb + t < p.ldp; ++t)
              arow[jb + t] = reinterpret_cast<const __nv_bfloat16*>(o)[t];
          }
        }
        // shifted copy into the band ring
        const int cbase = kKT * n + 127 - r + 64 * half + 32 * k;
        // the 32-run crosses at most one chunk boundary, at t = split
        const int split = 128 - (cbase & 127);
        const int o0 = ((cbase >> 7) & 3) * (kQT * 128) + (cbase & 127);
        const int o1 = (((cbase >> 7) + 1) & 3) * (kQT * 128) - split;
#pragma unroll
        for (int t = 0; t < 32; ++t)
          myring[(t < split ? o0 : o1) + t] = reinterpret_cast<const __nv_bfloat16*>(o)[t];
      }
      if (n == nt - 1 && half == 1) {
        // band columns after this row's last key (chunk nt)
        const int c1 = kKT * (nt + 1);
        for (int c = kKT * n + 255 - r; c < c1; ++c) myring[((c >> 7) & 3) * (kQT * 128) + (c & 127)] = zb;
      }
      fence_proxy_async_smem();
      named_sync(1, kSoftWarps * 32);
      // band chunk n (and after the last key tile, chunk n + 1) is complete
      // for every row.  Chunks starting at p >= 0 go out as one TMA bulk
      // store; the few starting left of p = 0 (short rows: T - 1 - i0 < 127)
      // are copied by the threads (TMA store boxes need p >= 0).  Chunk m is
      // rewritten by key tile m + 3, after two more barriers: the elected
      // thread's wait for all but the newest store covers that.
      for (int m = n; m <= (n == nt - 1 ? n + 1 : n); ++m) {
        const int c0 = P0 + kKT * m;
        const __nv_bfloat16* chunk = ring + (m & 3) * (kQT * 128);
        if (c0 >= 0) {
          if (warp == 4 && lane == 0) tma_store_3d(&mBD, chunk, c0, i0, hb);
        } else {
          const int tid = threadIdx.x - 128, rr = tid >> 1, cc0 = (tid & 1) * 64;
          if (i0 + rr < p.T) {
            __nv_bfloat16* dst = p.gbd + ((int64_t)hb * p.T + i0 + rr) * p.ldp;
            for (int cc = cc0; cc < cc0 + 64; ++cc) {
              const int64_t pp = (int64_t)c0 + cc;
              if (pp >= 0 && pp < p.ldp) dst[pp] = chunk[rr * 128 + cc];
            }
          }
        }
      }
      if (warp == 4 && lane == 0) bulk_wait_read_1();
    }
    if (lane == 0) tma_store_wait_all();  // dAC tiles (and, warp 4, the dBD chunks) written
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 256);
}

// ---------------------------------------------------------------------------
// Forward with P.V folded in (head dim 64): xl_attn_fwd_kernel<1>, plus per
// pass-2 key step the normalised P tile written once into a 128B-swizzled
// [128 x 64] shared tile -- the A operand of
//     O += P V_step                       128 x 64   (TMEM cols 256..319)
// and the source of P's TMA store -- so the head-dim-wide P.V GEMM over the
// stored P (and the head merge of its output) disappear; O is written
// straight into the merged ctx rows.  Pass 2 keeps one score buffer (TMEM
// cols 0..255) so O fits beside it.
// NS: K + R band stages; NB: P tile / V tile buffers (NB = 2: the softmax
// warps write step u+1's P while O += P V of step u still reads step u's)
template <int NS, int NB>
constexpr int fwd_pv_smem() {
  return 1024 + 2 * 16384 /*Qu, Qv*/ + NS * 32768 /*K + R band stages*/ + NB * 8192 /*V*/ + NB * 16384 /*P tile*/ +
         kSoftWarps * kRingWarp * 4 + 2 * kQT * 2 * 4 /*stats*/ + 256;
}

struct FwdPvParams {
  FwdParams f;
  __nv_bfloat16* ctx;  // merged rows: head h's dh_out columns at h * dh_out, row pitch ld_ctx
  int d;
  int dh_out;          // the model's head dim (<= 64: the operands' pads past it are zero)
  int64_t ld_ctx;
};

template <int NS, int NB>
__global__ void __launch_bounds__(kThreadsFwd, 1)
    xl_attn_fwd_pv_kernel(const __grid_constant__ CUtensorMap mQu, const __grid_constant__ CUtensorMap mQv,
                          const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mR,
                          const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mP,
                          const FwdPvParams pp) {
  const FwdParams& p = pp.f;
  using C = FwdCfg<1>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t* sQu = smem;
  uint8_t* sQv = smem + C::QBytes;
  uint8_t* stages = smem + 2 * C::QBytes;
  uint8_t* sV0 = stages + NS * C::StageBytes;  // 1024-aligned, NB x 8 KB
  uint8_t* sP0 = sV0 + NB * 8192;              // NB x 16 KB
  float* ring = reinterpret_cast<float*>(sP0 + NB * 16384);
  float* stats = ring + kSoftWarps * kRingWarp;  // [half][row][max, sum]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stats + 2 * kQT * 2);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;        // [NS]
  uint64_t* kv_empty = kv_full + NS;   // [NS]
  uint64_t* s_full = kv_empty + NS;    // [2]
  uint64_t* s_empty = s_full + 2;      // [2]
  uint64_t* v_full = s_empty + 2;      // [NB]
  uint64_t* v_empty = v_full + NB;     // [NB]
  uint64_t* p_full = v_empty + NB;     // [NB]
  uint64_t* p_free = p_full + NB;      // [NB]
  uint64_t* o_full = p_free + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int hb, qt;
  cta_tile(p.nqt, p.heavy_first, hb, qt);
  const int h = hb / p.B, b = hb % p.B;
  const int i0 = qt * kQT;
  const int imax = min(i0 + kQT, p.T) - 1;
  const int jt_lo = p.lo / kFKT, jt_hi = min(p.M + imax, p.Kl - 1) / kFKT;
  const int per_pass = jt_hi - jt_lo + 1;
  const int nsteps = 2 * per_pass;
  // buffer of step n: pass 1 alternates 0 / 1, pass 2 always 0.  Use index
  // of that buffer (its mbarrier phase = use & 1):
  auto buf_of = [&](int n) { return n < per_pass ? (n & 1) : 0; };
  auto use_of = [&](int n) {
    if (n < per_pass) return n >> 1;
    return (per_pass + 1) / 2 + (n - per_pass);  // pass 1 used buffer 0 ceil(per_pass / 2) times
  };
  // the last pass-1 use of buffer 1 (its TMEM columns hold O in pass 2)
  const int last_b1 = per_pass >= 2 ? ((per_pass - 2) | 1) : -1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQu);
    tma_prefetch(&mQv);
    tma_prefetch(&mK);
    tma_prefetch(&mR);
    tma_prefetch(&mV);
    tma_prefetch(&mP);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int bb = 0; bb < 2; ++bb) {
      mbar_init(&s_full[bb], 1);
      mbar_init(&s_empty[bb], kSoftWarps * 32);
    }
    for (int bb = 0; bb < NB; ++bb) {
      mbar_init(&v_full[bb], 1);
      mbar_init(&v_empty[bb], 1);
      mbar_init(&p_full[bb], kSoftWarps * 32);
      mbar_init(&p_free[bb], 1);
    }
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t t_o = tmem_base + 256;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_expect_tx(q_full, 2 * C::QBytes);
      tma_atoms<1>(sQu, &mQu, q_full, kQT, i0, hb);
      tma_atoms<1>(sQv, &mQv, q_full, kQT, i0, hb);
      int s = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nsteps; ++n) {
        mbar_wait(&kv_empty[s], ph ^ 1);
        const int j0 = (jt_lo + n % per_pass) * kFKT;
        uint8_t* sk = stages + s * C::StageBytes;
        mbar_expect_tx(&kv_full[s], C::StageBytes);
        tma_atoms<1>(sk, &mK, &kv_full[s], kFKT, j0, hb);
        tma_atoms<1>(sk + C::KBytes, &mR, &kv_full[s], kFBand, p.T - kQT - i0 + j0, h);
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
        if (n >= per_pass) {
          const int u = n - per_pass;  // V of pass-2 step u, MN-major B of O += P V
          const int vb = u % NB;
          mbar_wait(&v_empty[vb], ((u / NB) & 1) ^ 1);
          mbar_expect_tx(&v_full[vb], 8192);
          tma_load_3d(sV0 + vb * 8192, &mV, &v_full[vb], 0, j0, hb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t id_ac = umma_idesc(false, false, false, kQT, kFKT);
      const uint32_t id_bd = umma_idesc(false, false, false, kQT, kFBand);
      const uint32_t id_pv = umma_idesc(false, false, true, kQT, 64);
      const uint32_t qa = smem_u32(sQu), qb = smem_u32(sQv), pa0 = smem_u32(sP0), va0 = smem_u32(sV0);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int u) {
        const int pb = u % NB;
        const uint32_t pa = pa0 + pb * 16384, va = va0 + pb * 8192;
        mbar_wait(&p_full[pb], (u / NB) & 1);
        mbar_wait(&v_full[pb], (u / NB) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(t_o, umma_desc(pa + 32 * k, 16, 1024), umma_desc(va + k * 2048, 8192, 1024), id_pv,
                        (u | k) != 0);
        tc_commit(&p_free[pb]);
        tc_commit(&v_empty[pb]);
      };
      int s = 0;
      uint32_t ph = 0;
      for (int n = 0; n < nsteps; ++n) {
        const int buf = buf_of(n);
        mbar_wait(&s_empty[buf], (use_of(n) & 1) ^ 1);
        mbar_wait(&kv_full[s], ph);
        tc_fence_after();
        const uint32_t kb = smem_u32(stages + s * C::StageBytes), rb = kb + C::KBytes;
        const uint32_t d = tmem_base + buf * kFBuf;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(d, atom_desc<1>(qa, kQT, k), atom_desc<1>(kb, kFKT, k), id_ac, k > 0);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(d + kFKT, atom_desc<1>(qb, kQT, k), atom_desc<1>(rb, kFBand, k), id_bd, k > 0);
        tc_commit(&kv_empty[s]);
        tc_commit(&s_full[buf]);
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
        if (n == per_pass && last_b1 >= 0) {
          // O's columns were pass-1 buffer 1: drained by the softmax warps?
          mbar_wait(&s_empty[1], use_of(last_b1) & 1);
        }
        if (n > per_pass) issue_pv(n - per_pass - 1);
      }
      issue_pv(per_pass - 1);
      tc_commit(o_full);
    }
  } else if (warp >= 4) {
    // ---------------- softmax: row r = 32 q + lane, key columns [32 half, +32) of each step ----------------
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const int i = i0 + r;
    const bool row_ok = i < p.T;
    const int jhi = p.M + i;
    float* myring = ring + (warp - 4) * kRingWarp + lane * kRing;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    const int cb0 = 96 - 32 * q + 32 * half;
    const int off = 31 - lane;
    __nv_bfloat16* prow = p.p + ((int64_t)hb * p.T + i) * p.ldp;
    const int rsw = r & 7;
    float m = -INFINITY, l = 0.f, inv = 0.f;
    for (int n = 0; n < nsteps; ++n) {
      const bool pass2 = n >= per_pass;
      if (n == per_pass) {
        stats[(half * kQT + r) * 2] = m;
        stats[(half * kQT + r) * 2 + 1] = l;
        named_sync(1, kSoftWarps * 32);
        const float mo = stats[((1 - half) * kQT + r) * 2], lo_ = stats[((1 - half) * kQT + r) * 2 + 1];
        const float mm = fmaxf(m, mo);
        const float ll = (m == -INFINITY ? 0.f : l * ex2(m - mm)) + (mo == -INFINITY ? 0.f : lo_ * ex2(mo - mm));
        m = mm;
        inv = ll > 0.f ? 1.f / ll : 0.f;
        if (row_ok) {
          const uint4 z = make_uint4(0, 0, 0, 0);
          const int64_t a0 = half ? (int64_t)(jt_hi + 1) * kFKT : 0;
          const int64_t a1 = half ? p.ldp : (int64_t)jt_lo * kFKT;
          for (int64_t c = a0; c < a1; c += 8) *reinterpret_cast<uint4*>(prow + c) = z;
        }
      }
      const int buf = buf_of(n);
      const int jb = (jt_lo + n % per_pass) * kFKT + 32 * half;
      mbar_wait(&s_full[buf], use_of(n) & 1);
      tc_fence_after();
      const uint32_t tb = tl + buf * kFBuf;
      uint32_t v0[32], v1[32], a[32];
      tmem_ld32_async(tb + kFKT + cb0, v0);
      tmem_ld32_async(tb + kFKT + cb0 + 32, v1);
      tmem_ld32_async(tb + 32 * half, a);
      tmem_wait_ld(v0);
      tmem_wait_ld(v1);
      tmem_wait_ld(a);
      tc_fence_before();
      mbar_arrive(&s_empty[buf]);
      stage_band(myring, 0, v0, lane);
      stage_band(myring, 1, v1, lane);
      __syncwarp();
      float sv[32];
      float cm = -INFINITY;
      if (jb >= p.lo && jb + 31 <= p.M + i0 + 32 * q) {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          sv[t] = (__uint_as_float(a[t]) + myring[off + t]) * p.c2;
          cm = fmaxf(cm, sv[t]);
        }
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int j = jb + t;
          const float x = (__uint_as_float(a[t]) + myring[off + t]) * p.c2;
          sv[t] = (j >= p.lo && j <= jhi) ? x : -INFINITY;
          cm = fmaxf(cm, sv[t]);
        }
      }
      __syncwarp();
      if (!pass2) {
        const float mn = fmaxf(m, cm);
        if (mn != -INFINITY) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int t = 0; t < 32; ++t) acc[t & 3] += ex2(sv[t] - mn);
          l = (m == -INFINITY ? 0.f : l * ex2(m - mn)) + ((acc[0] + acc[1]) + (acc[2] + acc[3]));
          m = mn;
        }
      } else {
        const int u = n - per_pass;
        uint32_t w[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(ex2(sv[2 * t] - m) * inv, ex2(sv[2 * t + 1] - m) * inv);
          w[t] = row_ok ? *reinterpret_cast<uint32_t*>(&b2) : 0u;
        }
        // P tile buffer u % NB is free once O += P V of step u - NB and this
        // quarter's TMA store of it have read it
        const int pb = u % NB;
        uint8_t* sPb = sP0 + pb * 16384;
        if (u >= NB) mbar_wait(&p_free[pb], ((u / NB) - 1) & 1);
        if (half == 0 && lane == 0) {
          if constexpr (NB == 1) tma_store_wait_read();
          else bulk_wait_read_1();  // the newest store reads the other buffer
        }
        named_sync(2 + q, 64);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(sPb + r * 128 + (((4 * half + c) ^ rsw) << 4)) =
              make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        fence_proxy_async_smem();
        mbar_arrive(&p_full[pb]);
        named_sync(2 + q, 64);
        // this quarter's 32 rows x 64 keys of P (the map clips rows past T and columns past ldp)
        const int j0 = jb - 32 * half;
        if (half == 0 && lane == 0 && j0 < p.ldp && i0 + 32 * q < p.T)
          tma_store_3d_p(&mP, sPb + 32 * q * 128, j0, i0 + 32 * q, hb);
      }
    }
    // ---- O = P V: rows of this lane quarter, head columns [32 half, +32) -> merged ctx
    mbar_wait(o_full, 0);
    tc_fence_after();
    uint32_t o[32];
    tmem_ld32(tl + 256 + 32 * half, o);
    if (row_ok && pp.dh_out == 64 && pp.ld_ctx % 8 == 0) {
      uint4* dst = reinterpret_cast<uint4*>(pp.ctx + ((int64_t)b * p.T + i) * pp.ld_ctx + h * 64 + 32 * half);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t ww[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2 * e]), __uint_as_float(o[8 * c + 2 * e + 1]));
          ww[e] = *reinterpret_cast<uint32_t*>(&b2);
        }
        dst[c] = make_uint4(ww[0], ww[1], ww[2], ww[3]);
      }
    } else if (row_ok) {  // a head dim padded to 64: its real columns, at the merged rows' pitch
      __nv_bfloat16* dst = pp.ctx + ((int64_t)b * p.T + i) * pp.ld_ctx + (int64_t)h * pp.dh_out;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int col = 32 * half + c;
        if (col < pp.dh_out) dst[col] = __float2bfloat16_rn(__uint_as_float(o[c]));
      }
    }
    if (half == 0 && lane == 0) tma_store_wait_all();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// ---------------------------------------------------------------------------
// Backward with the query gradients fused (head dim 64, T % 128 == 0): the
// kernel above, plus per key tile n
//     dQu += dS_n K_n                   128 x 64    (TMEM cols 256..319)
//     dQv += dBDband_c R_c  (c = n)     128 x 64    (TMEM cols 320..383)
// on the tensor cores.  dS_n is written once into a 128B-swizzled [128 x 128]
// shared tile -- the A operand of dQu and the source of the dAC TMA stores --
// and, shifted, into a 3-chunk ring in band coordinates whose chunk n (complete
// after key tile n) is the A operand of dQv against the 128 relative-encoding
// rows it covers and the source of the dBD TMA stores.  This removes the two
// head-dim-wide GEMMs dQu = dAC K and dQv = dBD R that re-read the 185 MB
// dAC / dBD matrices per block at the C3 shape.
constexpr int kRing3 = 3;
constexpr int kChunkBytes = 128 * 128 * 2;  // 128 rows x 128 band columns, two SW128 atoms
// P tiles arrive by TMA (two 128B-swizzled 64-key atoms) one tile ahead of
// the softmax warps: the per-thread P row loads of xl_attn_bwd_kernel were
// the kernel's dominant stall (ncu: long-scoreboard on the bf16 unpack)
constexpr int kDqSmem = 1024 + 16384 /*G*/ + 16384 /*V*/ + 16384 /*K*/ + 16384 /*R*/ + kChunkBytes /*P*/ +
                        kRing3 * kChunkBytes + kChunkBytes /*dS tile*/ + 256 /*barriers*/;

// byte offset of (row r, column c) in a [128 x 128] bf16 tile of two 128B-swizzled 64-column atoms
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  return (uint32_t)((c >> 6) * (128 * 128) + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + ((c & 7) << 1));
}

struct DqParams {
  BwdParams b;
  float* gqu;  // [H*B*T, 64] fp32 (rows hb*T + i)
  float* gqv;
  int d_in_kernel;      // persistent kernel: warps 2-3 compute the D rows (no separate D pass)
  __nv_bfloat16* gqkv;  // optional (persistent kernel): bf16(dQu + dQv) straight into the merged g_qkv rows
                        // [B*M memory rows; B*T current rows] x 3d, query columns (xl_merge_grads' arithmetic)
  float* bias_part;  // optional [2][B*nqt][H*64]: per-CTA column sums of dQu (u) and dQv (v) -- a
                     // [rows, cols] block per bias that a column-sum finish reduces
  float* d_rows;     // optional [HB*T]: D_i = dO_i . O_i for xl_attn_bwd_kv
  int no_dac;        // dAC is not written (xl_attn_bwd_kv computes dK from dS itself)
  unsigned long long* trace;  // RP_XL_DQ_TRACE=<cta>: that CTA's event times (diagnostics)
  int trace_cta;
  int zero_rows;              // margins zeroed by the softmax warps, a row per thread: with dAC (twice the
                              // margins; two warps are then the tail), or RP_XL_DQ_ZERO_ROWS=1 (A/B)
};

// out[lane] = sum over the warp's 32 rows of column `lane` of v[0..31]
// (butterfly transpose-reduce: 31 shuffles; a fixed summation tree)
__device__ __forceinline__ float warp_colsum32(float (&a)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = lane & s;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const float send = upper ? a[k] : a[k + s];
      const float keep = upper ? a[k + s] : a[k];
      a[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return a[0];
}

// (the traced CTA comes as a kernel parameter: a global load in the probe
// itself stalled the producer thread for microseconds and faked TMA stalls)
__device__ __forceinline__ void dq_trace(unsigned long long* tr, int ev, int idx, int cta) {
  if (tr && (int)blockIdx.x == cta && idx < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[ev * 32 + idx] = t;
  }
}

__global__ void __launch_bounds__(kThreadsBwd, 1)
    xl_attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap mG, const __grid_constant__ CUtensorMap mV,
                          const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mR,
                          const __grid_constant__ CUtensorMap mBD, const __grid_constant__ CUtensorMap mAC,
                          const __grid_constant__ CUtensorMap mP, const DqParams dq) {
  const BwdParams& p = dq.b;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t* sG = smem;
  uint8_t* sV = smem + 16384;
  uint8_t* sK = smem + 2 * 16384;
  uint8_t* sR = smem + 3 * 16384;
  uint8_t* sP = smem + 4 * 16384;
  uint8_t* ring = sP + kChunkBytes;
  uint8_t* sA = ring + kRing3 * kChunkBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + kChunkBytes);
  uint64_t* g_full = bars;
  uint64_t* v_full = bars + 1;
  uint64_t* v_empty = bars + 2;
  uint64_t* p_full = bars + 17;   // [2]
  uint64_t* p_empty = bars + 19;  // [2]: the dQu MMA has read the tile's dS (written over its P)
  uint64_t* acc_full = bars + 5;   // [2]
  uint64_t* acc_empty = bars + 7;  // [2]
  uint64_t* kr_full = bars + 9;
  uint64_t* kr_empty = bars + 10;
  uint64_t* ds_ready = bars + 11;
  uint64_t* ring_free = bars + 13;  // [3]
  uint64_t* dq_full = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);
  // P tile n in buffer n & 1 (the former dS tile is the second buffer): each
  // thread writes its dS over the P values it read, and the dQu MMA reads it
  // there -- no dS tile, so a tile's dS stores no longer wait for the
  // previous tile's dQu MMA
  auto pbuf = [&](int n) -> uint8_t* { return (n & 1) ? sA : sP; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) dq_trace(dq.trace, 0, 0, dq.trace_cta);
  int hb, qt;
  cta_tile(p.nqt, p.heavy_first, hb, qt);
  const int h = hb / p.B, b = hb % p.B;
  const int i0 = qt * kQT;
  const int imax = min(i0 + kQT, p.T) - 1;
  const int jt_lo = p.lo / kKT, jt_hi = min(p.M + imax, p.Kl - 1) / kKT;
  const int nt = jt_hi - jt_lo + 1;
  const int P0 = p.T - kQT - i0 + jt_lo * kKT;  // band column 0 in dBD / R-row coordinates (>= 0: T % 128 == 0)

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mG);
    tma_prefetch(&mV);
    tma_prefetch(&mK);
    tma_prefetch(&mR);
    tma_prefetch(&mBD);
    tma_prefetch(&mAC);
    tma_prefetch(&mP);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(g_full, 1);
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kSoftWarps * 32);
    }
    mbar_init(kr_full, 1);
    mbar_init(kr_empty, 1);
    mbar_init(ds_ready, 1);
    for (int c = 0; c < kRing3; ++c) mbar_init(&ring_free[c], 1);
    mbar_init(dq_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t t_dqu = tmem_base + 256, t_dqv = tmem_base + 320;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_expect_tx(g_full, 16384);
      tma_atoms<1>(sG, &mG, g_full, kQT, i0, hb);
      for (int n = 0; n <= nt; ++n) {
        if (n < nt) {
          mbar_wait(v_empty, (n & 1) ^ 1);
          mbar_expect_tx(v_full, 16384);
          tma_atoms<1>(sV, &mV, v_full, kKT, (jt_lo + n) * kKT, hb);
          const int pb = n & 1;
          mbar_wait(&p_empty[pb], ((n >> 1) & 1) ^ 1);
          dq_trace(dq.trace, 1, n, dq.trace_cta);
          mbar_expect_tx(&p_full[pb], kChunkBytes);
          tma_load_3d(pbuf(n), &mP, &p_full[pb], (jt_lo + n) * kKT, i0, hb);
          tma_load_3d(pbuf(n) + 128 * 128, &mP, &p_full[pb], (jt_lo + n) * kKT + 64, i0, hb);
        }
        // K tile n (MN-major B of dQu) and relative-encoding rows of band chunk n
        // (MN-major B of dQv); after the last tile only the rows of chunk nt
        mbar_wait(kr_empty, (n & 1) ^ 1);
        mbar_expect_tx(kr_full, n < nt ? 32768 : 16384);
        if (n < nt) tma_load_3d(sK, &mK, kr_full, 0, (jt_lo + n) * kKT, hb);
        tma_load_3d(sR, &mR, kr_full, 0, P0 + kKT * n, h);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t id_dp = umma_idesc(false, false, false, kQT, kKT);
      const uint32_t id_dq = umma_idesc(false, false, true, kQT, 64);
      const uint32_t ga = smem_u32(sG), ka = smem_u32(sK), ra = smem_u32(sR);
      const uint32_t rg = smem_u32(ring);
      mbar_wait(g_full, 0);
      auto issue_dq = [&](int n) {
        mbar_wait(ds_ready, n & 1);
        dq_trace(dq.trace, 2, n, dq.trace_cta);
        mbar_wait(kr_full, n & 1);
        tc_fence_after();
        const uint32_t ch = rg + (uint32_t)((n % kRing3) * kChunkBytes), aa = smem_u32(pbuf(n));
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc_mma<false>(t_dqu, atom_desc<1>(aa, kQT, k), umma_desc(ka + k * 2048, 16384, 1024), id_dq, (n | k) != 0);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc_mma<false>(t_dqv, atom_desc<1>(ch, kQT, k), umma_desc(ra + k * 2048, 16384, 1024), id_dq, (n | k) != 0);
        tc_commit(&p_empty[n & 1]);
        tc_commit(&ring_free[n % kRing3]);
        tc_commit(kr_empty);
      };
      for (int n = 0; n < nt; ++n) {
        const int s = n & 1;
        mbar_wait(&acc_empty[s], ((n >> 1) & 1) ^ 1);
        mbar_wait(v_full, n & 1);
        dq_trace(dq.trace, 3, n, dq.trace_cta);
        tc_fence_after();
        const uint32_t vb = smem_u32(sV);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma<false>(tmem_base + s * kKT, atom_desc<1>(ga, kQT, k), atom_desc<1>(vb, kKT, k), id_dp, k > 0);
        tc_commit(v_empty);
        tc_commit(&acc_full[s]);
        if (n >= 1) issue_dq(n - 1);
      }
      issue_dq(nt - 1);
      // band chunk nt (the columns right of the last key tile) is complete with tile nt-1
      mbar_wait(kr_full, nt & 1);
      tc_fence_after();
      const uint32_t ch = rg + (uint32_t)((nt % kRing3) * kChunkBytes);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc_mma<false>(t_dqv, atom_desc<1>(ch, kQT, k), umma_desc(ra + k * 2048, 16384, 1024), id_dq, 1u);
      tc_commit(dq_full);
    }
  } else if (warp >= 4) {
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const int i = i0 + r;
    const int jhi = p.M + i;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    const int64_t rowoff = ((int64_t)hb * p.T + i) * p.ldp;
    const __nv_bfloat16* prow = p.p + rowoff;
    __nv_bfloat16* arow = p.gac + rowoff;
    __nv_bfloat16* brow = p.gbd + rowoff;
    // D_i = g_ctx_i . ctx_i over this head's 64 columns
    float D = 0.f;
    {
      const int64_t mo = ((int64_t)b * p.T + i) * p.d + h * 64;
      const uint4* g4 = reinterpret_cast<const uint4*>(p.gctx + mo);
      const uint4* c4 = reinterpret_cast<const uint4*>(p.ctx + mo);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 gu = g4[c], cu = c4[c];
        const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w}, cw[4] = {cu.x, cu.y, cu.z, cu.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[e]));
          const float2 cf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cw[e]));
          D = fmaf(gf.x, cf.x, D);
          D = fmaf(gf.y, cf.y, D);
        }
      }
      if (dq.d_rows && half == 0) dq.d_rows[(int64_t)hb * p.T + i] = D;
      if (dq.zero_rows) {
        if (half == 0) {
          if (!dq.no_dac) zero_row(arow, 0, (int64_t)jt_lo * kKT);
          zero_row(brow, 0, lmin(lmax(P0, 0), p.ldp));
        } else {
          if (!dq.no_dac) zero_row(arow, lmin((int64_t)(jt_hi + 1) * kKT, p.ldp), p.ldp);
          zero_row(brow, lmin(lmax((int64_t)P0 + kKT * (nt + 1), 0), p.ldp), p.ldp);
        }
      }
    }
    if (r == 0 && half == 0) dq_trace(dq.trace, 4, 0, dq.trace_cta);  // prologue (D, zero margins) done
    auto ring_at = [&](int bc) -> __nv_bfloat16* {  // band column bc of row r
      return reinterpret_cast<__nv_bfloat16*>(ring + (bc >> 7) % kRing3 * kChunkBytes + sw128_off(r, bc & 127));
    };
    const __nv_bfloat16 zb = __float2bfloat16_rn(0.f);
    auto zero_ring = [&](int c0, int c1) {  // band columns [c0, c1) of row r: 16-byte chunks inside
      int c = c0;
      for (; c < c1 && (c & 7); ++c) *ring_at(c) = zb;
      for (; c + 8 <= c1; c += 8) *reinterpret_cast<uint4*>(ring_at(c)) = make_uint4(0u, 0u, 0u, 0u);
      for (; c < c1; ++c) *ring_at(c) = zb;
    };
    // band columns before this row's first key (chunk 0)
    if (half == 0) zero_ring(0, 127 - r);
    for (int n = 0; n < nt; ++n) {
      const int s = n & 1;
      const int jt0 = (jt_lo + n) * kKT + 64 * half;
      // this row's 64 P values of the tile from the swizzled smem tile (zero past ldp: TMA fill)
      uint4 pr[2][4];
      mbar_wait(&p_full[n & 1], (n >> 1) & 1);
      if (r == 0 && half == 0) dq_trace(dq.trace, 5, n, dq.trace_cta);
      uint8_t* const tile = pbuf(n);
      {
        const uint8_t* prow_s = tile + half * (128 * 128) + r * 128;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            pr[k][c] = *reinterpret_cast<const uint4*>(prow_s + (((4 * k + c) ^ (r & 7)) << 4));
      }
      mbar_wait(&acc_full[s], (n >> 1) & 1);
      tc_fence_after();
      uint32_t dp[2][32];
      tmem_ld32(tl + s * kKT + 64 * half, dp[0]);
      tmem_ld32(tl + s * kKT + 64 * half + 32, dp[1]);
      tc_fence_before();
      mbar_arrive(&acc_empty[s]);
      if (r == 0 && half == 0) dq_trace(dq.trace, 6, n, dq.trace_cta);
      // dS goes over this thread's own P values (no wait); the upper band
      // chunk of this tile is reused from tile n - 2, whose dQv MMA must be
      // done (its TMA store was retired before barrier n - 1)
      if (n >= 2) mbar_wait(&ring_free[(n + 1) % kRing3], ((n - 2) / kRing3) & 1);
      if (r == 0 && half == 0) dq_trace(dq.trace, 7, n, dq.trace_cta);
      if (lane == 0) tma_store_wait_read();
      __syncwarp();
      const int rsw = r & 7;
      uint8_t* arow_s = tile + half * (128 * 128) + r * 128;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int jb = jt0 + 32 * k;
        uint32_t o[16];
        // P is zero outside the window, but dP there is not: mask explicitly
        // (runs wholly inside the window -- all but the diagonal and memory
        // edge tiles -- skip the per-element test)
        const bool inside = jb >= p.lo && jb + 31 <= jhi;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t w[4] = {pr[k][c].x, pr[k][c].y, pr[k][c].z, pr[k][c].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 pf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
            const int t = 8 * c + 2 * e;
            const int j = jb + t;
            float a0 = pf.x * (__uint_as_float(dp[k][t]) - D) * p.scale;
            float a1 = pf.y * (__uint_as_float(dp[k][t + 1]) - D) * p.scale;
            if (!inside) {
              a0 = (j >= p.lo && j <= jhi) ? a0 : 0.f;
              a1 = (j + 1 >= p.lo && j + 1 <= jhi) ? a1 : 0.f;
            }
            __nv_bfloat162 b2 = __floats2bfloat162_rn(a0, a1);
            o[t >> 1] = *reinterpret_cast<uint32_t*>(&b2);
          }
        }
        // dS row segment into the swizzled tile (16-byte chunks 4k .. 4k+3 of this half's atom)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(arow_s + (((4 * k + c) ^ rsw) << 4)) =
              make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        // shifted copy into the band ring: the 32-run crosses at most one
        // 64-column atom boundary -- two segments of constant (chunk, atom)
        const int cb = kKT * n + 127 - r + 64 * half + 32 * k;
        const int split = 64 - (cb & 63);
        uint8_t* seg0 = ring + ((cb >> 7) % kRing3) * kChunkBytes + ((cb >> 6) & 1) * (128 * 128) + r * 128;
        const int c1 = cb + split;
        uint8_t* seg1 = ring + ((c1 >> 7) % kRing3) * kChunkBytes + ((c1 >> 6) & 1) * (128 * 128) + r * 128;
        const int e0 = cb & 63;
        // run element t of this row in the ring (a 4-byte aligned pair never
        // straddles the 64-column atom boundary: both start parities keep
        // the pairs inside one atom)
        auto at = [&](int t) -> uint8_t* {
          const bool lo = t < split;
          const int e = lo ? e0 + t : t - split;
          return (lo ? seg0 : seg1) + ((((e >> 3) ^ rsw) << 4) | ((e & 7) << 1));
        };
        if ((cb & 1) == 0) {  // pairs land on 4-byte words: 16 word stores
#pragma unroll
          for (int m = 0; m < 16; ++m) *reinterpret_cast<uint32_t*>(at(2 * m)) = o[m];
        } else {  // shifted by one element: an edge half-word each side, 15 re-paired words
          *reinterpret_cast<unsigned short*>(at(0)) = (unsigned short)(o[0] & 0xffffu);
#pragma unroll
          for (int m = 0; m < 15; ++m) *reinterpret_cast<uint32_t*>(at(2 * m + 1)) = __byte_perm(o[m], o[m + 1], 0x5432);
          *reinterpret_cast<unsigned short*>(at(31)) = (unsigned short)(o[15] >> 16);
        }
      }
      if (n == nt - 1 && half == 1) zero_ring(kKT * n + 255 - r, kKT * (nt + 1));  // after this row's last key
      fence_proxy_async_smem();
      __syncwarp();
      // this warp's 32 x 64 dAC block straight from the swizzled dS tile
      if (!dq.no_dac && lane == 0 && jt0 < p.ldp) {
        tma_store_3d(&mAC, tile + half * (128 * 128) + 32 * q * 128, jt0, i0 + 32 * q, hb);
        // the tile is reloaded (P of tile n + 2) once the dQu MMA released it:
        // this store must have read it before ds_ready
        tma_store_wait_read();
      }
      // earlier dBD chunk stores have read the ring (all but the newest bulk
      // group: this tile's dAC store, which nobody waits for here)
      if (warp == 4 && lane == 0) bulk_wait_read_1();
      if (r == 0 && half == 0) dq_trace(dq.trace, 8, n, dq.trace_cta);
      named_sync(1, kSoftWarps * 32);
      if (warp == 4 && lane == 0) {
        dq_trace(dq.trace, 9, n, dq.trace_cta);
        mbar_arrive(ds_ready);
        for (int m = n; m <= (n == nt - 1 ? n + 1 : n); ++m) {
          const uint8_t* ch = ring + (m % kRing3) * kChunkBytes;
          const int c0 = P0 + kKT * m;
          if (c0 < p.ldp) tma_store_3d(&mBD, ch, c0, i0, hb);
          if (c0 + 64 < p.ldp) tma_store_3d(&mBD, ch + 128 * 128, c0 + 64, i0, hb);
        }
      }
    }
    // ---- dQu / dQv epilogue: rows of this lane quarter, columns [32 half, +32)
    if (r == 0 && half == 0) dq_trace(dq.trace, 10, 0, dq.trace_cta);
    mbar_wait(dq_full, 0);
    if (r == 0 && half == 0) dq_trace(dq.trace, 10, 1, dq.trace_cta);
    tc_fence_after();
    uint32_t v[32];
    const int64_t orow = ((int64_t)hb * p.T + i) * 64 + 32 * half;
    tmem_ld32(tl + 256 + 32 * half, v);
    float4* du = reinterpret_cast<float4*>(dq.gqu + orow);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      du[c] = make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]), __uint_as_float(v[4 * c + 2]),
                          __uint_as_float(v[4 * c + 3]));
    float colsum_u = 0.f, colsum_v = 0.f;
    if (dq.bias_part) {  // rows past T are zero in TMEM (their dS is zero)
      float a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = __uint_as_float(v[c]);
      colsum_u = warp_colsum32(a, lane);
    }
    tmem_ld32(tl + 320 + 32 * half, v);
    float4* dv = reinterpret_cast<float4*>(dq.gqv + orow);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      dv[c] = make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]), __uint_as_float(v[4 * c + 2]),
                          __uint_as_float(v[4 * c + 3]));
    if (dq.bias_part) {
      float a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = __uint_as_float(v[c]);
      colsum_v = warp_colsum32(a, lane);
      // the four lane-quarter warps of this column half, summed in quarter
      // order through the (now idle) dO tile
      float* red = reinterpret_cast<float*>(sG);
      red[((half * 2 + 0) * 4 + q) * 32 + lane] = colsum_u;
      red[((half * 2 + 1) * 4 + q) * 32 + lane] = colsum_v;
      named_sync(1, kSoftWarps * 32);
      if (q == 0) {
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const float* rr = red + (half * 2 + w) * 4 * 32 + lane;
          const float s = ((rr[0] + rr[32]) + rr[64]) + rr[96];
          const int hh = hb / p.B, bb = hb - hh * p.B;
          dq.bias_part[(((int64_t)w * p.B + bb) * p.nqt + qt) * p.H * 64 + hh * 64 + 32 * half + lane] = s;
        }
      }
    }
    if (lane == 0) tma_store_wait_all();
  } else if (!dq.zero_rows) {
    // warps 2 and 3 (otherwise idle): the columns outside the key tiles this
    // query tile sees (dAC = 0) and the dBD margins outside the stored band
    // chunks, as coalesced 16-byte stores (all bounds are multiples of 128
    // columns: T % 128 == 0) -- in the softmax warps, one row per thread,
    // these stores held the prologue up for several microseconds
    const int64_t bl = lmin(lmax(P0, 0), p.ldp), br = lmin(lmax((int64_t)P0 + kKT * (nt + 1), 0), p.ldp);
    const int64_t al = lmin((int64_t)jt_lo * kKT, p.ldp), ar = lmin((int64_t)(jt_hi + 1) * kKT, p.ldp);
    auto zero = [&](__nv_bfloat16* row, int64_t a, int64_t e) {
      for (int64_t c = a + 8 * lane; c < e; c += 256) *reinterpret_cast<uint4*>(row + c) = make_uint4(0u, 0u, 0u, 0u);
    };
    for (int rr = warp - 2; rr < kQT; rr += 2) {
      const int64_t rowoff = ((int64_t)hb * p.T + i0 + rr) * p.ldp;
      zero(p.gbd + rowoff, 0, bl);
      zero(p.gbd + rowoff, br, p.ldp);
      if (!dq.no_dac) {
        zero(p.gac + rowoff, 0, al);
        zero(p.gac + rowoff, ar, p.ldp);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) dq_trace(dq.trace, 10, 2, dq.trace_cta);
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

// Persistent form of xl_attn_bwd_dq for the production path (no dAC; D rows
// from xl_d_rows): one CTA per SM walks the (head*batch, query tile) items in
// the heavy-first order, with the TMA / MMA / softmax pipelines running on
// across items.  The per-CTA overhead of the one-item kernel -- ~5 us from
// CTA start to the first tile (first TMA on each descriptor, D-row loads under
// full-GPU traffic) and ~4-6 us of epilogue -- was a third of each ~30 us CTA
// (RP_XL_DQ_TRACE); here the producer fetches the next item's dO / v / P
// tiles while the softmax warps finish the current item.  The arithmetic and
// every store are those of xl_attn_bwd_dq_kernel (bitwise equal outputs).
__global__ void d_rows_kernel(const __nv_bfloat16* __restrict__ gctx, const __nv_bfloat16* __restrict__ ctx,
                              float* __restrict__ d_rows, int B, int T, int H, int d) {
  // D[(h*B + b)*T + i] = g_ctx[b*T + i, h*64 : +64] . ctx[same], in bwd_dq's order
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)H * B * T) return;
  const int hb = (int)(idx / T), i = (int)(idx - (int64_t)hb * T), h = hb / B, b = hb - h * B;
  const int64_t mo = ((int64_t)b * T + i) * d + h * 64;
  const uint4* g4 = reinterpret_cast<const uint4*>(gctx + mo);
  const uint4* c4 = reinterpret_cast<const uint4*>(ctx + mo);
  float D = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 gu = g4[c], cu = c4[c];
    const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w}, cw[4] = {cu.x, cu.y, cu.z, cu.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[e]));
      const float2 cf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cw[e]));
      D = fmaf(gf.x, cf.x, D);
      D = fmaf(gf.y, cf.y, D);
    }
  }
  d_rows[idx] = D;
}

struct DqItem {
  int hb, qt, h, b, i0, jt_lo, jt_hi, nt, P0;
};

__device__ __forceinline__ DqItem dq_item(const BwdParams& p, int it) {
  DqItem w;
  const int nhb = p.H * p.B;
  w.qt = p.heavy_first ? p.nqt - 1 - it / nhb : it % p.nqt;
  w.hb = p.heavy_first ? it % nhb : it / p.nqt;
  w.h = w.hb / p.B;
  w.b = w.hb % p.B;
  w.i0 = w.qt * kQT;
  const int imax = min(w.i0 + kQT, p.T) - 1;
  w.jt_lo = p.lo / kKT;
  w.jt_hi = min(p.M + imax, p.Kl - 1) / kKT;
  w.nt = w.jt_hi - w.jt_lo + 1;
  w.P0 = p.T - kQT - w.i0 + w.jt_lo * kKT;
  return w;
}

__global__ void __launch_bounds__(kThreadsBwd, 1)
    xl_attn_bwd_dq_persist_kernel(const __grid_constant__ CUtensorMap mG, const __grid_constant__ CUtensorMap mV,
                                  const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mR,
                                  const __grid_constant__ CUtensorMap mBD, const __grid_constant__ CUtensorMap mP,
                                  const DqParams dq) {
  const BwdParams& p = dq.b;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sG = smem;
  uint8_t* sV = smem + 16384;
  uint8_t* sK = smem + 2 * 16384;
  uint8_t* sR = smem + 3 * 16384;
  uint8_t* sP = smem + 4 * 16384;
  uint8_t* ring = sP + kChunkBytes;
  uint8_t* sA = ring + kRing3 * kChunkBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + kChunkBytes);
  uint64_t* g_full = bars;
  uint64_t* g_empty = bars + 1;
  uint64_t* v_full = bars + 2;
  uint64_t* v_empty = bars + 3;
  uint64_t* acc_full = bars + 4;   // [2]
  uint64_t* acc_empty = bars + 6;  // [2]
  uint64_t* kr_full = bars + 8;
  uint64_t* kr_empty = bars + 9;
  uint64_t* ds_ready = bars + 10;
  uint64_t* ring_free = bars + 11;  // [3]
  uint64_t* dq_full = bars + 14;
  uint64_t* dq_empty = bars + 15;
  uint64_t* p_full = bars + 16;   // [2]
  uint64_t* p_empty = bars + 18;  // [2]
  uint64_t* d_ready = bars + 20;  // [2]: an item's D rows written (warps 2-3)
  uint64_t* d_taken = bars + 22;  // [2]: and read by the softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  auto pbuf = [&](int g) -> uint8_t* { return (g & 1) ? sA : sP; };
  const int n_items = p.H * p.B * p.nqt;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mG);
    tma_prefetch(&mV);
    tma_prefetch(&mK);
    tma_prefetch(&mR);
    tma_prefetch(&mBD);
    tma_prefetch(&mP);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(g_full, 1);
    mbar_init(g_empty, 1);
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kSoftWarps * 32);
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], 1);
    }
    mbar_init(kr_full, 1);
    mbar_init(kr_empty, 1);
    mbar_init(ds_ready, 1);
    for (int c = 0; c < kRing3; ++c) mbar_init(&ring_free[c], 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, kSoftWarps * 32);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&d_ready[s], 64);
      mbar_init(&d_taken[s], kSoftWarps * 32);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t t_dqu = tmem_base + 256, t_dqv = tmem_base + 320;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (runs ahead across items) ----------------
      int gt = 0, gk = 0, gv = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        const DqItem w = dq_item(p, it);
        mbar_wait(g_empty, (li & 1) ^ 1);  // the previous item's last dP has read dO
        mbar_expect_tx(g_full, 16384);
        tma_atoms<1>(sG, &mG, g_full, kQT, w.i0, w.hb);
        for (int n = 0; n <= w.nt; ++n) {
          if (n < w.nt) {
            mbar_wait(v_empty, (gv & 1) ^ 1);
            mbar_expect_tx(v_full, 16384);
            tma_atoms<1>(sV, &mV, v_full, kKT, (w.jt_lo + n) * kKT, w.hb);
            ++gv;
            const int pb = gt & 1;
            mbar_wait(&p_empty[pb], ((gt >> 1) & 1) ^ 1);
            dq_trace(dq.trace, 1, gt, dq.trace_cta);
            mbar_expect_tx(&p_full[pb], kChunkBytes);
            tma_load_3d(pbuf(gt), &mP, &p_full[pb], (w.jt_lo + n) * kKT, w.i0, w.hb);
            tma_load_3d(pbuf(gt) + 128 * 128, &mP, &p_full[pb], (w.jt_lo + n) * kKT + 64, w.i0, w.hb);
            ++gt;
          }
          if (n < w.nt) {
            // K tile n and the relative-encoding rows of band chunk n
            mbar_wait(kr_empty, (gk & 1) ^ 1);
            mbar_expect_tx(kr_full, 32768);
            tma_load_3d(sK, &mK, kr_full, 0, (w.jt_lo + n) * kKT, w.hb);
            tma_load_3d(sR, &mR, kr_full, 0, w.P0 + kKT * n, w.h);
            ++gk;
          } else {
            // the rows of the last band chunk nt go into the v tile, free once
            // the item's last dP has read it: they no longer queue behind the
            // last tile's dQ MMAs on the single K / R buffer (the item's dQ
            // read-out waited ~2 us for them)
            mbar_wait(v_empty, (gv & 1) ^ 1);
            mbar_expect_tx(v_full, 16384);
            tma_load_3d(sV, &mR, v_full, 0, w.P0 + kKT * n, w.h);
            ++gv;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t id_dp = umma_idesc(false, false, false, kQT, kKT);
      const uint32_t id_dq = umma_idesc(false, false, true, kQT, 64);
      const uint32_t ga = smem_u32(sG), ka = smem_u32(sK), ra = smem_u32(sR), vb = smem_u32(sV);
      const uint32_t rg = smem_u32(ring);
      int gt = 0, gk = 0, gv = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        const DqItem w = dq_item(p, it);
        const int gt0 = gt;  // the item's first tile
        auto issue_dq = [&](int n) {
          const int g = gt0 + n;
          if (n == 0) mbar_wait(dq_empty, (li & 1) ^ 1);  // the previous item's dQ read out
          mbar_wait(ds_ready, g & 1);
          dq_trace(dq.trace, 2, g, dq.trace_cta);
          mbar_wait(kr_full, gk & 1);
          tc_fence_after();
          const uint32_t ch = rg + (uint32_t)((n % kRing3) * kChunkBytes), aa = smem_u32(pbuf(g));
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tc_mma<false>(t_dqu, atom_desc<1>(aa, kQT, k), umma_desc(ka + k * 2048, 16384, 1024), id_dq, (n | k) != 0);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tc_mma<false>(t_dqv, atom_desc<1>(ch, kQT, k), umma_desc(ra + k * 2048, 16384, 1024), id_dq, (n | k) != 0);
          tc_commit(&p_empty[g & 1]);
          tc_commit(&ring_free[n % kRing3]);
          tc_commit(kr_empty);
          ++gk;
        };
        mbar_wait(g_full, li & 1);
        for (int n = 0; n < w.nt; ++n, ++gt) {
          const int s = gt & 1;
          mbar_wait(&acc_empty[s], ((gt >> 1) & 1) ^ 1);
          mbar_wait(v_full, gv & 1);
          dq_trace(dq.trace, 3, gt, dq.trace_cta);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma<false>(tmem_base + s * kKT, atom_desc<1>(ga, kQT, k), atom_desc<1>(vb, kKT, k), id_dp, k > 0);
          tc_commit(v_empty);
          ++gv;
          tc_commit(&acc_full[s]);
          if (n == w.nt - 1) tc_commit(g_empty);
          if (n >= 1) issue_dq(n - 1);
        }
        issue_dq(w.nt - 1);
        // band chunk nt (the columns right of the last key tile) is complete with
        // tile nt-1; its relative-encoding rows are in the v tile
        mbar_wait(v_full, gv & 1);
        tc_fence_after();
        const uint32_t ch = rg + (uint32_t)((w.nt % kRing3) * kChunkBytes);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc_mma<false>(t_dqv, atom_desc<1>(ch, kQT, k), umma_desc(vb + k * 2048, 16384, 1024), id_dq, 1u);
        tc_commit(v_empty);
        ++gv;
        tc_commit(dq_full);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    const int rsw = r & 7;
    int ring_uses[kRing3] = {0, 0, 0};  // dQv commits to each ring slot so far (the MMA issuer's count)
    int gt = 0, li = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const DqItem w = dq_item(p, it);
      const int i = w.i0 + r;
      const int jhi = p.M + i;
      float D;
      if (dq.d_in_kernel) {  // written by warps 2-3 (one item ahead), read here
        mbar_wait(&d_ready[li & 1], (li >> 1) & 1);
        D = *reinterpret_cast<volatile const float*>(dq.d_rows + (int64_t)w.hb * p.T + i);
        mbar_arrive(&d_taken[li & 1]);
      } else {
        D = dq.d_rows[(int64_t)w.hb * p.T + i];
      }
      // the previous item's band chunk stores have read the ring and its
      // dQv MMAs are done (dq_full, waited in its epilogue): chunk 0 restarts
      if (warp == 4 && lane == 0) tma_store_wait_read();
      named_sync(1, kSoftWarps * 32);
      auto ring_at = [&](int bc) -> __nv_bfloat16* {  // band column bc of row r
        return reinterpret_cast<__nv_bfloat16*>(ring + (bc >> 7) % kRing3 * kChunkBytes + sw128_off(r, bc & 127));
      };
      const __nv_bfloat16 zb = __float2bfloat16_rn(0.f);
      auto zero_ring = [&](int c0, int c1) {  // band columns [c0, c1) of row r: 16-byte chunks inside
        int c = c0;
        for (; c < c1 && (c & 7); ++c) *ring_at(c) = zb;
        for (; c + 8 <= c1; c += 8) *reinterpret_cast<uint4*>(ring_at(c)) = make_uint4(0u, 0u, 0u, 0u);
        for (; c < c1; ++c) *ring_at(c) = zb;
      };
      if (half == 0) zero_ring(0, 127 - r);  // band columns before this row's first key (chunk 0)
      if (r == 0 && half == 0) dq_trace(dq.trace, 4, li, dq.trace_cta);
      for (int n = 0; n < w.nt; ++n, ++gt) {
        const int s = gt & 1;
        const int jt0 = (w.jt_lo + n) * kKT + 64 * half;
        uint4 pr[2][4];
        mbar_wait(&p_full[gt & 1], (gt >> 1) & 1);
        if (r == 0 && half == 0) dq_trace(dq.trace, 5, gt, dq.trace_cta);
        uint8_t* const tile = pbuf(gt);
        {
          const uint8_t* prow_s = tile + half * (128 * 128) + r * 128;
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int c = 0; c < 4; ++c) pr[k][c] = *reinterpret_cast<const uint4*>(prow_s + (((4 * k + c) ^ rsw) << 4));
        }
        mbar_wait(&acc_full[s], (gt >> 1) & 1);
        tc_fence_after();
        uint32_t dp[2][32];
        tmem_ld32(tl + s * kKT + 64 * half, dp[0]);
        tmem_ld32(tl + s * kKT + 64 * half + 32, dp[1]);
        tc_fence_before();
        mbar_arrive(&acc_empty[s]);
        if (r == 0 && half == 0) dq_trace(dq.trace, 6, gt, dq.trace_cta);
        // the upper band chunk of this tile is reused from tile n - 2 of this
        // item, whose dQv MMA must be done
        if (n >= 2) {
          const int slot = (n + 1) % kRing3;
          mbar_wait(&ring_free[slot], (ring_uses[slot] - 1) & 1);
        }
        if (r == 0 && half == 0) dq_trace(dq.trace, 7, gt, dq.trace_cta);
        if (lane == 0) tma_store_wait_read();
        __syncwarp();
        uint8_t* arow_s = tile + half * (128 * 128) + r * 128;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int jb = jt0 + 32 * k;
          uint32_t o[16];
          const bool inside = jb >= p.lo && jb + 31 <= jhi;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t wv[4] = {pr[k][c].x, pr[k][c].y, pr[k][c].z, pr[k][c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 pf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
              const int t = 8 * c + 2 * e;
              const int j = jb + t;
              float a0 = pf.x * (__uint_as_float(dp[k][t]) - D) * p.scale;
              float a1 = pf.y * (__uint_as_float(dp[k][t + 1]) - D) * p.scale;
              if (!inside) {
                a0 = (j >= p.lo && j <= jhi) ? a0 : 0.f;
                a1 = (j + 1 >= p.lo && j + 1 <= jhi) ? a1 : 0.f;
              }
              __nv_bfloat162 b2 = __floats2bfloat162_rn(a0, a1);
              o[t >> 1] = *reinterpret_cast<uint32_t*>(&b2);
            }
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(arow_s + (((4 * k + c) ^ rsw) << 4)) =
                make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
          const int cb = kKT * n + 127 - r + 64 * half + 32 * k;
          const int split = 64 - (cb & 63);
          uint8_t* seg0 = ring + ((cb >> 7) % kRing3) * kChunkBytes + ((cb >> 6) & 1) * (128 * 128) + r * 128;
          const int c1 = cb + split;
          uint8_t* seg1 = ring + ((c1 >> 7) % kRing3) * kChunkBytes + ((c1 >> 6) & 1) * (128 * 128) + r * 128;
          const int e0 = cb & 63;
          auto at = [&](int t) -> uint8_t* {
            const bool lo = t < split;
            const int e = lo ? e0 + t : t - split;
            return (lo ? seg0 : seg1) + ((((e >> 3) ^ rsw) << 4) | ((e & 7) << 1));
          };
          if ((cb & 1) == 0) {
#pragma unroll
            for (int m = 0; m < 16; ++m) *reinterpret_cast<uint32_t*>(at(2 * m)) = o[m];
          } else {
            *reinterpret_cast<unsigned short*>(at(0)) = (unsigned short)(o[0] & 0xffffu);
#pragma unroll
            for (int m = 0; m < 15; ++m) *reinterpret_cast<uint32_t*>(at(2 * m + 1)) = __byte_perm(o[m], o[m + 1], 0x5432);
            *reinterpret_cast<unsigned short*>(at(31)) = (unsigned short)(o[15] >> 16);
          }
        }
        if (n == w.nt - 1 && half == 1) zero_ring(kKT * n + 255 - r, kKT * (w.nt + 1));  // after this row's last key
        fence_proxy_async_smem();
        __syncwarp();
        if (warp == 4 && lane == 0) tma_store_wait_read();
        if (r == 0 && half == 0) dq_trace(dq.trace, 8, gt, dq.trace_cta);
        named_sync(1, kSoftWarps * 32);
        if (r == 0 && half == 0) dq_trace(dq.trace, 9, gt, dq.trace_cta);
        ++ring_uses[n % kRing3];  // the dQv MMA of this tile commits ring_free[n % 3]
        if (warp == 4 && lane == 0) {
          mbar_arrive(ds_ready);
          for (int m = n; m <= (n == w.nt - 1 ? n + 1 : n); ++m) {
            const uint8_t* ch = ring + (m % kRing3) * kChunkBytes;
            const int c0 = w.P0 + kKT * m;
            if (c0 < p.ldp) tma_store_3d(&mBD, ch, c0, w.i0, w.hb);
            if (c0 + 64 < p.ldp) tma_store_3d(&mBD, ch + 128 * 128, c0 + 64, w.i0, w.hb);
          }
        }
      }
      // ---- dQu / dQv epilogue: rows of this lane quarter, columns [32 half, +32)
      mbar_wait(dq_full, li & 1);
      if (r == 0 && half == 0) dq_trace(dq.trace, 10, li, dq.trace_cta);
      tc_fence_after();
      uint32_t vu[32], vv[32];
      tmem_ld32(tl + 256 + 32 * half, vu);
      tmem_ld32(tl + 320 + 32 * half, vv);
      tc_fence_before();
      mbar_arrive(dq_empty);  // the next item's dQ MMAs may overwrite the accumulators
      if (dq.gqkv) {
        // the merged query gradient: bf16(dQu + dQv) in the current row's query columns
        uint4* dst = reinterpret_cast<uint4*>(
            dq.gqkv + ((int64_t)p.B * p.M + (int64_t)w.b * p.T + i) * (3 * p.d) + w.h * 64 + 32 * half);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t = 8 * c + 2 * e;
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(vu[t]) + __uint_as_float(vv[t]),
                                                      __uint_as_float(vu[t + 1]) + __uint_as_float(vv[t + 1]));
            o4[e] = *reinterpret_cast<uint32_t*>(&b2);
          }
          dst[c] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
      } else {
        const int64_t orow = ((int64_t)w.hb * p.T + i) * 64 + 32 * half;
        float4* du = reinterpret_cast<float4*>(dq.gqu + orow);
        float4* dv = reinterpret_cast<float4*>(dq.gqv + orow);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          du[c] = make_float4(__uint_as_float(vu[4 * c]), __uint_as_float(vu[4 * c + 1]), __uint_as_float(vu[4 * c + 2]),
                              __uint_as_float(vu[4 * c + 3]));
          dv[c] = make_float4(__uint_as_float(vv[4 * c]), __uint_as_float(vv[4 * c + 1]), __uint_as_float(vv[4 * c + 2]),
                              __uint_as_float(vv[4 * c + 3]));
        }
      }
      if (dq.bias_part) {
        float a[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) a[c] = __uint_as_float(vu[c]);
        const float colsum_u = warp_colsum32(a, lane);
#pragma unroll
        for (int c = 0; c < 32; ++c) a[c] = __uint_as_float(vv[c]);
        const float colsum_v = warp_colsum32(a, lane);
        // the four lane-quarter warps of this column half, summed in quarter
        // order through ring slot (nt + 1) % 3: it held chunk nt - 2, whose
        // dBD stores were read before tile nt - 1's barrier and whose dQv MMA
        // is done (dq_full).  The next item's start barrier orders these reads
        // before its ring writes.
        float* red = reinterpret_cast<float*>(ring + ((w.nt + 1) % kRing3) * kChunkBytes);
        red[((half * 2 + 0) * 4 + q) * 32 + lane] = colsum_u;
        red[((half * 2 + 1) * 4 + q) * 32 + lane] = colsum_v;
        named_sync(1, kSoftWarps * 32);
        if (q == 0) {
#pragma unroll
          for (int wq = 0; wq < 2; ++wq) {
            const float* rr = red + (half * 2 + wq) * 4 * 32 + lane;
            const float sum = ((rr[0] + rr[32]) + rr[64]) + rr[96];
            dq.bias_part[(((int64_t)wq * p.B + w.b) * p.nqt + w.qt) * p.H * 64 + w.h * 64 + 32 * half + lane] = sum;
          }
        }
      }
    }
    if (lane == 0) tma_store_wait_all();
  } else {
    // warps 2 and 3: each item's D rows (one item ahead of the softmax warps:
    // D_i = g_ctx_i . ctx_i, bwd_dq's arithmetic, into d_rows for bwd_kv as
    // well), then the dBD margins outside its band chunks (coalesced)
    int li = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const DqItem w = dq_item(p, it);
      if (dq.d_in_kernel) {
        if (li >= 2) mbar_wait(&d_taken[li & 1], ((li >> 1) - 1) & 1);  // bounded lookahead: the barrier's phase
        for (int rr = (warp - 2) * 32 + lane; rr < kQT; rr += 64) {
          const int i = w.i0 + rr;
          const int64_t mo = ((int64_t)w.b * p.T + i) * p.d + w.h * 64;
          const uint4* g4 = reinterpret_cast<const uint4*>(p.gctx + mo);
          const uint4* c4 = reinterpret_cast<const uint4*>(p.ctx + mo);
          float D = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 gu = g4[c], cu = c4[c];
            const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w}, cw[4] = {cu.x, cu.y, cu.z, cu.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[e]));
              const float2 cf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cw[e]));
              D = fmaf(gf.x, cf.x, D);
              D = fmaf(gf.y, cf.y, D);
            }
          }
          dq.d_rows[(int64_t)w.hb * p.T + i] = D;
        }
        __threadfence_block();
        mbar_arrive(&d_ready[li & 1]);
      }
      const int64_t bl = lmin(lmax(w.P0, 0), p.ldp), br = lmin(lmax((int64_t)w.P0 + kKT * (w.nt + 1), 0), p.ldp);
      for (int rr = warp - 2; rr < kQT; rr += 2) {
        __nv_bfloat16* row = p.gbd + ((int64_t)w.hb * p.T + w.i0 + rr) * p.ldp;
        for (int64_t c = 8 * lane; c < bl; c += 256) *reinterpret_cast<uint4*>(row + c) = make_uint4(0u, 0u, 0u, 0u);
        for (int64_t c = br + 8 * lane; c < p.ldp; c += 256)
          *reinterpret_cast<uint4*>(row + c) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

// Key-major backward of the key-side gradients (head dim 64, bf16; after
// xl_attn_bwd_dq, which leaves D_i = dO_i . O_i per query row).  Work item =
// (head*batch, 128-key tile); per query tile that sees the key tile
//     dP   = dO_q V^T            TMEM cols 0..255 (two buffers), lanes = queries
//     dS   = P (dP - D) scale    bwd_dq's dAC arithmetic, bf16, written over the P tile
//     dV  += P_q^T dO_q          lanes = keys (A = the TMA'd P tile, MN-major)
//     dK  += dS_q^T Qu_q                      (A = the same tile, now dS, MN-major)
// with dV / dK double-buffered per item (TMEM cols 256 + 128 b: dV, +64: dK).
// Persistent: one CTA per SM walks the items (memory-side key tiles, which
// every query tile sees, first) and the pipelines run on across item
// boundaries -- an item has only 1..4 query tiles.  P is the one DRAM stream
// (dO, q+u and v tiles are re-read across key tiles from L2): it has its own
// producer thread and kKvP stages.  Each thread overwrites exactly the P
// values it read with its dS (same rows, same columns), once the dV MMA of
// the step has read the tile -- so dS needs no buffer of its own and has as
// many as P (a separate single dS tile chained every step's dS stores behind
// the previous step's dK).  dP / dV and dK have separate issuing threads, so
// neither waits on the other's operands.  Sixteen softmax warps, four per TMEM
// lane quarter, 32 key columns each.
// Measured at C3 (tools/prof_xl_fused.py, RP_XL_KV_TRACE event timelines):
// ~76 us, ~1.2 us per step, bound by the P stream -- a 32 KB tile lands
// ~5.7 us after its TMA issue (~3.2 TB/s of 256-byte row segments), and the
// shared memory holds four stages.  The banded dV / dK GEMMs it replaces took
// 37 us each, plus the dAC matrix (16 us of xl_attn_bwd_dq).
// This is the K = 16 MMA sequence of the banded dV / dK GEMMs over P and dAC
// (the same operands in the same order), so the result is bitwise theirs --
// without the dAC matrix (185 MB written and read per block at C3) or the
// GEMMs' second read of P.
constexpr int kKvP = 4;
constexpr int kKvSoft = 16;                       // softmax warps
constexpr int kKvThreads = 128 + 32 * kKvSoft;    // + TMA (P), MMA (dP, dV), TMEM + MMA (dK), TMA (dO / q+u / v)
constexpr int kKvSmem = 1024 + 2 * 16384 /*V*/ + 2 * 16384 /*dO*/ + 2 * 16384 /*Qu*/ + kKvP * kChunkBytes /*P, dS*/ +
                        512 /*barriers*/;

struct KvParams {
  const float* D;     // [HB*T]
  __nv_bfloat16* gk;  // [HB, Kl, 64]
  __nv_bfloat16* gv;
  int T, M, Kl, lo, nkt, HB;
  float scale;
  unsigned long long* trace;  // RP_XL_KV_TRACE: CTA 0's event times (diagnostics)
  __nv_bfloat16* gqkv;  // optional: dK / dV straight into the merged g_qkv rows (key / value columns)
  int B, d;
};

__device__ __forceinline__ void kv_trace(const KvParams& p, int ev, int idx) {
  if (p.trace && blockIdx.x == 0 && idx < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[ev * 64 + idx] = t;
  }
}

// item -> (key tile, head*batch, first query tile, query tiles)
__device__ __forceinline__ void kv_item(const KvParams& p, int it, int& kt, int& hb, int& qt_lo, int& nq) {
  kt = it / p.HB;
  hb = it - kt * p.HB;
  // query i sees key j <= M + i: the first query tile with a query at or past j0 - M
  qt_lo = max(kt * kKT - p.M, 0) / kQT;
  nq = p.T / kQT - qt_lo;
}

__global__ void __launch_bounds__(kKvThreads, 1)
    xl_attn_bwd_kv_kernel(const __grid_constant__ CUtensorMap mG, const __grid_constant__ CUtensorMap mV,
                          const __grid_constant__ CUtensorMap mU, const __grid_constant__ CUtensorMap mP,
                          const KvParams p) {
  constexpr int NP = kKvP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sV = smem;            // [2] per item
  uint8_t* sG = sV + 2 * 16384;  // [2] per step
  uint8_t* sU = sG + 2 * 16384;  // [2]
  uint8_t* sP = sU + 2 * 16384;  // [NP] x two 64-key atoms: P, then dS
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + NP * kChunkBytes);
  uint64_t* v_full = bars;          // [2]
  uint64_t* v_empty = bars + 2;     // [2]
  uint64_t* g_full = bars + 4;      // [2]
  uint64_t* g_empty = bars + 6;     // [2]
  uint64_t* u_full = bars + 8;      // [2]
  uint64_t* u_empty = bars + 10;    // [2]
  uint64_t* acc_full = bars + 12;   // [2]
  uint64_t* acc_empty = bars + 14;  // [2]
  uint64_t* kv_full = bars + 16;    // [2]: an item's dV / dK complete
  uint64_t* kv_empty = bars + 18;   // [2]: and read out
  uint64_t* p_full = bars + 20;     // [NP]: P landed
  uint64_t* pv_done = p_full + NP;  // [NP]: the dV MMA has read P (dS may overwrite it)
  uint64_t* ds_ready = pv_done + NP;  // [NP]: dS written (every softmax thread)
  uint64_t* p_empty = ds_ready + NP;  // [NP]: the dK MMA has read dS
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_empty + NP);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = p.HB * p.nkt;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mG);
    tma_prefetch(&mV);
    tma_prefetch(&mU);
    tma_prefetch(&mP);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&g_full[s], 1);
      mbar_init(&g_empty[s], 1);
      mbar_init(&u_full[s], 1);
      mbar_init(&u_empty[s], 1);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kKvSoft * 32);
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], kKvSoft * 32);
    }
    for (int s = 0; s < NP; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&pv_done[s], 1);
      mbar_init(&ds_ready[s], kKvSoft * 32);  // every softmax thread, after its own proxy fence
      mbar_init(&p_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: the P stream ----------------
      int gs = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        int kt, hb, qt_lo, nq;
        kv_item(p, it, kt, hb, qt_lo, nq);
        const int j0 = kt * kKT;
        for (int n = 0; n < nq; ++n, ++gs) {
          const int ps = gs % NP;
          mbar_wait(&p_empty[ps], ((gs / NP) & 1) ^ 1);
          kv_trace(p, 1, gs);
          mbar_expect_tx(&p_full[ps], kChunkBytes);
          const int i0 = (qt_lo + n) * kQT;
          tma_load_3d(sP + ps * kChunkBytes, &mP, &p_full[ps], j0, i0, hb);
          tma_load_3d(sP + ps * kChunkBytes + 128 * 128, &mP, &p_full[ps], j0 + 64, i0, hb);
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ---------------- TMA producer: v per item, dO / q+u per step (L2-resident) ----------------
      int gs = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        int kt, hb, qt_lo, nq;
        kv_item(p, it, kt, hb, qt_lo, nq);
        const int vb = li & 1;
        mbar_wait(&v_empty[vb], ((li >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[vb], 16384);
        tma_load_3d(sV + vb * 16384, &mV, &v_full[vb], 0, kt * kKT, hb);
        for (int n = 0; n < nq; ++n, ++gs) {
          const int i0 = (qt_lo + n) * kQT, s = gs & 1;
          const uint32_t ph = ((gs >> 1) & 1) ^ 1;
          mbar_wait(&g_empty[s], ph);
          kv_trace(p, 0, gs);
          mbar_expect_tx(&g_full[s], 16384);
          tma_load_3d(sG + s * 16384, &mG, &g_full[s], 0, i0, hb);
          mbar_wait(&u_empty[s], ph);
          kv_trace(p, 2, gs);
          mbar_expect_tx(&u_full[s], 16384);
          tma_load_3d(sU + s * 16384, &mU, &u_full[s], 0, i0, hb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: dP and dV (need only the TMA'd tiles) ----------------
      const uint32_t id_dp = umma_idesc(false, false, false, kQT, kKT);
      const uint32_t id_kv = umma_idesc(false, true, true, kKT, 64);
      int gs = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        int kt, hb, qt_lo, nq;
        kv_item(p, it, kt, hb, qt_lo, nq);
        const int kb = li & 1;
        const uint32_t t_dv = tmem_base + 256 + 128 * kb;
        const uint32_t vaddr = smem_u32(sV + kb * 16384);
        mbar_wait(&v_full[kb], (li >> 1) & 1);
        mbar_wait(&kv_empty[kb], ((li >> 1) & 1) ^ 1);  // item li - 2's dV / dK read out
        for (int n = 0; n < nq; ++n, ++gs) {
          const int s = gs & 1, ps = gs % NP;
          mbar_wait(&acc_empty[s], ((gs >> 1) & 1) ^ 1);
          kv_trace(p, 5, gs);
          mbar_wait(&g_full[s], (gs >> 1) & 1);
          kv_trace(p, 6, gs);
          tc_fence_after();
          const uint32_t ga = smem_u32(sG + s * 16384);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma<false>(tmem_base + s * kKT, atom_desc<1>(ga, kQT, k), atom_desc<1>(vaddr, kKT, k), id_dp, k > 0);
          tc_commit(&acc_full[s]);
          if (n == nq - 1) tc_commit(&v_empty[kb]);
          mbar_wait(&p_full[ps], (gs / NP) & 1);
          kv_trace(p, 7, gs);
          tc_fence_after();
          const uint32_t pa = smem_u32(sP + ps * kChunkBytes);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tc_mma<false>(t_dv, umma_desc(pa + k * 2048, 16384, 1024), umma_desc(ga + k * 2048, 16384, 1024), id_kv,
                          (n | k) != 0);
          tc_commit(&pv_done[ps]);
          tc_commit(&g_empty[s]);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ---------------- MMA issuer: dK (waits for each step's dS) ----------------
      // A second issuing thread: with one, a step's dK queued behind the next
      // step's P tile (dV) or the next dV behind this dK, and each step paid
      // that wait.  dK of an item's last step completing implies the item's dV
      // did (the softmax warps wrote that dS only after its dV), so its commit
      // alone signals the item's dV / dK.
      const uint32_t id_kv = umma_idesc(false, true, true, kKT, 64);
      int gs = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        int kt, hb, qt_lo, nq;
        kv_item(p, it, kt, hb, qt_lo, nq);
        const int kb = li & 1;
        const uint32_t t_dk = tmem_base + 256 + 128 * kb + 64;
        mbar_wait(&kv_empty[kb], ((li >> 1) & 1) ^ 1);
        for (int n = 0; n < nq; ++n, ++gs) {
          const int ps = gs % NP, us = gs & 1;
          mbar_wait(&ds_ready[ps], (gs / NP) & 1);
          kv_trace(p, 3, gs);
          mbar_wait(&u_full[us], (gs >> 1) & 1);
          kv_trace(p, 4, gs);
          tc_fence_after();
          const uint32_t aa = smem_u32(sP + ps * kChunkBytes), ua = smem_u32(sU + us * 16384);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tc_mma<false>(t_dk, umma_desc(aa + k * 2048, 16384, 1024), umma_desc(ua + k * 2048, 16384, 1024), id_kv,
                          (n | k) != 0);
          tc_commit(&p_empty[ps]);
          tc_commit(&u_empty[us]);
          if (n == nq - 1) tc_commit(&kv_full[kb]);
        }
      }
    }
  } else if (warp >= 4) {
    // lane quarter q (TMEM lanes 32q..: query rows, then key rows), key columns [32 part, +32)
    const int q = warp & 3, part = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const int rsw = r & 7;
    const int atom = part >> 1, cb = (part & 1) * 4;  // 64-key swizzle atom and 16-byte chunk base
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
    int gs = 0, li = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      int kt, hb, qt_lo, nq;
      kv_item(p, it, kt, hb, qt_lo, nq);
      const int j0 = kt * kKT, kb = li & 1;
      for (int n = 0; n < nq; ++n, ++gs) {
        const int s = gs & 1, ps = gs % NP;
        const int i = (qt_lo + n) * kQT + r;
        const int jhi = p.M + i;
        const float D = p.D[(int64_t)hb * p.T + i];
        uint8_t* row_s = sP + ps * kChunkBytes + atom * (128 * 128) + r * 128;
        uint4 pr[4];
        mbar_wait(&p_full[ps], (gs / NP) & 1);
        if (r == 0 && part == 0) kv_trace(p, 8, gs);
#pragma unroll
        for (int c = 0; c < 4; ++c) pr[c] = *reinterpret_cast<const uint4*>(row_s + (((cb + c) ^ rsw) << 4));
        mbar_wait(&acc_full[s], (gs >> 1) & 1);
        if (r == 0 && part == 0) kv_trace(p, 9, gs);
        tc_fence_after();
        uint32_t dp[32];
        tmem_ld32(tl + s * kKT + 32 * part, dp);
        tc_fence_before();
        mbar_arrive(&acc_empty[s]);
        uint32_t o[16];
        {
          const int jb = j0 + 32 * part;
          const bool inside = jb >= p.lo && jb + 31 <= jhi;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t w[4] = {pr[c].x, pr[c].y, pr[c].z, pr[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 pf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
              const int t = 8 * c + 2 * e;
              const int j = jb + t;
              float a0 = pf.x * (__uint_as_float(dp[t]) - D) * p.scale;
              float a1 = pf.y * (__uint_as_float(dp[t + 1]) - D) * p.scale;
              if (!inside) {
                a0 = (j >= p.lo && j <= jhi) ? a0 : 0.f;
                a1 = (j + 1 >= p.lo && j + 1 <= jhi) ? a1 : 0.f;
              }
              __nv_bfloat162 b2 = __floats2bfloat162_rn(a0, a1);
              o[t >> 1] = *reinterpret_cast<uint32_t*>(&b2);
            }
          }
        }
        // dS over this thread's own P values, once the dV MMA has read the tile
        mbar_wait(&pv_done[ps], (gs / NP) & 1);
        if (r == 0 && part == 0) kv_trace(p, 10, gs);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(row_s + (((cb + c) ^ rsw) << 4)) =
              make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        fence_proxy_async_smem();
        mbar_arrive(&ds_ready[ps]);
        if (r == 0 && part == 0) kv_trace(p, 11, gs);
        if (lane == 0) kv_trace(p, 15 + warp - 4, gs);  // every softmax warp's arrival
      }
      // ---- this item's dV (parts 0, 1) / dK (parts 2, 3): key rows of this lane quarter
      if (r == 0 && part == 0) kv_trace(p, 12, li);
      mbar_wait(&kv_full[kb], (li >> 1) & 1);
      if (r == 0 && part == 0) kv_trace(p, 13, li);
      tc_fence_after();
      const int j = j0 + r;
      uint32_t v[32];
      tmem_ld32(tl + 256 + 128 * kb + 32 * part, v);
      tc_fence_before();
      mbar_arrive(&kv_empty[kb]);
      if (j < p.Kl) {
        uint4* dst;
        if (p.gqkv) {  // merged rows: memory rows b*M + j, then current rows B*M + b*T + (j - M)
          const int h = hb / p.B, b = hb - h * p.B;
          const int64_t row = j < p.M ? (int64_t)b * p.M + j : (int64_t)p.B * p.M + (int64_t)b * p.T + (j - p.M);
          dst = reinterpret_cast<uint4*>(p.gqkv + row * (3 * p.d) + (part < 2 ? 2 : 1) * p.d + h * 64 + 32 * (part & 1));
        } else {
          dst = reinterpret_cast<uint4*>((part < 2 ? p.gv : p.gk) + ((int64_t)hb * p.Kl + j) * 64 + 32 * (part & 1));
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t ob[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 b2 =
                __floats2bfloat162_rn(__uint_as_float(v[8 * c + 2 * e]), __uint_as_float(v[8 * c + 2 * e + 1]));
            ob[e] = *reinterpret_cast<uint32_t*>(&b2);
          }
          dst[c] = make_uint4(ob[0], ob[1], ob[2], ob[3]);
        }
      }
      if (r == 0 && part == 0) kv_trace(p, 14, li);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

}  // namespace

// u / v gradients from xl_attn_bwd_dq's per-CTA column sums: head h sums its
// B * nqt partials in (b, query tile) order
__global__ void dq_bias_finish_kernel(const float* __restrict__ part, float* __restrict__ gu, float* __restrict__ gv,
                                      int H, int B, int nqt) {
  const int h = blockIdx.x, w = blockIdx.y, c = threadIdx.x;  // 64 threads
  const int64_t ld = (int64_t)H * 64;
  const float* src = part + (int64_t)w * B * nqt * ld + h * 64 + c;
  float s = 0.f;
  const int n = B * nqt;
  int k = 0;
  for (; k + 4 <= n; k += 4) {  // four loads in flight, additions in order
    const float v0 = src[k * ld], v1 = src[(k + 1) * ld];
    const float v2 = src[(k + 2) * ld], v3 = src[(k + 3) * ld];
    s += v0;
    s += v1;
    s += v2;
    s += v3;
  }
  for (; k < n; ++k) s += src[k * ld];
  (w ? gv : gu)[h * 64 + c] = s;
}

int64_t xl_dq_bias_part_bytes(int H, int64_t B, int64_t Tn) { return 2 * (int64_t)H * B * (Tn / kQT) * 64 * 4; }

int xl_dq_bias_finish(const float* part, float* gu, float* gv, int H, int64_t B, int64_t Tn, cudaStream_t st) {
  if (H <= 0 || B <= 0 || Tn % kQT) return set_error(RP_ERR_DIMENSION, "xl_dq_bias_finish: bad shape");
  dq_bias_finish_kernel<<<dim3(H, 2), 64, 0, st>>>(part, gu, gv, H, (int)B, (int)(Tn / kQT));
  return check_launch("xl_dq_bias_finish");
}

// RP_XL_ORDER=0 restores the (head*batch)-major CTA order (A/B switch)
static int xl_heavy_first() {
  static const int v = getenv("RP_XL_ORDER") ? atoi(getenv("RP_XL_ORDER")) : 1;
  return v;
}

int xl_attn_fwd(const void* qu, const void* qv, const void* kh, const void* rh, void* probs, int64_t ldp, int64_t B,
                int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale, cudaStream_t st) {
  if (dh != 64 && dh != 128) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: head dim must be 64 or 128 (got %d)", dh);
  const int64_t Kl = M + Tn, HB = (int64_t)H * B;
  if (ldp < Kl || ldp % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: ldp must be >= M+T and a multiple of 8");
  if (mem_len < 0 || mem_len > M) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: mem_len out of range");
  if ((reinterpret_cast<uintptr_t>(probs) & 15) != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd: P not 16B aligned");
  CUtensorMap mqu, mqv, mk, mr;
  RP_TRY0(tma_map_bf16(&mqu, qu, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mqv, qv, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mk, kh, dh, Kl, dh, HB, Kl * dh, 64, kFKT));
  RP_TRY0(tma_map_bf16(&mr, rh, dh, Kl, dh, H, Kl * dh, 64, kFBand));
  CUtensorMap mp;
  RP_TRY0(tma_map_bf16_store32(&mp, probs, ldp, Tn, ldp, HB));
  static uint64_t attr_done = 0;
  if (first_on_device(attr_done)) {
    cudaFuncSetAttribute(xl_attn_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_fwd<1>());
    cudaFuncSetAttribute(xl_attn_fwd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_fwd<2>());
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
  p.heavy_first = xl_heavy_first();
  p.c2 = scale * 1.4426950408889634f;
  static const int dbg = getenv("RP_XL_DBG") ? atoi(getenv("RP_XL_DBG")) : 0;
  p.dbg = dbg;
  const int64_t grid = HB * p.nqt;
  if (grid <= 0) return RP_OK;
  if (dh == 64)
    xl_attn_fwd_kernel<1><<<(unsigned)grid, kThreadsFwd, smem_fwd<1>(), st>>>(mqu, mqv, mk, mr, mp, p);
  else
    xl_attn_fwd_kernel<2><<<(unsigned)grid, kThreadsFwd, smem_fwd<2>(), st>>>(mqu, mqv, mk, mr, mp, p);
  return check_launch("xl_attn_fwd");
}


int xl_attn_bwd(const void* gctx_h, const void* vh, const void* probs, void* gac, void* gbd, int64_t ldp,
                const void* gctx, const void* ctx, int64_t B, int64_t Tn, int64_t M, int H, int dh, int mem_len,
                float scale, cudaStream_t st) {
  if (dh != 64 && dh != 128) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd: head dim must be 64 or 128 (got %d)", dh);
  // dBD chunks are TMA-stored at column T - 128 - i0 + 128 n: 16-byte aligned only for T % 8 == 0
  if (Tn % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd: T must be a multiple of 8 (got %lld)", (long long)Tn);
  const int64_t Kl = M + Tn, HB = (int64_t)H * B;
  if (ldp < Kl || ldp % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd: ldp must be >= M+T and a multiple of 8");
  if (mem_len < 0 || mem_len > M) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd: mem_len out of range");
  for (const void* q : {probs, (const void*)gac, (const void*)gbd, gctx, ctx})
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd: unaligned operand");
  CUtensorMap mg, mv, mbd;
  RP_TRY0(tma_map_bf16(&mg, gctx_h, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mv, vh, dh, Kl, dh, HB, Kl * dh, 64, kKT));
  RP_TRY0(tma_map_bf16(&mbd, gbd, ldp, Tn, ldp, HB, Tn * ldp, 128, kQT, false));
  CUtensorMap mac;
  RP_TRY0(tma_map_bf16_store32(&mac, gac, ldp, Tn, ldp, HB));
  static uint64_t attr_done = 0;
  if (first_on_device(attr_done)) {
    cudaFuncSetAttribute(xl_attn_bwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bwd<1>());
    cudaFuncSetAttribute(xl_attn_bwd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bwd<2>());
  }
  BwdParams p;
  p.p = static_cast<const __nv_bfloat16*>(probs);
  p.gac = static_cast<__nv_bfloat16*>(gac);
  p.gbd = static_cast<__nv_bfloat16*>(gbd);
  p.gctx = static_cast<const __nv_bfloat16*>(gctx);
  p.ctx = static_cast<const __nv_bfloat16*>(ctx);
  p.ldp = ldp;
  p.B = (int)B;
  p.T = (int)Tn;
  p.M = (int)M;
  p.Kl = (int)Kl;
  p.lo = (int)(M - mem_len);
  p.nqt = (int)((Tn + kQT - 1) / kQT);
  p.heavy_first = xl_heavy_first();
  p.H = H;
  p.d = H * dh;
  p.scale = scale;
  const int64_t grid = HB * p.nqt;
  if (grid <= 0) return RP_OK;
  if (dh == 64)
    xl_attn_bwd_kernel<1><<<(unsigned)grid, kThreadsBwd, smem_bwd<1>(), st>>>(mg, mv, mbd, mac, p);
  else
    xl_attn_bwd_kernel<2><<<(unsigned)grid, kThreadsBwd, smem_bwd<2>(), st>>>(mg, mv, mbd, mac, p);
  return check_launch("xl_attn_bwd");
}

bool xl_dq_persistent() {
  static int persist = -1;
  if (persist < 0) {
    const char* e = getenv("RP_XL_DQ_PERSIST");
    persist = (e && e[0] == '0') ? 0 : 1;
  }
  return persist == 1;
}

int xl_attn_bwd_dq(const void* gctx_h, const void* vh, const void* kh, const void* rh, const void* probs, void* gac,
                   void* gbd, int64_t ldp, const void* gctx, const void* ctx, float* gqu, float* gqv, int64_t B,
                   int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale, cudaStream_t st, float* bias_part,
                   float* d_rows, void* gqkv) {
  if (dh != 64) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: head dim must be 64 (got %d)", dh);
  if (Tn % 128 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: T must be a multiple of 128");
  const int64_t Kl = M + Tn, HB = (int64_t)H * B;
  if (ldp < Kl || ldp % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: ldp must be >= M+T, multiple of 8");
  if (mem_len < 0 || mem_len > M) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: mem_len out of range");
  for (const void* q : {probs, (const void*)gac, (const void*)gbd, gctx, ctx, (const void*)gqu, (const void*)gqv})
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: unaligned operand");
  CUtensorMap mg, mv, mk, mr, mbd, mac, mp;
  RP_TRY0(tma_map_bf16(&mp, probs, ldp, Tn, ldp, HB, Tn * ldp, 64, kQT));
  RP_TRY0(tma_map_bf16(&mg, gctx_h, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mv, vh, dh, Kl, dh, HB, Kl * dh, 64, kKT));
  RP_TRY0(tma_map_bf16(&mk, kh, dh, Kl, dh, HB, Kl * dh, 64, kKT));
  RP_TRY0(tma_map_bf16(&mr, rh, dh, Kl, dh, H, Kl * dh, 64, kKT));
  RP_TRY0(tma_map_bf16(&mbd, gbd, ldp, Tn, ldp, HB, Tn * ldp, 64, kQT));
  // gac NULL: no dAC (xl_attn_bwd_kv forms dK from dS itself); the map is then never used
  RP_TRY0(tma_map_bf16(&mac, gac ? gac : gbd, ldp, Tn, ldp, HB, Tn * ldp, 64, 32));
  static uint64_t attr_done = 0;
  if (first_on_device(attr_done))
    cudaFuncSetAttribute(xl_attn_bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDqSmem);
  DqParams q{};
  BwdParams& p = q.b;
  p.p = static_cast<const __nv_bfloat16*>(probs);
  p.gac = static_cast<__nv_bfloat16*>(gac);
  p.gbd = static_cast<__nv_bfloat16*>(gbd);
  p.gctx = static_cast<const __nv_bfloat16*>(gctx);
  p.ctx = static_cast<const __nv_bfloat16*>(ctx);
  p.ldp = ldp;
  p.B = (int)B;
  p.T = (int)Tn;
  p.M = (int)M;
  p.Kl = (int)Kl;
  p.lo = (int)(M - mem_len);
  p.nqt = (int)(Tn / kQT);
  p.heavy_first = xl_heavy_first();
  p.H = H;
  p.d = H * dh;
  p.scale = scale;
  q.gqu = gqu;
  q.gqv = gqv;
  q.bias_part = bias_part;
  q.d_rows = d_rows;
  q.no_dac = gac == nullptr;
  const bool persist = xl_dq_persistent();
  q.gqkv = static_cast<__nv_bfloat16*>(gqkv);
  if (gqkv && !(persist && q.no_dac && d_rows))
    return set_error(RP_ERR_INVALID, "xl_attn_bwd_dq: merged query-gradient rows need the persistent kernel "
                                     "(no dAC, D rows, RP_XL_DQ_PERSIST != 0)");
  if (gqkv && (reinterpret_cast<uintptr_t>(gqkv) & 15) != 0)
    return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: unaligned merged rows");
  if (persist && q.no_dac && d_rows) {
    // the production path: D rows first (one pass over g_ctx / ctx), then the
    // persistent kernel (one CTA per SM over the (head*batch, query tile) items)
    if ((reinterpret_cast<uintptr_t>(d_rows) & 3) != 0)
      return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: unaligned D rows");
    const int64_t rows = HB * Tn;
    static const int d_sep = getenv("RP_XL_DQ_DPASS") ? atoi(getenv("RP_XL_DQ_DPASS")) : 0;  // 1: separate D pass
    q.d_in_kernel = d_sep ? 0 : 1;
    if (rows > 0 && d_sep)
      d_rows_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(gctx),
                                                                    static_cast<const __nv_bfloat16*>(ctx), d_rows,
                                                                    (int)B, (int)Tn, H, H * dh);
    p.ldp = ldp;
    p.B = (int)B;
    p.T = (int)Tn;
    p.M = (int)M;
    p.Kl = (int)Kl;
    p.lo = (int)(M - mem_len);
    p.nqt = (int)(Tn / kQT);
    p.heavy_first = xl_heavy_first();
    p.H = H;
    p.d = H * dh;
    p.scale = scale;
    p.p = static_cast<const __nv_bfloat16*>(probs);
    p.gbd = static_cast<__nv_bfloat16*>(gbd);
    q.gqu = gqu;
    q.gqv = gqv;
    const int64_t items = HB * p.nqt;
    if (items <= 0) return RP_OK;
    static uint64_t attr_p = 0;
    if (first_on_device(attr_p))
      cudaFuncSetAttribute(xl_attn_bwd_dq_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDqSmem);
    static int sms[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (sms[dev & 63] == 0) {
      int v = 0;
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      sms[dev & 63] = v > 0 ? v : 148;
    }
    int64_t grid = std::min<int64_t>(items, sms[dev & 63]);
    if (const char* e = getenv("RP_XL_DQ_CTAS"))  // tests: fewer CTAs, several items each
      if (atoi(e) > 0) grid = std::min<int64_t>(grid, atoi(e));
    static unsigned long long* ptrace = nullptr;
    const bool tr = getenv("RP_XL_DQ_TRACE") != nullptr;
    if (tr) {
      if (!ptrace) cudaMalloc(&ptrace, 11 * 32 * 8);
      cudaMemsetAsync(ptrace, 0, 11 * 32 * 8, st);
      q.trace_cta = atoi(getenv("RP_XL_DQ_TRACE"));
      q.trace = ptrace;
    }
    xl_attn_bwd_dq_persist_kernel<<<(unsigned)grid, kThreadsBwd, kDqSmem, st>>>(mg, mv, mk, mr, mbd, mp, q);
    if (tr) {
      unsigned long long h[11 * 32];
      cudaMemcpyAsync(h, ptrace, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      unsigned long long t0 = ~0ull;
      for (int i = 0; i < 11 * 32; ++i)
        if (h[i] && h[i] < t0) t0 = h[i];
      static const char* names[11] = {"-", "P:P", "M:dsrdy", "M:vfull", "S:item", "S:pfull", "S:acc",
                                      "S:ring", "S:stored", "S:ds", "S:dqfull"};
      for (int ev = 1; ev < 11; ++ev) {
        fprintf(stderr, "%-9s", names[ev]);
        for (int i = 0; i < 32; ++i) fprintf(stderr, " %6.2f", h[ev * 32 + i] ? (h[ev * 32 + i] - t0) * 1e-3 : -1.0);
        fprintf(stderr, "\n");
      }
    }
    return check_launch("xl_attn_bwd_dq (persistent)");
  }
  // C3 A/B: without dAC, warps 2-3 zeroing the dBD margins 182 -> 176 us; with dAC 202 -> 208 us
  q.zero_rows = gac != nullptr;
  if (const char* e = getenv("RP_XL_DQ_ZERO_ROWS")) q.zero_rows = atoi(e);
  if ((reinterpret_cast<uintptr_t>(d_rows) & 3) != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_dq: unaligned D rows");
  const int64_t grid = HB * p.nqt;
  if (grid <= 0) return RP_OK;
  static unsigned long long* trace = nullptr;
  const bool tr = getenv("RP_XL_DQ_TRACE") != nullptr;
  if (tr) {
    if (!trace) cudaMalloc(&trace, 11 * 32 * 8);
    cudaMemsetAsync(trace, 0, 11 * 32 * 8, st);
    q.trace_cta = atoi(getenv("RP_XL_DQ_TRACE"));
    q.trace = trace;
  }
  xl_attn_bwd_dq_kernel<<<(unsigned)grid, kThreadsBwd, kDqSmem, st>>>(mg, mv, mk, mr, mbd, mac, mp, q);
  if (tr) {
    unsigned long long h[11 * 32];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const unsigned long long t0 = h[0];
    static const char* names[11] = {"start", "P:P", "M:dsrdy", "M:vfull", "S:prolog", "S:pfull", "S:acc",
                                    "S:ring", "S:stored", "S:ds", "S:epi"};
    for (int ev = 0; ev < 11; ++ev) {
      fprintf(stderr, "%-9s", names[ev]);
      for (int i = 0; i < 12; ++i) fprintf(stderr, " %6.2f", h[ev * 32 + i] ? (h[ev * 32 + i] - t0) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
  return check_launch("xl_attn_bwd_dq");
}

int xl_attn_bwd_kv(const void* gctx_h, const void* vh, const void* qu, const void* probs, int64_t ldp,
                   const float* d_rows, void* gk, void* gv, int64_t B, int64_t Tn, int64_t M, int H, int dh, int mem_len,
                   float scale, cudaStream_t st, void* gqkv) {
  if (dh != 64) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_kv: head dim must be 64 (got %d)", dh);
  if (Tn % 128 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_kv: T must be a multiple of 128");
  const int64_t Kl = M + Tn, HB = (int64_t)H * B;
  if (ldp < Kl || ldp % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_kv: ldp must be >= M+T, multiple of 8");
  if (mem_len < 0 || mem_len > M) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_kv: mem_len out of range");
  if (!d_rows || (!gqkv && (!gk || !gv))) return set_error(RP_ERR_INVALID, "xl_attn_bwd_kv: null output or D rows");
  for (const void* q : {probs, gctx_h, vh, qu, gqkv ? gqkv : (const void*)gk, gqkv ? gqkv : (const void*)gv})
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_kv: unaligned operand");
  CUtensorMap mg, mv, mu, mp;
  RP_TRY0(tma_map_bf16(&mp, probs, ldp, Tn, ldp, HB, Tn * ldp, 64, kQT));
  RP_TRY0(tma_map_bf16(&mg, gctx_h, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mv, vh, dh, Kl, dh, HB, Kl * dh, 64, kKT));
  RP_TRY0(tma_map_bf16(&mu, qu, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  static uint64_t attr_done = 0;
  if (first_on_device(attr_done))
    cudaFuncSetAttribute(xl_attn_bwd_kv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kKvSmem);
  KvParams p{};
  p.D = d_rows;
  p.gk = static_cast<__nv_bfloat16*>(gk);
  p.gv = static_cast<__nv_bfloat16*>(gv);
  p.T = (int)Tn;
  p.M = (int)M;
  p.Kl = (int)Kl;
  p.lo = (int)(M - mem_len);
  p.nkt = (int)((Kl + kKT - 1) / kKT);
  p.HB = (int)HB;
  p.scale = scale;
  p.gqkv = static_cast<__nv_bfloat16*>(gqkv);
  p.B = (int)B;
  p.d = H * dh;
  if (gqkv && B * M > 0) {
    // the memory rows carry no query gradient: zero their query columns
    if (cudaMemset2DAsync(gqkv, (size_t)3 * p.d * 2, 0, (size_t)p.d * 2, (size_t)(B * M), st) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "xl_attn_bwd_kv: memset of the memory rows' query gradient");
  }
  const int64_t items = HB * p.nkt;
  if (items <= 0) return RP_OK;
  if (items >= (1LL << 31)) return set_error(RP_ERR_DIMENSION, "xl_attn_bwd_kv: too many key tiles");
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (sms[dev & 63] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev & 63] = v > 0 ? v : 148;
  }
  int64_t grid = std::min<int64_t>(items, sms[dev & 63]);  // persistent: one CTA per SM
  if (const char* e = getenv("RP_XL_KV_CTAS"))  // tests: fewer CTAs, several items each
    if (atoi(e) > 0) grid = std::min<int64_t>(grid, atoi(e));
  static unsigned long long* trace = nullptr;
  const bool tr = getenv("RP_XL_KV_TRACE") != nullptr;
  if (tr) {
    if (!trace) cudaMalloc(&trace, 31 * 64 * 8);
    cudaMemsetAsync(trace, 0, 31 * 64 * 8, st);
    p.trace = trace;
  }
  xl_attn_bwd_kv_kernel<<<(unsigned)grid, kKvThreads, kKvSmem, st>>>(mg, mv, mu, mp, p);
  if (tr) {
    unsigned long long h[31 * 64];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < 31 * 64; ++i)
      if (h[i] && h[i] < t0) t0 = h[i];
    static const char* names[15] = {"P:G", "P:P", "P:U", "M:dsrdy", "M:ufull", "M:accE", "M:gfull", "M:pfull",
                                    "S:pfull", "S:acc", "S:afree", "S:ds", "S:epiW", "S:epiGo", "S:epiDone"};
    for (int ev = 0; ev < 31; ++ev) {
      fprintf(stderr, "%-9s", ev < 15 ? names[ev] : "S:w");
      for (int i = 0; i < 40; ++i) fprintf(stderr, " %6.2f", h[ev * 64 + i] ? (h[ev * 64 + i] - t0) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
  return check_launch("xl_attn_bwd_kv");
}

int xl_attn_fwd_pv(const void* qu, const void* qv, const void* kh, const void* vh, const void* rh, void* probs,
                   int64_t ldp, void* ctx, int64_t B, int64_t Tn, int64_t M, int H, int dh, int mem_len, float scale,
                   cudaStream_t st, int dh_out, int64_t ld_ctx) {
  if (dh != 64) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd_pv: head dim must be 64 (got %d)", dh);
  if (dh_out <= 0) dh_out = dh;
  if (ld_ctx <= 0) ld_ctx = (int64_t)H * dh_out;
  if (dh_out > 64 || ld_ctx < (int64_t)H * dh_out)
    return set_error(RP_ERR_DIMENSION, "xl_attn_fwd_pv: output head dim <= 64, ctx pitch >= H * dh_out");
  const int64_t Kl = M + Tn, HB = (int64_t)H * B;
  if (ldp < Kl || ldp % 8 != 0) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd_pv: ldp must be >= M+T, multiple of 8");
  if (mem_len < 0 || mem_len > M) return set_error(RP_ERR_DIMENSION, "xl_attn_fwd_pv: mem_len out of range");
  if ((reinterpret_cast<uintptr_t>(probs) & 15) != 0 || (reinterpret_cast<uintptr_t>(ctx) & 1) != 0)
    return set_error(RP_ERR_DIMENSION, "xl_attn_fwd_pv: unaligned operand");
  CUtensorMap mqu, mqv, mk, mr, mv, mp;
  RP_TRY0(tma_map_bf16(&mqu, qu, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mqv, qv, dh, Tn, dh, HB, Tn * dh, 64, kQT));
  RP_TRY0(tma_map_bf16(&mk, kh, dh, Kl, dh, HB, Kl * dh, 64, kFKT));
  RP_TRY0(tma_map_bf16(&mr, rh, dh, Kl, dh, H, Kl * dh, 64, kFBand));
  RP_TRY0(tma_map_bf16(&mv, vh, dh, Kl, dh, HB, Kl * dh, 64, kFKT));
  RP_TRY0(tma_map_bf16(&mp, probs, ldp, Tn, ldp, HB, Tn * ldp, 64, 32));
  // RP_XL_PV_BUF: 1 = one P / V tile and three K + R stages; 2 = double-buffered P / V, two stages
  static const int pv_buf = getenv("RP_XL_PV_BUF") ? atoi(getenv("RP_XL_PV_BUF")) : 2;
  static uint64_t attr_done = 0;
  if (first_on_device(attr_done)) {
    cudaFuncSetAttribute(xl_attn_fwd_pv_kernel<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_pv_smem<3, 1>());
    cudaFuncSetAttribute(xl_attn_fwd_pv_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_pv_smem<2, 2>());
  }
  FwdPvParams pp{};
  FwdParams& p = pp.f;
  p.p = static_cast<__nv_bfloat16*>(probs);
  p.ldp = ldp;
  p.B = (int)B;
  p.T = (int)Tn;
  p.M = (int)M;
  p.Kl = (int)Kl;
  p.lo = (int)(M - mem_len);
  p.nqt = (int)((Tn + kQT - 1) / kQT);
  p.heavy_first = xl_heavy_first();
  p.c2 = scale * 1.4426950408889634f;
  p.dbg = 0;
  pp.ctx = static_cast<__nv_bfloat16*>(ctx);
  pp.d = H * dh;
  pp.dh_out = dh_out;
  pp.ld_ctx = ld_ctx;
  const int64_t grid = HB * p.nqt;
  if (grid <= 0) return RP_OK;
  if (pv_buf == 1)
    xl_attn_fwd_pv_kernel<3, 1><<<(unsigned)grid, kThreadsFwd, fwd_pv_smem<3, 1>(), st>>>(mqu, mqv, mk, mr, mv, mp, pp);
  else
    xl_attn_fwd_pv_kernel<2, 2><<<(unsigned)grid, kThreadsFwd, fwd_pv_smem<2, 2>(), st>>>(mqu, mqv, mk, mr, mv, mp, pp);
  return check_launch("xl_attn_fwd_pv");
}

}  // namespace rp
