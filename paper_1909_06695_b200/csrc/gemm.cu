// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
// Replaces the reference's fixed-order fp64 contractions `kernels.mm` /
// `kernels.bmm` (reference pkg/src/ringpipe/kernels.py:23-48, 68-81) for every
// dense contraction of the block (layers.py:176-195, 218-247) and the tied head
// (layers.py:269, 310-321).
//
//   C[b](M x N) = epilogue( alpha * A[b](M x K) * B[b](K x N) )
//
// A is K-major ([M,K] row-major) or MN-major ([K,M] row-major); B is K-major
// ([N,K] row-major) or MN-major ([K,N] row-major).  Operands are staged by TMA
// into 128B-swizzled shared memory, one elected thread issues tcgen05.mma into
// a double-buffered TMEM accumulator, and four epilogue warps drain TMEM with
// tcgen05.ld and apply the fused epilogue (bias/ReLU, bias/dropout/residual,
// logsumexp partials for the tied-vocab cross-entropy, or the softmax-CE
// gradient dz).  "tf32x3" runs three accumulation passes (hi*hi + hi*lo +
// lo*hi) over pre-split operands to reach fp32 accuracy on the tf32 pipe.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "rp_internal.h"

namespace rp {

template <bool kTf32, int BN_, int kCta_ = 1>
struct GemmCfg {
  static constexpr int kCta = kCta_;       // 2: CTA pair shares one 256-row tile (cta_group::2)
  static constexpr int BM = 128;           // rows of A / D per CTA
  static constexpr int BM_TILE = 128 * kCta;
  static constexpr int BN = BN_;
  static constexpr int B_ROWS = BN / kCta;  // N rows of B staged per CTA
  static constexpr int ELEM = kTf32 ? 4 : 2;
  static constexpr int BK = 128 / ELEM;     // one 128-byte swizzle row of K
  static constexpr int UK = kTf32 ? 8 : 16;  // K per tcgen05.mma
  static constexpr int CHUNK = 128 / ELEM;  // MN elements per 128B chunk (MN-major)
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = B_ROWS * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // 192 KB of operand stages in flight per SM (measured: 5 stages of a CTA
  // pair starve the long-K head GEMMs more than a second store tile helps)
  static constexpr int PIPE_BYTES = 196608;
  static constexpr int STAGES = (PIPE_BYTES / STAGE_BYTES) > 8 ? 8 : (PIPE_BYTES / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN < 32) ? 32 : 2 * BN;
  static constexpr int OUT_BUFS = 1;  // per-warp TMA-store tiles (2 costs a pipeline stage: measured slower)
  static constexpr int STAGE_OUT = OUT_BUFS * 8 * 32 * 64;  // per-warp 32x32 bf16 staging tiles (TMA store)
  static constexpr int STAGE_IN = 8 * 32 * 64;   // per-warp 32x32 bf16 residual tiles (TMA load); LSE reuses it
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGE_OUT + STAGE_IN + 1024 + 256;
};

struct GemmParams {
  int M, N, K, batch;
  int a_mn, b_mn, passes;
  int m_tiles, n_tiles, num_tiles, kb_per_pass;
  int out_bf16, epi;
  float alpha;
  void* C;
  int64_t ldc, stride_c;
  const float* bias;
  const void* resid;
  int64_t ld_resid, stride_resid;
  uint64_t drop_seed, drop_thr, drop_pos0;
  float drop_scale;
  int drop_on;
  const int64_t* targets;
  const float* lse;
  float* partial;
  float* target_logit;
  float ce_scale;
  int vec_ok;
  int vec2_ok;  // fp32 C with 8-byte aligned rows (an even pitch: d 410): float2 stores
  int resid_vec;
  int ksplit;  // > 0: unit b is split b / bsz of matrix b % bsz, K range [split*ksplit, (split+1)*ksplit)
  int bsz;     // matrices in the batch (the split-K partials are laid out [split][matrix])
  int n_fast;  // raster: N tiles fastest
  int tma_store;  // bf16 C written by TMA bulk stores from a swizzled smem tile
  int tma_resid;  // bf16 residual / aux read by TMA bulk loads into a swizzled smem tile
  int k_lo_sign;  // banded A: row m is zero for k < m + k_lo_off (sign +1); 0 = dense
  int k_lo_off;
};

// First k-block of a tile's K loop: a banded A skips the leading all-zero
// k-blocks of the tile's first row (the same range for producer and MMA)
template <int BM_TILE, int BK>
__device__ __forceinline__ int tile_kb_lo(const GemmParams& p, int mb) {
  if (p.k_lo_sign <= 0) return 0;
  const int k = mb * BM_TILE + p.k_lo_off;
  const int kb = k > 0 ? k / BK : 0;
  return kb < p.kb_per_pass ? kb : p.kb_per_pass - 1;
}

__device__ __forceinline__ void store_chunk(const GemmParams& p, int64_t m, int n0, int b,
                                            const float (&v)[32]) {
  const int64_t base = (int64_t)b * p.stride_c + m * p.ldc + n0;
  if (p.vec_ok && n0 + 32 <= p.N) {
    if (p.out_bf16) {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.C) + base);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 t = __floats2bfloat162_rn(v[q * 8 + 2 * h], v[q * 8 + 2 * h + 1]);
          w[h] = *reinterpret_cast<uint32_t*>(&t);
        }
        dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else {
      float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.C) + base);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  } else if (p.vec2_ok && n0 + 32 <= p.N) {
    float2* dst = reinterpret_cast<float2*>(reinterpret_cast<float*>(p.C) + base);
#pragma unroll
    for (int q = 0; q < 16; ++q) dst[q] = make_float2(v[2 * q], v[2 * q + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (n0 + j < p.N) {
        if (p.out_bf16)
          reinterpret_cast<__nv_bfloat16*>(p.C)[base + j] = __float2bfloat16_rn(v[j]);
        else
          reinterpret_cast<float*>(p.C)[base + j] = v[j];
      }
    }
  }
}

// 32 consecutive residual / aux elements of row m (same dtype as C), vectorised
// when the row chunk is in bounds and 16-byte aligned.
__device__ __forceinline__ void load_chunk(const GemmParams& p, int64_t m, int n0, int b, float (&r)[32]) {
  const int64_t base = (int64_t)b * p.stride_resid + m * p.ld_resid + n0;
  if (p.resid_vec && n0 + 32 <= p.N) {
    if (p.out_bf16) {
      const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.resid) + base);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = src[q];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const __nv_bfloat162 t = *reinterpret_cast<const __nv_bfloat162*>(&w[h]);
          const float2 f = __bfloat1622float2(t);
          r[q * 8 + 2 * h] = f.x;
          r[q * 8 + 2 * h + 1] = f.y;
        }
      }
    } else {
      const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.resid) + base);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = src[q];
        r[4 * q] = f.x;
        r[4 * q + 1] = f.y;
        r[4 * q + 2] = f.z;
        r[4 * q + 3] = f.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      r[j] = (n0 + j < p.N) ? (p.out_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.resid)[base + j])
                                          : reinterpret_cast<const float*>(p.resid)[base + j])
                            : 0.f;
  }
}

// Raw bf16 bits of 32 consecutive residual / aux elements (4 x 16B), issued
// one chunk ahead so the load latency hides behind the current chunk's math.
__device__ __forceinline__ void fetch_raw_bf16(const GemmParams& p, int64_t m, int n0, int b, uint4 (&raw)[4]) {
  const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.resid) +
                                                    ((int64_t)b * p.stride_resid + m * p.ld_resid + n0));
#pragma unroll
  for (int q = 0; q < 4; ++q) raw[q] = src[q];
}
__device__ __forceinline__ void unpack_raw_bf16(const uint4 (&raw)[4], float (&r)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t w[4] = {raw[q].x, raw[q].y, raw[q].z, raw[q].w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
      r[q * 8 + 2 * h] = f.x;
      r[q * 8 + 2 * h + 1] = f.y;
    }
  }
}
// 32 bias values as 8 broadcast float4 loads (or scalar at the ragged edge)
__device__ __forceinline__ void load_bias(const GemmParams& p, int n0, bool full, float (&bb)[32]) {
  if (!p.bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j) bb[j] = 0.f;
  } else if (full && (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0) {
    const float4* s = reinterpret_cast<const float4*>(p.bias + n0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 f = s[q];
      bb[4 * q] = f.x;
      bb[4 * q + 1] = f.y;
      bb[4 * q + 2] = f.z;
      bb[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) bb[j] = (n0 + j < p.N) ? p.bias[n0 + j] : 0.f;
  }
}

__device__ __forceinline__ float fast_exp2(float x) {
#if defined(RP_EXP_EXPERIMENT) && RP_EXP_EXPERIMENT == 1
  return x * 0.5f + 1.0f;  // diagnostic only: no MUFU
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

// One warp's 32x32 bf16 chunk (lane = row) -> 64B-swizzled smem tile -> one
// TMA bulk store.  The swizzle (16B chunk k of row r at k ^ ((r>>1)&3)) matches
// CU_TENSOR_MAP_SWIZZLE_64B and keeps the st.shared at 4 wavefronts.
template <int kBufs>
__device__ __forceinline__ void emit_tma(const CUtensorMap& mapC, uint8_t* tile, const float (&v)[32], int lane,
                                         int col0, int row0) {
  // the store that last used this tile (kBufs emits ago) finished reading smem
  if (lane == 0) {
    if constexpr (kBufs == 2)
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else
      tma_store_wait_read();
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      __nv_bfloat162 t = __floats2bfloat162_rn(v[k * 8 + 2 * h], v[k * 8 + 2 * h + 1]);
      w[h] = *reinterpret_cast<uint32_t*>(&t);
    }
    const int off = lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4);
    *reinterpret_cast<uint4*>(tile + off) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) tma_store_2d(&mapC, tile, col0, row0);
}

// Tile raster: the dimension with fewer tiles runs fastest, so consecutive
// CTAs share the operand along the other dimension (L2 reuse instead of a
// second DRAM stream).  The batch / split-K index is slowest.
__device__ __forceinline__ void decode_tile(const GemmParams& p, int tile, int& mb, int& nb, int& b) {
  if (p.n_fast) {
    nb = tile % p.n_tiles;
    const int rest = tile / p.n_tiles;
    mb = rest % p.m_tiles;
    b = rest / p.m_tiles;
  } else {
    mb = tile % p.m_tiles;
    const int rest = tile / p.m_tiles;
    nb = rest % p.n_tiles;
    b = rest / p.n_tiles;
  }
}

template <bool kTf32, int BN, int kCta>
__global__ void __launch_bounds__(384, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA_lo,
                const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapB_lo,
                const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapR,
                const GemmParams p) {
  using Cfg = GemmCfg<kTf32, BN, kCta>;
  static_assert(kCta == 1 || !kTf32, "CTA-pair mode is bf16 only");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t* stage_out = smem + Cfg::STAGES * Cfg::STAGE_BYTES;  // 1024-aligned
  uint8_t* stage_in = stage_out + Cfg::STAGE_OUT;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_in + Cfg::STAGE_IN);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* in_bar = tmem_empty + 2;  // [8] per epilogue warp: residual tile landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(in_bar + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = kCta == 2 ? cluster_rank() : 0;  // CTA rank within the pair
  const bool leader = crank == 0;
  const int tile0 = blockIdx.x / kCta, tstep = gridDim.x / kCta;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    if (p.passes > 1) {
      tma_prefetch(&mapA_lo);
      tma_prefetch(&mapB_lo);
    }
    if (p.tma_store) tma_prefetch(&mapC);
    if (p.tma_resid) tma_prefetch(&mapR);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      // 1 CTA: every epilogue thread arrives; pair: one arrival per epilogue
      // warp of both CTAs, on the leader's barrier
      mbar_init(&tmem_empty[a], kCta == 2 ? 16 : 256);
    }
    for (int w = 0; w < 8; ++w) mbar_init(&in_bar[w], 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (kCta == 2)
      tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
    else
      tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCta == 2) cluster_sync();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // alloc, descriptor prefetch) overlapped the previous kernel's tail; wait
  // for its results before touching global memory, and let the next kernel
  // start its own prologue as our CTAs retire.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t stage = 0, phase = 0;
      for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
        int mb, nb, b;
        decode_tile(p, tile, mb, nb, b);
        const int m0 = mb * Cfg::BM_TILE + crank * Cfg::BM, n0 = nb * BN + crank * Cfg::B_ROWS;
        const int kbase = p.ksplit ? (b / p.bsz) * p.ksplit : 0;
        const int bc = p.ksplit ? b % p.bsz : b;
        const int kb_lo = tile_kb_lo<Cfg::BM_TILE, Cfg::BK>(p, mb);
        for (int pass = 0; pass < p.passes; ++pass) {
          const CUtensorMap* ma = (pass == 2) ? &mapA_lo : &mapA;
          const CUtensorMap* mbm = (pass == 1) ? &mapB_lo : &mapB;
          for (int kb = kb_lo; kb < p.kb_per_pass; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
            uint8_t* sb = sa + Cfg::A_BYTES;
            const int k0 = kbase + kb * Cfg::BK;
            if constexpr (kCta == 2) {
              // both CTAs' bytes complete on the leader's barrier
              const uint32_t fb = leader_addr(&full[stage]);
              if (leader) mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
              if (!p.a_mn) {
                tma_load_3d_pair(sa, ma, fb, k0, m0, bc);
              } else {
#pragma unroll
                for (int c = 0; c < Cfg::BM / Cfg::CHUNK; ++c)
                  tma_load_3d_pair(sa + c * (Cfg::BK * 128), ma, fb, m0 + c * Cfg::CHUNK, k0, bc);
              }
              if (!p.b_mn) {
                tma_load_3d_pair(sb, mbm, fb, k0, n0, bc);
              } else {
#pragma unroll
                for (int c = 0; c < Cfg::B_ROWS / Cfg::CHUNK; ++c)
                  tma_load_3d_pair(sb + c * (Cfg::BK * 128), mbm, fb, n0 + c * Cfg::CHUNK, k0, bc);
              }
            } else {
              mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
              if (!p.a_mn) {
                tma_load_3d(sa, ma, &full[stage], k0, m0, bc);
              } else {
#pragma unroll
                for (int c = 0; c < Cfg::BM / Cfg::CHUNK; ++c)
                  tma_load_3d(sa + c * (Cfg::BK * 128), ma, &full[stage], m0 + c * Cfg::CHUNK, k0, bc);
              }
              if (!p.b_mn) {
                tma_load_3d(sb, mbm, &full[stage], k0, n0, bc);
              } else {
#pragma unroll
                for (int c = 0; c < BN / Cfg::CHUNK; ++c)
                  tma_load_3d(sb + c * (Cfg::BK * 128), mbm, &full[stage], n0 + c * Cfg::CHUNK, k0, bc);
              }
            }
            if (++stage == Cfg::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (single thread; the pair's leader) ----------------
      const uint32_t idesc = umma_idesc(kTf32, p.a_mn, p.b_mn, Cfg::BM_TILE, BN);
      const uint32_t a_lbo = p.a_mn ? Cfg::BK * 128 : 16;
      const uint32_t b_lbo = p.b_mn ? Cfg::BK * 128 : 16;
      const uint32_t a_step = p.a_mn ? Cfg::UK * 128 : 32;
      const uint32_t b_step = p.b_mn ? Cfg::UK * 128 : 32;
      // tf32 MN-major tiles are 128B-swizzled with 32B atoms (4 K-rows per atom)
      const uint32_t a_lay = (kTf32 && p.a_mn) ? 1u : 2u, b_lay = (kTf32 && p.b_mn) ? 1u : 2u;
      const uint32_t a_sbo = (kTf32 && p.a_mn) ? 512u : 1024u, b_sbo = (kTf32 && p.b_mn) ? 512u : 1024u;
      uint32_t stage = 0, phase = 0;
      int local = 0;
      for (int tile = tile0; tile < p.num_tiles; tile += tstep, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int mb_, nb_, b_;
        decode_tile(p, tile, mb_, nb_, b_);
        const int kb_lo = tile_kb_lo<Cfg::BM_TILE, Cfg::BK>(p, mb_);
        for (int pass = 0; pass < p.passes; ++pass) {
          for (int kb = kb_lo; kb < p.kb_per_pass; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
              const uint64_t ad = umma_desc(sa + k * a_step, a_lbo, a_sbo, a_lay);
              const uint64_t bd = umma_desc(sb + k * b_step, b_lbo, b_sbo, b_lay);
              if constexpr (kCta == 2)
                tc_mma_pair(d_tmem, ad, bd, idesc, (pass | (kb - kb_lo) | k) != 0 ? 1u : 0u);
              else
                tc_mma<kTf32>(d_tmem, ad, bd, idesc, (pass | (kb - kb_lo) | k) != 0 ? 1u : 0u);
            }
            if constexpr (kCta == 2)
              tc_commit_pair(&empty[stage]);
            else
              tc_commit(&empty[stage]);
            if (++stage == Cfg::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        if constexpr (kCta == 2)
          tc_commit_pair(&tmem_full[acc]);
        else
          tc_commit(&tmem_full[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 8 warps, two per TMEM lane quarter ----------------
    // warp w may only touch TMEM lanes 32*(w%4)..+31; the two warps of a quarter
    // split the tile's columns in halves.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    constexpr int kHalf = BN / 64;  // 32-column chunks per half
    uint8_t* my_out_base = stage_out + (warp - 4) * 2048 * Cfg::OUT_BUFS;  // 32 rows x 64 B, 64B-swizzled
    int out_buf = 0;
    uint8_t* my_in = stage_in + (warp - 4) * 2048;          // residual / aux tile, same layout
    uint64_t* my_bar = &in_bar[warp - 4];
    uint32_t in_phase = 0;
    const float kLog2e = 1.4426950408889634f;
    int local = 0;
    for (int tile = tile0; tile < p.num_tiles; tile += tstep, ++local) {
      int mb, nb, b;
      decode_tile(p, tile, mb, nb, b);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int64_t mrow0 = (int64_t)mb * Cfg::BM_TILE + crank * Cfg::BM;  // this CTA's first row
      const int64_t m = mrow0 + q * 32 + lane;
      const bool row_ok = m < p.M;
      const int64_t grow = (int64_t)b * p.M + m;  // row index over the folded batch
      const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);

      float run_max = -INFINITY, run_sum = 0.f;
      int64_t tgt = -1;
      float lse2 = 0.f;  // lse*log2e - log2(ce_scale)
      if (row_ok && (p.epi == RP_EPI_LSE_PARTIAL || p.epi == RP_EPI_CE_GRAD)) {
        tgt = p.targets[grow];
        if (p.epi == RP_EPI_CE_GRAD) lse2 = p.lse[grow] * kLog2e - __log2f(p.ce_scale);
      }
      // epilogues without an aux input (store, bias+ReLU, CE gradient; bf16
      // math): the TMEM load of the next 32-column chunk is in flight while
      // this chunk is processed and stored -- the epilogue is latency-bound
      // at two warps per SM sub-partition (measured: CE pass 2.24 -> 1.82 ms
      // at C2; the LSE pass did not gain and keeps the generic loop)
      bool head_fast = false;
#ifndef RP_HEAD_FAST_OFF
#define RP_HEAD_FAST_OFF 0
#endif
#ifndef RP_LSE_FAST_OFF
#define RP_LSE_FAST_OFF 0
#endif
      if constexpr (!kTf32 && kHalf % 2 == 0 && !RP_HEAD_FAST_OFF) {
        const bool no_aux = p.epi == RP_EPI_CE_GRAD || p.epi == RP_EPI_STORE || p.epi == RP_EPI_BIAS_RELU;
        if (no_aux && (p.tma_store || p.epi != RP_EPI_CE_GRAD)) {
          head_fast = true;
          const int trow = (int)((int64_t)b * p.M + mrow0 + q * 32);
          auto chunk = [&](const uint32_t (&r)[32], int c) {
            const int n0 = nb * BN + c * 32;
            if (n0 >= p.N) return;  // warp-uniform
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            const bool full = n0 + 32 <= p.N;
            if (!row_ok) {
              if (p.tma_store) {  // rows past M: zeros, clipped by the TMA store
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0.f;
                emit_tma<Cfg::OUT_BUFS>(mapC, my_out_base, v, lane, n0, trow);
              }
              return;
            }
            if (p.epi == RP_EPI_CE_GRAD) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = fast_exp2(fmaf(v[j], kLog2e, -lse2));
              if ((uint64_t)(tgt - n0) < 32ull) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (tgt == n0 + j) v[j] -= p.ce_scale;
              }
            } else if (p.epi == RP_EPI_BIAS_RELU) {
              float bb[32];
              load_bias(p, n0, full, bb);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = fmaxf(fmaf(v[j], p.alpha, bb[j]), 0.f);
            } else if (p.alpha != 1.f) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
            }
            if (p.tma_store)
              emit_tma<Cfg::OUT_BUFS>(mapC, my_out_base, v, lane, n0, trow);
            else
              store_chunk(p, m, n0, b, v);
          };
          const int c0 = half * kHalf;
          uint32_t ra[32], rb[32];
          tmem_ld32_async(t_row + c0 * 32, ra);
          tmem_wait_ld(ra);
#pragma unroll 1
          for (int cc = 0; cc < kHalf; cc += 2) {
            tmem_ld32_async(t_row + (c0 + cc + 1) * 32, rb);
            chunk(ra, c0 + cc);
            tmem_wait_ld(rb);
            if (cc + 2 < kHalf) tmem_ld32_async(t_row + (c0 + cc + 2) * 32, ra);
            chunk(rb, c0 + cc + 1);
            if (cc + 2 < kHalf) tmem_wait_ld(ra);
          }
        } else if (p.epi == RP_EPI_LSE_PARTIAL && !RP_LSE_FAST_OFF) {
          // online log-sum-exp over this half's columns, next TMEM chunk in
          // flight; no per-chunk epilogue dispatch.  Same operation order as
          // the generic loop (bitwise equal): columns past N enter as -inf.
          head_fast = true;
          auto lse_chunk = [&](const uint32_t (&r)[32], int c) {
            const int n0 = nb * BN + c * 32;
            if (n0 >= p.N || !row_ok) return;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if (n0 + 32 > p.N) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j >= p.N) v[j] = -INFINITY;
            }
            float cm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int j = 0; j < 32; ++j) cm[j & 3] = fmaxf(cm[j & 3], v[j]);
            const float nmax = fmaxf(run_max, fmaxf(fmaxf(cm[0], cm[1]), fmaxf(cm[2], cm[3])));
            const float nm2 = nmax * kLog2e;
            float s[4] = {run_sum * fast_exp2(run_max * kLog2e - nm2), 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 32; ++j) s[j & 3] += fast_exp2(fmaf(v[j], kLog2e, -nm2));
            run_max = nmax;
            run_sum = (s[0] + s[1]) + (s[2] + s[3]);
            if ((uint64_t)(tgt - n0) < 32ull) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (tgt == n0 + j) p.target_logit[grow] = v[j];
            }
          };
          const int c0 = half * kHalf;
          uint32_t ra[32], rb[32];
          tmem_ld32_async(t_row + c0 * 32, ra);
          tmem_wait_ld(ra);
#pragma unroll 1
          for (int cc = 0; cc < kHalf; cc += 2) {
            tmem_ld32_async(t_row + (c0 + cc + 1) * 32, rb);
            lse_chunk(ra, c0 + cc);
            tmem_wait_ld(rb);
            if (cc + 2 < kHalf) tmem_ld32_async(t_row + (c0 + cc + 2) * 32, ra);
            lse_chunk(rb, c0 + cc + 1);
            if (cc + 2 < kHalf) tmem_wait_ld(ra);
          }
        }
      }
      if (!head_fast) {
      // residual / aux: TMA bulk-loads one 32x32 tile per warp, one chunk
      // ahead (coalesced), else per-row loads prefetched one chunk ahead
      const bool uses_aux = p.epi == RP_EPI_RELU_GRAD || p.epi == RP_EPI_GELU_GRAD ||
                            (p.epi == RP_EPI_BIAS_DROPOUT_RESIDUAL && p.resid);
      const bool tma_aux = uses_aux && p.tma_resid;
      const bool aux = !tma_aux && uses_aux && p.out_bf16 && p.resid_vec;
      const int trow0 = (int)((int64_t)b * p.M + mrow0 + q * 32);
      uint4 nxt[4];
      bool nxt_ok = false;
      {
        const int nf = nb * BN + half * kHalf * 32;
        if (tma_aux && nf < p.N && lane == 0) {
          mbar_expect_tx(my_bar, 2048);
          tma_load_2d(my_in, &mapR, my_bar, nf, trow0);
        }
        if (aux && row_ok && nf + 32 <= p.N) {
          fetch_raw_bf16(p, m, nf, b, nxt);
          nxt_ok = true;
        }
      }
#pragma unroll 1
      for (int cc = 0; cc < kHalf; ++cc) {
        const int c = half * kHalf + cc;
        const int n0 = nb * BN + c * 32;
        uint4 cur[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
        bool cur_ok = nxt_ok;
        nxt_ok = false;
        if (tma_aux && n0 < p.N) {
          // tile c landed: copy this lane's row (64B-swizzled) to registers,
          // then reuse the buffer for tile c+1
          mbar_wait(my_bar, in_phase);
          in_phase ^= 1;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            cur[k] = *reinterpret_cast<const uint4*>(my_in + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4));
          cur_ok = true;
          __syncwarp();
          if (lane == 0 && cc + 1 < kHalf && n0 + 32 < p.N) {
            mbar_expect_tx(my_bar, 2048);
            tma_load_2d(my_in, &mapR, my_bar, n0 + 32, trow0);
          }
        }
        if (aux && row_ok && cc + 1 < kHalf && n0 + 64 <= p.N) {
          fetch_raw_bf16(p, m, n0 + 32, b, nxt);
          nxt_ok = true;
        }
        uint32_t r[32];
        tmem_ld32(t_row + c * 32, r);
        if (n0 >= p.N) continue;  // warp-uniform
        if (!row_ok) {
          // rows past M: the TMA store clips them, but the warp must still
          // take part in the cooperative smem tile
          if (p.tma_store && p.epi != RP_EPI_LSE_PARTIAL) {
            float z[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) z[j] = 0.f;
            emit_tma<Cfg::OUT_BUFS>(mapC, my_out_base + out_buf * 2048, z, lane, n0,
                                    (int)((int64_t)b * p.M + mrow0 + q * 32));
            out_buf ^= (Cfg::OUT_BUFS - 1);
          }
          continue;
        }
        const bool full = n0 + 32 <= p.N;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const int trow = trow0;
#define RP_EMIT()                                                                   \
  do {                                                                              \
    if (p.tma_store) {                                                              \
      emit_tma<Cfg::OUT_BUFS>(mapC, my_out_base + out_buf * 2048, v, lane, n0, trow); \
      out_buf ^= (Cfg::OUT_BUFS - 1);                                               \
    } else {                                                                        \
      store_chunk(p, m, n0, b, v);                                                  \
    }                                                                               \
  } while (0)
        switch (p.epi) {
          case RP_EPI_STORE:
            if (p.alpha != 1.f) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
            }
            RP_EMIT();
            break;
          case RP_EPI_BIAS_RELU: {
            float bb[32];
            load_bias(p, n0, full, bb);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fmaxf(fmaf(v[j], p.alpha, bb[j]), 0.f);
            RP_EMIT();
            break;
          }
          case RP_EPI_BIAS_DROPOUT_RESIDUAL: {
            float rr[32], bb[32];
            if (cur_ok) {
              unpack_raw_bf16(cur, rr);
            } else if (p.resid) {
              load_chunk(p, m, n0, b, rr);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) rr[j] = 0.f;
            }
            load_bias(p, n0, full, bb);
            const uint64_t pos_row = p.drop_pos0 + (uint64_t)grow * (uint64_t)p.N + (uint64_t)n0;
            const uint64_t z0 = dropout_z(p.drop_seed, pos_row);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float t = fmaf(v[j], p.alpha, bb[j]);
              if (p.drop_on) t = dropout_keep_z(z0 + (uint64_t)j * kGolden, p.drop_thr) ? t * p.drop_scale : 0.f;
              v[j] = t + rr[j];
            }
            RP_EMIT();
            break;
          }
          case RP_EPI_LSE_PARTIAL: {
            float cm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            if (full) {
#pragma unroll
              for (int j = 0; j < 32; ++j) cm[j & 3] = fmaxf(cm[j & 3], v[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < p.N) cm[j & 3] = fmaxf(cm[j & 3], v[j]);
            }
            const float nmax = fmaxf(run_max, fmaxf(fmaxf(cm[0], cm[1]), fmaxf(cm[2], cm[3])));
            const float nm2 = nmax * kLog2e;
            float s[4] = {run_sum * fast_exp2(run_max * kLog2e - nm2), 0.f, 0.f, 0.f};
            if (full) {
#pragma unroll
              for (int j = 0; j < 32; ++j) s[j & 3] += fast_exp2(fmaf(v[j], kLog2e, -nm2));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < p.N) s[j & 3] += fast_exp2(fmaf(v[j], kLog2e, -nm2));
            }
            run_max = nmax;
            run_sum = (s[0] + s[1]) + (s[2] + s[3]);
            if ((uint64_t)(tgt - n0) < 32ull) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (tgt == n0 + j) p.target_logit[grow] = v[j];
            }
            break;
          }
          case RP_EPI_RELU_GRAD: {
            // out = acc * (aux > 0), aux = the ReLU output h1 (layers.py:221)
            float rr[32];
            if (cur_ok)
              unpack_raw_bf16(cur, rr);
            else
              load_chunk(p, m, n0, b, rr);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = rr[j] > 0.f ? v[j] * p.alpha : 0.f;
            RP_EMIT();
            break;
          }
          case RP_EPI_GELU_GRAD: {
            // out = acc * gelu'(z1), gelu'(z) = Phi(z) + z phi(z), aux = the pre-activation z1
            float rr[32];
            if (cur_ok)
              unpack_raw_bf16(cur, rr);
            else
              load_chunk(p, m, n0, b, rr);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float z = rr[j];
              const float cdf = 0.5f * (1.f + erff(z * 0.70710678118654752f));
              const float pdf = 0.39894228040143268f * __expf(-0.5f * z * z);
              v[j] = v[j] * p.alpha * fmaf(z, pdf, cdf);
            }
            RP_EMIT();
            break;
          }
          case RP_EPI_CE_GRAD: {
            // dz = softmax * scale - onehot * scale, scale folded into the exponent
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fast_exp2(fmaf(v[j], kLog2e, -lse2));
            if ((uint64_t)(tgt - n0) < 32ull) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (tgt == n0 + j) v[j] -= p.ce_scale;
            }
            RP_EMIT();
            break;
          }
          default:
            break;
        }
      }
#undef RP_EMIT
      }  // !head_fast
      if (p.epi == RP_EPI_LSE_PARTIAL && row_ok) {
        // each column half writes its own (max, sum) partial -- partial is
        // [rows, 2 * n_tiles, 2]; the CE finish merges them, so the two
        // halves never wait on each other (no per-tile barrier)
        float* dst = p.partial + (grow * (2 * p.n_tiles) + 2 * nb + half) * 2;
        dst[0] = run_max;
        dst[1] = run_sum;
      }
      tc_fence_before();
      if constexpr (kCta == 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_addr(&tmem_empty[acc]));
      } else {
        mbar_arrive(&tmem_empty[acc]);
      }
    }
  }

  if (warp >= 4 && p.tma_store && lane == 0) tma_store_wait_read();  // smem may be released
  tc_fence_before();
  __syncthreads();
  if constexpr (kCta == 2) cluster_sync();  // the leader's MMAs wrote both CTAs' TMEM
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kCta == 2)
      tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// split-K: out[m, n] = sum_s part[s][m, n] in fixed order (deterministic).
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int S, int64_t M, int64_t N, int64_t sstride,
                                     float* __restrict__ out, int64_t ldo) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= M * N) return;
  const int64_t m = i / N, n = i - m * N;
  if ((N & 3) == 0 && (ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    float4 acc = *reinterpret_cast<const float4*>(part + i);
    for (int s = 1; s < S; ++s) {
      const float4 v = *reinterpret_cast<const float4*>(part + s * sstride + i);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    *reinterpret_cast<float4*>(out + m * ldo + n) = acc;
  } else {
    for (int64_t e = i; e < min(i + 4, M * N); ++e) {
      float acc = part[e];
      for (int s = 1; s < S; ++s) acc += part[s * sstride + e];
      const int64_t mm = e / N, nn = e - mm * N;
      out[mm * ldo + nn] = acc;
    }
  }
}

int splitk_reduce(const float* part, int S, int64_t M, int64_t N, float* out, int64_t ldo, cudaStream_t st) {
  const int64_t n4 = (M * N + 3) / 4;
  if (n4 == 0) return RP_OK;
  splitk_reduce_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(part, S, M, N, M * N, out, ldo);
  return check_launch("splitk_reduce");
}

// ---------------------------------------------------------------------------
// fp32 -> (hi, lo) split for the 3-pass tf32 path.  Both halves are rounded to
// nearest tf32 here, so the tensor core consumes them exactly whatever its own
// fp32->tf32 conversion does; the residual |x - hi - lo| <= 2^-24 |x| is
// unbiased (truncating lo instead leaves a bias that grows like sqrt(K)).
__device__ __forceinline__ float round_tf32(float v) {
  uint32_t b = __float_as_uint(v);
  if ((b & 0x7F800000u) == 0x7F800000u) return v;  // inf / nan unchanged
  b += 0x0FFFu + ((b >> 13) & 1u);
  return __uint_as_float(b & 0xFFFFE000u);
}

__global__ void tf32_split_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t rows, int64_t cols, int64_t ld_src,
                                  int64_t ld_dst) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float v = x[r * ld_src + c];
    const float h = round_tf32(v);
    hi[r * ld_dst + c] = h;
    lo[r * ld_dst + c] = round_tf32(v - h);
  }
}

// ---------------------------------------------------------------------------
// host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

// rows x inner matrix (inner contiguous), `batch` copies at `bstride` elements.
int make_map(CUtensorMap* map, const void* ptr, bool tf32, int64_t inner, int64_t rows, int64_t ld,
             int64_t batch, int64_t bstride, int box_inner, int box_rows, bool mn_major, bool swizzle = true) {
  auto enc = encoder();
  if (!enc) return set_error(RP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int e = tf32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0)
    return set_error(RP_ERR_DIMENSION, "GEMM operand base must be 16-byte aligned");
  if ((ld * e) % 16 != 0) return set_error(RP_ERR_DIMENSION, "GEMM leading dimension must be a multiple of 16 bytes");
  if (batch <= 1) bstride = ld * std::max<int64_t>(rows, 1);
  if ((bstride * e) % 16 != 0) return set_error(RP_ERR_DIMENSION, "GEMM batch stride must be a multiple of 16 bytes");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)std::max<int64_t>(batch, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * e), (cuuint64_t)(bstride * e)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   !swizzle ? CU_TENSOR_MAP_SWIZZLE_NONE
                   : (tf32 && mn_major) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RP_OK;
}

bool pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RP_2CTA");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RP_NO_PDL");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& c = n[dev & 63];
  if (c == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    c = v > 0 ? v : 148;
  }
  return c;
}

template <bool kTf32, int BN, int kCta>
int launch(const rp_gemm_args& a, cudaStream_t stream) {
  using Cfg = GemmCfg<kTf32, BN, kCta>;
  static uint64_t attr_done = 0;
  if (first_on_device(attr_done))
    cudaFuncSetAttribute(gemm_kernel<kTf32, BN, kCta>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
  CUtensorMap ma, mal, mb, mbl;
  const int ks = a.k_splits > 1 ? a.k_splits : 1;
  if (ks > 1 && a.epilogue != RP_EPI_STORE) return set_error(RP_ERR_INVALID, "split-K needs the plain store epilogue");
  const int64_t kchunk = ks > 1 ? ((a.K + ks - 1) / ks + Cfg::BK - 1) / Cfg::BK * Cfg::BK : a.K;
  const int64_t batch = std::max<int64_t>(a.batch, 1);
  int st;
  // A: K-major -> inner K, rows M ; MN-major -> inner M, rows K
  if (!a.a_mn_major)
    st = make_map(&ma, a.A, kTf32, a.K, a.M, a.lda, batch, a.stride_a, Cfg::BK, Cfg::BM, false);
  else
    st = make_map(&ma, a.A, kTf32, a.M, a.K, a.lda, batch, a.stride_a, Cfg::CHUNK, Cfg::BK, true);
  if (st) return st;
  if (!a.b_mn_major)
    st = make_map(&mb, a.B, kTf32, a.K, a.N, a.ldb, batch, a.stride_b, Cfg::BK, Cfg::B_ROWS, false);
  else
    st = make_map(&mb, a.B, kTf32, a.N, a.K, a.ldb, batch, a.stride_b, Cfg::CHUNK, Cfg::BK, true);
  if (st) return st;
  int passes = 1;
  mal = ma;
  mbl = mb;
  if (a.math == RP_MATH_TF32X3) {
    if (!a.A_lo || !a.B_lo) return set_error(RP_ERR_INVALID, "tf32x3 GEMM needs split operands A_lo/B_lo");
    passes = 3;
    if (!a.a_mn_major)
      st = make_map(&mal, a.A_lo, kTf32, a.K, a.M, a.lda, batch, a.stride_a, Cfg::BK, Cfg::BM, false);
    else
      st = make_map(&mal, a.A_lo, kTf32, a.M, a.K, a.lda, batch, a.stride_a, Cfg::CHUNK, Cfg::BK, true);
    if (st) return st;
    if (!a.b_mn_major)
      st = make_map(&mbl, a.B_lo, kTf32, a.K, a.N, a.ldb, batch, a.stride_b, Cfg::BK, Cfg::B_ROWS, false);
    else
      st = make_map(&mbl, a.B_lo, kTf32, a.N, a.K, a.ldb, batch, a.stride_b, Cfg::CHUNK, Cfg::BK, true);
    if (st) return st;
  }
  CUtensorMap mc;
  std::memset(&mc, 0, sizeof(mc));
  bool tma_store = false;
  {
    auto enc = encoder();
    const int64_t rows_c = a.M * batch;
    // folded-batch rows must not spill into the next batch: M % BM == 0 when batched
    const bool packed_batch = batch == 1 || (a.stride_c == a.M * a.ldc && a.M % Cfg::BM == 0);
    if (enc && a.out_dtype == RP_BF16 && ks == 1 && a.C && packed_batch &&
        (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && (a.ldc * 2) % 16 == 0 && a.N >= 32 &&
        a.epilogue != RP_EPI_LSE_PARTIAL && rows_c < (1LL << 31)) {
      cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)rows_c};
      cuuint64_t strides[1] = {(cuuint64_t)(a.ldc * 2)};
      cuuint32_t box[2] = {32, 32};
      cuuint32_t estr[2] = {1, 1};
      tma_store = enc(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.C, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  CUtensorMap mr;
  std::memset(&mr, 0, sizeof(mr));
  bool tma_resid = false;
  {
    auto enc = encoder();
    const int64_t rows_r = a.M * batch;
    const bool uses = a.residual && (a.epilogue == RP_EPI_RELU_GRAD || a.epilogue == RP_EPI_GELU_GRAD ||
                                     a.epilogue == RP_EPI_BIAS_DROPOUT_RESIDUAL);
    const bool packed = batch == 1 || (a.stride_residual == a.M * a.ld_residual && a.M % Cfg::BM == 0);
    if (enc && uses && a.out_dtype == RP_BF16 && ks == 1 && packed &&
        (reinterpret_cast<uintptr_t>(a.residual) & 15) == 0 && (a.ld_residual * 2) % 16 == 0 && a.N >= 32 &&
        rows_r < (1LL << 31) && !getenv("RP_NO_TMA_RESID")) {
      cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)rows_r};
      cuuint64_t strides[1] = {(cuuint64_t)(a.ld_residual * 2)};
      cuuint32_t box[2] = {32, 32};
      cuuint32_t estr[2] = {1, 1};
      tma_resid = enc(&mr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.residual), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  GemmParams p{};
  p.tma_store = tma_store;
  p.tma_resid = tma_resid;
  if (a.k_lo_sign > 0 && (ks > 1 || a.k_lo_off < INT32_MIN / 2 || a.k_lo_off > INT32_MAX / 2))
    return set_error(RP_ERR_INVALID, "banded A: no split-K, |k_lo_off| < 2^30");
  p.k_lo_sign = a.k_lo_sign > 0 ? 1 : 0;
  p.k_lo_off = (int)a.k_lo_off;
  p.M = (int)a.M;
  p.N = (int)a.N;
  p.K = (int)a.K;
  p.batch = ks > 1 ? ks * (int)batch : (int)batch;
  p.ksplit = ks > 1 ? (int)kchunk : 0;
  p.bsz = (int)batch;
  p.a_mn = a.a_mn_major;
  p.b_mn = a.b_mn_major;
  p.passes = passes;
  p.m_tiles = (int)((a.M + Cfg::BM_TILE - 1) / Cfg::BM_TILE);
  p.n_tiles = (int)((a.N + BN - 1) / BN);
  p.num_tiles = p.m_tiles * p.n_tiles * p.batch;
  p.n_fast = p.n_tiles < p.m_tiles;
  p.kb_per_pass = (int)((kchunk + Cfg::BK - 1) / Cfg::BK);
  p.out_bf16 = a.out_dtype == RP_BF16;
  p.epi = a.epilogue;
  p.alpha = a.alpha;
  p.C = a.C;
  p.ldc = a.ldc;
  p.stride_c = a.stride_c;
  p.bias = a.bias;
  p.resid = a.residual;
  p.ld_resid = a.ld_residual;
  p.stride_resid = a.stride_residual;
  p.drop_seed = a.drop_seed;
  p.drop_thr = a.drop_threshold;
  p.drop_pos0 = a.drop_pos0;
  p.drop_scale = a.drop_scale;
  p.drop_on = a.drop_enabled;
  p.targets = a.targets;
  p.lse = a.lse;
  p.partial = a.partial;
  p.target_logit = a.target_logit;
  p.ce_scale = a.ce_scale;
  const int oe = p.out_bf16 ? 2 : 4;
  p.resid_vec = ((reinterpret_cast<uintptr_t>(a.residual) & 15) == 0) && ((a.ld_residual * oe) % 16 == 0) &&
                ((a.stride_residual * oe) % 16 == 0 || batch == 1);
  p.vec_ok = ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0) && ((a.ldc * oe) % 16 == 0) &&
             ((a.stride_c * oe) % 16 == 0 || p.batch == 1);
  p.vec2_ok = !p.out_bf16 && ((reinterpret_cast<uintptr_t>(a.C) & 7) == 0) && (a.ldc % 2 == 0) &&
              (a.stride_c % 2 == 0 || p.batch == 1);
  if (p.num_tiles == 0) return RP_OK;
  int grid = std::min(p.num_tiles * kCta, num_sms() / kCta * kCta);
  if (a.max_ctas > 0) grid = std::min(grid, std::max(kCta, a.max_ctas / kCta * kCta));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kCta;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kCta > 1 ? 2 : 1;
  cudaError_t err = cudaLaunchKernelEx(&cfg, gemm_kernel<kTf32, BN, kCta>, ma, mal, mb, mbl, mc, mr, p);
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(RP_ERR_CUDA, "gemm launch: %s", cudaGetErrorString(err));
  return RP_OK;
}

}  // namespace

int tma_map_bf16_store32(CUtensorMap* map, const void* ptr, int64_t inner, int64_t rows, int64_t ld, int64_t batch) {
  auto enc = encoder();
  if (!enc) return set_error(RP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * 2) % 16 != 0)
    return set_error(RP_ERR_DIMENSION, "store map: 16-byte aligned rows required");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)std::max<int64_t>(batch, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(ld * 2 * rows)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RP_OK;
}

int tma_map_bf16(CUtensorMap* map, const void* ptr, int64_t inner, int64_t rows, int64_t ld, int64_t batch,
                 int64_t bstride, int box_inner, int box_rows, bool swizzle) {
  return make_map(map, ptr, false, inner, rows, ld, batch, bstride, box_inner, box_rows, false, swizzle);
}

// N tile.  Default: the widest tile (256) whenever N > 128 -- narrower tiles
// read the A tile from shared memory more often per MMA and measured slower
// on every block GEMM (tools/prof_block.py: 0.458 vs 0.593 ms per block
// fwd+bwd).  RP_TILE_N_SPREAD=1 instead narrows N to give every SM two tiles.
int gemm_tile_n(int64_t M, int64_t N, int64_t batch) {
  static int spread = -1, waves = -1;
  if (spread < 0) {
    const char* e = getenv("RP_TILE_N_SPREAD");
    spread = (e && e[0] == '1') ? 1 : 0;
    const char* w = getenv("RP_TILE_WAVES");
    waves = (w && w[0] == '1') ? 1 : 0;
  }
  if (!spread && waves && N > 256 && N <= 1024 && M > 128 && pair_enabled()) {
    // RP_TILE_WAVES=1 (A/B switch, off by default): pick the 128-wide tile
    // when the 256-wide tiling leaves most of its last wave of CTA pairs idle
    // (a 128-wide tile modelled at half the work and ~15% lower efficiency),
    // e.g. the N = 512 block GEMMs at 11,264 rows (C3: 88 tiles on 74 pairs).
    // Measured slower on the C3 step (14.05 vs 13.75 ms): the narrow tiles
    // lose more than the model's 15%.
    const int64_t pairs = std::max<int64_t>(1, num_sms() / 2);
    const int64_t mt = (M + 255) / 256 * std::max<int64_t>(batch, 1);
    const int64_t w256 = (mt * ((N + 255) / 256) + pairs - 1) / pairs;
    const int64_t w128 = (mt * ((N + 127) / 128) + pairs - 1) / pairs;
    return (w128 * 128 * 115 < w256 * 256 * 100) ? 128 : 256;
  }
  if (!spread) return N > 128 ? 256 : (N > 64 ? 128 : 64);
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  const int64_t mt = (M + 127) / 128 * std::max<int64_t>(batch, 1);
  for (int bn : {256, 128}) {
    if (mt * ((N + bn - 1) / bn) >= 2 * 148) return bn;
  }
  return 64;
}

int gemm(const rp_gemm_args& a, cudaStream_t stream) {
  if (a.M < 0 || a.N < 0 || a.K <= 0) return set_error(RP_ERR_DIMENSION, "bad GEMM shape");
  if (a.M > INT32_MAX || a.N > INT32_MAX || a.K > INT32_MAX) return set_error(RP_ERR_DIMENSION, "GEMM dim too large");
  const bool tf32 = a.math != RP_MATH_BF16;
  int bn = a.tile_n > 0 ? a.tile_n : gemm_tile_n(a.M, a.N, a.k_splits > 1 ? a.k_splits * std::max<int64_t>(a.batch, 1) : a.batch);
  // dropout + residual epilogue after a short K loop: the per-element mask
  // hash dominates a tile, so 128 x 64 tiles spread it over every SM and
  // overlap it with the next tile's mainloop (tile choice never changes the
  // result: C3 out-projection 31 -> 24 us, tools/gemm_c3_shapes.py)
  if (a.tile_n <= 0 && !tf32 && a.epilogue == RP_EPI_BIAS_DROPOUT_RESIDUAL && a.drop_enabled && a.K <= 512) bn = 64;
  if (tf32) {
    if (bn == 256) return launch<true, 256, 1>(a, stream);
    if (bn == 128) return launch<true, 128, 1>(a, stream);
    return launch<true, 64, 1>(a, stream);
  }
  // bf16: CTA pairs (cta_group::2, 256-row tiles, half of B staged per CTA)
  // whenever there are rows for both CTAs of a pair
  if (bn >= 128 && a.M > 128 && pair_enabled()) {
    if (bn == 256) return launch<false, 256, 2>(a, stream);
    return launch<false, 128, 2>(a, stream);
  }
  if (bn == 256) return launch<false, 256, 1>(a, stream);
  if (bn == 128) return launch<false, 128, 1>(a, stream);
  return launch<false, 64, 1>(a, stream);
}

int tf32_split(const float* x, float* hi, float* lo, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
               cudaStream_t stream) {
  const int64_t n = rows * cols;
  if (n == 0) return RP_OK;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
  tf32_split_kernel<<<(int)blocks, threads, 0, stream>>>(x, hi, lo, rows, cols, ld_src, ld_dst);
  return check_launch("tf32_split");
}

}  // namespace rp
