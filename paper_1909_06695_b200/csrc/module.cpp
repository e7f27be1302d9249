// Module-level entry points (ModuleState.forward / recompute_backward,
// reference model.py:224-304): the layer loop of one pipeline module over the
// layer composites, so a non-Python host drives a module with two calls per
// step.  Same kernels in the same order as the Python host loop
// (paper_1909_06695_b200/model.py), so results are bitwise identical.
#include <algorithm>

#include "rp_internal.h"

namespace rp {
namespace {

#define RP_TRY(x)                \
  do {                           \
    if (int _e = (x)) return _e; \
  } while (0)

inline int64_t al256(int64_t b) { return (b + 255) / 256 * 256; }

rp_block_desc block_desc(const rp_module_desc& m, int layer) {
  rp_block_desc d{};
  d.B = m.B;
  d.T = m.T;
  d.d = m.d;
  d.f = m.f;
  d.dtype = m.dtype;
  d.max_ctas = m.max_ctas;
  d.drop_enabled = m.drop_enabled;
  d.drop_seed = m.drop_enabled ? m.layer_seeds[layer] : 0;
  d.drop_threshold = m.drop_threshold;
  d.drop_scale = m.drop_scale;
  d.activation = m.activation;
  return d;
}

rp_xl_block_desc xl_desc(const rp_module_desc& m, int layer) {
  rp_xl_block_desc d{};
  d.B = m.B;
  d.T = m.T;
  d.M = m.M;
  d.d = m.d;
  d.f = m.f;
  d.H = m.n_heads;
  d.dtype = m.dtype;
  d.drop_enabled = m.drop_enabled;
  d.activation = m.activation;
  d.max_ctas = m.max_ctas;
  d.mem_len = m.mem_len;
  d.drop_seed = m.drop_enabled ? m.layer_seeds[layer] : 0;
  d.drop_threshold = m.drop_threshold;
  d.drop_scale = m.drop_scale;
  d.ldk = (m.M + m.T + 7) / 8 * 8;
  d.fused = m.xl_fused;
  d.score_tile = m.score_tile;
  return d;
}

rp_head_desc head_desc(const rp_module_desc& m) { return rp_head_desc{m.B * m.T, m.d, m.vocab, m.dtype, 0}; }

int64_t layer_ws_bytes(const rp_module_desc& m) {
  int64_t b = 256;
  if (m.n_blocks > 0)
    b = std::max(b, m.n_heads > 0 ? xl_block_workspace_bytes(xl_desc(m, 0)) : block_workspace_bytes(block_desc(m, 0)));
  if (m.has_projection) b = std::max(b, head_workspace_bytes(head_desc(m)));
  if (m.has_embedding) b = std::max(b, embed_bwd_workspace_bytes(m.B * m.T, m.d));
  return al256(b);
}

int check_desc(const rp_module_desc& m) {
  if (m.n_blocks < 0 || m.B <= 0 || m.T <= 0 || m.d <= 0)
    return set_error(RP_ERR_DIMENSION, "module: bad shape");
  if (m.n_blocks == 0 && !m.has_embedding && !m.has_projection)
    return set_error(RP_ERR_INVALID, "module: empty layer slice");
  if (m.drop_enabled && !m.layer_seeds) return set_error(RP_ERR_INVALID, "module: dropout needs layer_seeds");
  if (m.n_heads < 0 || (m.n_heads > 0 && (m.d % m.n_heads || m.M < 0 || m.mem_len < 0 || m.mem_len > m.M)))
    return set_error(RP_ERR_DIMENSION, "module: bad Transformer-XL shape");
  if (m.dtype == RP_BF16 && (m.d % 8 || (m.n_blocks > 0 && m.f % 8) || (m.n_heads > 0 && (m.d / m.n_heads) % 8)))
    return set_error(RP_ERR_DIMENSION,
                     "module: the composite takes dense bf16 rows (d, d_ff, head dim multiples of 8); "
                     "pitched rows go through the op-level entry points");
  return RP_OK;
}

}  // namespace

int64_t module_workspace_bytes(const rp_module_desc& m) {
  return layer_ws_bytes(m) + 2 * al256(m.B * m.T * m.d * 4) + 256;
}

int module_forward(const rp_module_desc& m, const rp_module_weights& w, const rp_module_slot& s, void* out,
                   void* ws, int64_t ws_bytes, int32_t* flag, cudaStream_t st) {
  RP_TRY(check_desc(m));
  if (ws_bytes < module_workspace_bytes(m)) return set_error(RP_ERR_INVALID, "module workspace too small");
  const int64_t lws = layer_ws_bytes(m);
  const int n_acts = m.n_blocks + (m.has_projection ? 1 : 0);
  int layer = 0;
  if (m.has_embedding) {
    void* dst = n_acts > 0 ? s.acts[0] : out;
    const uint64_t seed = m.drop_enabled ? m.layer_seeds[0] : 0;
    RP_TRY(embed_fwd(m.dtype, s.tokens, w.tied, w.pos, dst, m.B, m.T, m.d, m.vocab, seed, m.drop_threshold,
                     m.drop_scale, m.drop_enabled, flag, st));
    layer = 1;
  }
  for (int j = 0; j < m.n_blocks; ++j) {
    void* dst = j + 1 < n_acts ? s.acts[j + 1] : out;
    if (!dst) return set_error(RP_ERR_INVALID, "module_forward: no output buffer for the last block");
    if (m.n_heads > 0) {
      if (!w.xl_blocks || !s.xl_tapes || !w.R) return set_error(RP_ERR_INVALID, "module_forward: XL module lacks XL blocks");
      RP_TRY(xl_block_forward(xl_desc(m, layer + j), w.xl_blocks[j], w.R, dst, s.xl_tapes[j], ws, lws, flag, st));
    } else {
      RP_TRY(block_forward(block_desc(m, layer + j), w.blocks[j], s.acts[j], dst, s.tapes[j], ws, lws, flag, st));
    }
  }
  if (m.has_projection)
    RP_TRY(head_forward(head_desc(m), s.acts[m.n_blocks], w.tied, s.targets, s.lse, s.loss, s.loss64, ws, lws, flag,
                        st));
  return RP_OK;
}

int module_backward(const rp_module_desc& m, const rp_module_weights& w, const rp_module_slot& s, const float* g_out,
                    float* g_in, const rp_module_grads& G, void* ws, int64_t ws_bytes, cudaStream_t st) {
  RP_TRY(check_desc(m));
  if (ws_bytes < module_workspace_bytes(m)) return set_error(RP_ERR_INVALID, "module workspace too small");
  const int64_t lws = layer_ws_bytes(m);
  const int64_t rows = m.B * m.T;
  float* gbuf[2] = {reinterpret_cast<float*>(static_cast<char*>(ws) + lws),
                    reinterpret_cast<float*>(static_cast<char*>(ws) + lws + al256(rows * m.d * 4))};
  const float* g = g_out;
  int ping = 1;
  if (m.has_projection) {
    float* vo = (G.tied && G.tied_alpha != 0.f) ? G.tied : nullptr;
    RP_TRY(head_backward(head_desc(m), s.acts[m.n_blocks], w.tied, s.targets, s.lse, gbuf[0], vo, G.tied_alpha,
                         G.tied_accumulate, ws, lws, st));
    g = gbuf[0];
  } else if (!g) {
    return set_error(RP_ERR_SCHEDULE, "module_backward: missing boundary gradient");
  }
  const int first_block_layer = m.has_embedding ? 1 : 0;
  for (int j = m.n_blocks - 1; j >= 0; --j) {
    float* g_next;
    if (j == 0 && !m.has_embedding && g_in) {
      g_next = g_in;
    } else {
      g_next = gbuf[ping];
      ping ^= 1;
    }
    if (m.n_heads > 0) {
      if (!w.xl_blocks || !s.xl_tapes || !G.xl_blocks || !w.R)
        return set_error(RP_ERR_INVALID, "module_backward: XL module lacks XL blocks");
      RP_TRY(xl_block_backward(xl_desc(m, first_block_layer + j), w.xl_blocks[j], w.R, s.xl_tapes[j], g, g_next,
                               G.xl_blocks[j], ws, lws, st));
    } else {
      RP_TRY(block_backward(block_desc(m, first_block_layer + j), w.blocks[j], s.acts[j], s.tapes[j], g, g_next,
                            G.blocks[j], ws, lws, st));
    }
    g = g_next;
  }
  if (m.has_embedding) {
    const uint64_t seed = m.drop_enabled ? m.layer_seeds[0] : 0;
    float* vi = (G.tied && G.tied_beta != 0.f) ? G.tied : nullptr;
    return embed_bwd(g, s.tokens, m.B, m.T, m.t_max, m.d, m.vocab, seed, m.drop_threshold, m.drop_scale, m.drop_enabled,
                     G.pos, vi, G.tied_beta, ws, st);
  }
  if (g_in && g != g_in) {
    if (cudaMemcpyAsync(g_in, g, rows * m.d * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return set_error(RP_ERR_CUDA, "module_backward: copy of the input gradient failed");
  }
  return RP_OK;
}

}  // namespace rp
