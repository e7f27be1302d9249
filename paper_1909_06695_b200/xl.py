"""Transformer-XL block on the device.

Relative-position multi-head attention with segment-level memory (Dai et al.
2019; fp64 restatement and its tests: oracle/xl.py) inside the reference's
pre-LN block (reference layers.py:168-253: LayerNorm, dropout positions, ReLU
FFN and residuals are unchanged).  There is no reference implementation, so
parity is pinned through the restatement.

Per slot the block keeps `xa` = [memory rows; current rows] (B*M + B*T rows
of d): the memory part is the previous segment's layer input (stop-gradient),
the current part is this segment's layer input, written in place by the
upstream layer or module.  Every contraction is a tcgen05 GEMM over
head-major operands; csrc/xl.cu does the head splits, the relative-shift
softmax and the gradient merges.
"""

import math
import os

import numpy as np
import torch

from . import _native as N
from . import ops
from . import layers as LY
from .layers import _pad8


def sinusoid(Kl, d, dtype, device):
    """R [Kl, d]: row p encodes distance Kl-1-p as [sin, cos] (XL's
    PositionalEmbedding over the descending pos_seq), evaluated in fp64."""
    dist = np.arange(Kl - 1, -1, -1, dtype=np.float64)
    inv = 1.0 / (10000.0 ** (np.arange(0, d, 2, dtype=np.float64) / d))
    ang = dist[:, None] * inv[None, :]
    R = np.concatenate([np.sin(ang), np.cos(ang)], axis=1)
    out = LY.empty_rows(Kl, d, dtype=dtype, device=device)  # a GEMM operand: 16-byte rows
    out.copy_(torch.from_numpy(R))
    return out


class XLTape:
    """Store-all intermediates of one XL block for one stale slot."""

    def __init__(self, B, T, M, d, f, H, dtype, device, activation="relu"):
        Kl = M + T
        self.activation = activation
        dh = d // H
        ldk = _pad8(Kl)
        # rows at 16-byte pitches for bf16 (LY.pad_cols: d 410, head dim 41, d_ff 2100)
        e = lambda *s: LY.empty_rows(*s, dtype=dtype, device=device)  # noqa: E731
        f32 = lambda *s: torch.empty(s, dtype=torch.float32, device=device)  # noqa: E731
        self.B, self.T, self.M, self.H, self.dh, self.Kl, self.ldk = B, T, M, H, dh, Kl, ldk
        # bf16 head dims below 64 that are not 16-byte rows (BASELINE
        # configs[3]: 41) ride in rows zero-padded to 64: the fused forward
        # (head dim 64) then takes them -- the pads add zero to every score
        # and to P v (the split kernels write the real columns only)
        self.dhp = 64 if (dtype == torch.bfloat16 and dh < 64 and dh % 8) else dh

        def heads(*s):
            if self.dhp == dh:
                return e(*s)
            return torch.zeros(*s[:-1], self.dhp, dtype=dtype, device=device)[..., :dh]

        self.xa = e(B * Kl, d)            # [memory rows; current rows]
        self.a = e(B * Kl, d)
        self.mean1, self.rstd1 = f32(B * Kl), f32(B * Kl)
        self.qkv = e(B * Kl, 3 * d)
        self.qu, self.qv = heads(H, B * T, dh), heads(H, B * T, dh)
        self.kh, self.vh = heads(H, B * Kl, dh), heads(H, B * Kl, dh)
        self.rh = heads(H, Kl, dh)
        self.probs_buf = torch.empty(H * B, T, ldk, dtype=dtype, device=device)
        self.probs = self.probs_buf[:, :, :Kl]
        self.ctx = e(B * T, d)
        self.x1 = e(B * T, d)
        self.m = e(B * T, d)
        self.h1 = e(B * T, f)
        self.z1 = e(B * T, f) if activation == "gelu" else None
        self.mean2, self.rstd2 = f32(B * T), f32(B * T)
        self.mem_len = 0

    @property
    def x(self):
        """This segment's layer input (the upstream writes it here)."""
        return self.xa[self.B * self.M:]

    @property
    def mem(self):
        return self.xa[: self.B * self.M]

    def nbytes(self):
        return sum(t.numel() * t.element_size() for t in vars(self).values() if torch.is_tensor(t))


def _bg(*a, **k):
    """The block's dense contractions (QKV / R / out-projection / FFN and their
    gradients): one tagged GEMM family for bench.py's roofline."""
    return ops.gemm(*a, probe="block_gemm", **k)


FUSED = os.environ.get("RP_XL_FUSED", "1") != "0"
# N tile of the dropout + residual epilogue GEMMs (out-projection, FFN out):
# 0 = the library default (A/B switch)
DROP_TILE = int(os.environ.get("RP_DROP_TILE", "0"))
# N tile of the unfused score / dP GEMMs (N = M + T keys, K = head dim <= 64:
# one k-block per tile, so the fp32 output epilogue dominates and 128-wide
# tiles waste less of it than the default 256 -- C4 shape, tools/xl_score_tiles.py:
# AC 117 -> 86 us, BD 75 -> 58 us, bitwise equal); 0 = the library default
SCORE_TILE = int(os.environ.get("RP_XL_SCORE_TILE", "128"))


def fused_ok(tp):
    """The fused attention kernels (csrc/xl_attn.cu) take bf16, head dim 64 or 128;
    other shapes and the fp32 check mode use the GEMM + softmax-kernel path."""
    return FUSED and tp.xa.dtype == torch.bfloat16 and tp.dh in (64, 128)


def fused_bwd_ok(tp):
    """The fused backward TMA-stores dBD chunks at column offsets T - 128 - i0
    + 128 n, which must be 16-byte aligned: T % 8 == 0."""
    return fused_ok(tp) and tp.T % 8 == 0


FUSED_DQ = os.environ.get("RP_XL_FUSED_DQ", "1") != "0"
FUSED_PV = os.environ.get("RP_XL_FUSED_PV", "1") != "0"
BANDED = os.environ.get("RP_XL_BANDED", "1") != "0"
FUSED_KV = os.environ.get("RP_XL_FUSED_KV", "1") != "0"


def fused_pv_ok(tp):
    """The forward with P.V folded in (xl_attn_fwd_pv): head dim 64, or a
    smaller one zero-padded to 64 in the tape (XLTape.dhp)."""
    if not FUSED_PV or tp.xa.dtype != torch.bfloat16:
        return False
    return (FUSED and tp.dh == 64) or (FUSED and getattr(tp, "dhp", tp.dh) == 64)


def fused_dq_ok(tp):
    """The backward with the query-gradient MMAs folded in (xl_attn_bwd_dq):
    head dim 64 and whole 128-query tiles."""
    return FUSED_DQ and fused_bwd_ok(tp) and tp.dh == 64 and tp.T % 128 == 0


def fused_kv_ok(tp):
    """dK / dV from the key-major kernel (xl_attn_bwd_kv) after xl_attn_bwd_dq,
    which then skips the dAC matrix."""
    return FUSED_KV and fused_dq_ok(tp)


# The engines run each XL block as ONE C-ABI call (rp_xl_block_forward /
# _backward: the same kernels in the same order, bitwise equal to the
# op-by-op path below, tests/test_module_abi_gpu.py) -- ~25 launches per block
# issued from C++ instead of Python, which keeps the host ahead of the GPU.
# The op-by-op path runs under the bench's instrumented window (ops.PROBE:
# per-launch events and FLOP tags), for widths the dense-row composite does
# not take (bf16 rows of d 410 / head dim 41: pitched), and with RP_XL_NATIVE=0.
NATIVE = os.environ.get("RP_XL_NATIVE", "1") != "0"


def native_ok(tp):
    if not NATIVE or ops.PROBE is not None:
        return False
    if tp.xa.dtype != torch.bfloat16:
        return True
    d, f = tp.H * tp.dh, tp.h1.shape[-1]
    return d % 8 == 0 and f % 8 == 0 and tp.dh % 8 == 0


def xl_block_forward(W, vecs, out, tp, R, drop, ws, flag, rows_total=0):
    """One XL block forward (native composite when native_ok, else op by op)."""
    if native_ok(tp):
        return xl_block_forward_native(W, vecs, out, tp, R, drop, ws, flag, rows_total)
    return xl_block_forward_ops(W, vecs, out, tp, R, drop, ws, flag, rows_total)


def xl_block_backward(W, vecs, tp, R, g_out, g_x, G, drop, ws, rows_total=0):
    """One XL block backward (native composite when native_ok, else op by op)."""
    if native_ok(tp):
        return xl_block_backward_native(W, vecs, tp, R, g_out, g_x, G, drop, ws, rows_total)
    return xl_block_backward_ops(W, vecs, tp, R, g_out, g_x, G, drop, ws, rows_total)


def xl_block_forward_ops(W, vecs, out, tp, R, drop, ws, flag, rows_total=0):
    """tp.xa holds [memory; x]; writes out [B*T, d] and the tape.  rows_total:
    token rows of the whole batch when this is one row block of it (the
    second dropout mask starts at rows_total * d; `drop` is already shifted
    to the block's first row)."""
    B, T, M, H, dh, Kl = tp.B, tp.T, tp.M, tp.H, tp.dh, tp.Kl
    d = H * dh
    n = (rows_total or B * T) * d
    cdt = tp.xa.dtype
    ops.layernorm_fwd(tp.xa, vecs["ln1_g"], vecs["ln1_b"], tp.a, tp.mean1, tp.rstd1, flag)
    _bg(tp.a, W["wqkv"], b_mn=True, out=tp.qkv)
    ops.xl_split_qkv(tp.qkv, vecs["r_w_bias"], vecs["r_r_bias"], tp.qu, tp.qv, tp.kh, tp.vh, B, T, M, H, dh)
    r = ws.get_rows("xl_r", (Kl, d), cdt)
    _bg(R, W["wr"], b_mn=True, out=r)
    ops.xl_split_heads(r, tp.rh, H, dh)
    pv_done = False
    if fused_pv_ok(tp):
        # scores + relative shift + masked softmax + P.V in one tcgen05 kernel (csrc/xl_attn.cu)
        with ops.span("xl_attn_fwd"):
            ops.xl_attn_fwd_pv(tp.qu, tp.qv, tp.kh, tp.vh, tp.rh, tp.probs_buf, tp.ctx, B, T, M, tp.mem_len,
                               1.0 / math.sqrt(dh))
        pv_done = True
    elif fused_ok(tp):
        # scores + relative shift + masked softmax in one tcgen05 kernel (csrc/xl_attn.cu)
        with ops.span("xl_attn_fwd"):
            ops.xl_attn_fwd(tp.qu, tp.qv, tp.kh, tp.rh, tp.probs_buf, B, T, M, tp.mem_len, 1.0 / math.sqrt(dh))
    else:
        ac = ws.get("xl_ac", (H * B, T, tp.ldk), torch.float32)[:, :, :Kl]
        bd = ws.get("xl_bd", (H, B * T, tp.ldk), torch.float32)[:, :, :Kl]
        with ops.span("xl_scores"):
            ops.gemm(tp.qu.view(H * B, T, dh), tp.kh.view(H * B, Kl, dh), out=ac, tile_n=SCORE_TILE)
            ops.gemm(tp.qv, tp.rh, out=bd, tile_n=SCORE_TILE)
        ops.xl_softmax_fwd(ac, bd, tp.probs_buf, T, M, tp.mem_len, 1.0 / math.sqrt(dh))
    if not pv_done:
        ctx_h = ws.get_rows("xl_ctx_h", (H * B, T, dh), cdt)
        ops.gemm(tp.probs, tp.vh.view(H * B, Kl, dh), b_mn=True, out=ctx_h)
        ops.xl_merge_heads(ctx_h.view(H, B * T, dh), tp.ctx, H, dh)
    d0 = None if drop is None else (drop[0], drop[1], drop[2], 0)
    _bg(tp.ctx, W["wo"], b_mn=True, out=tp.x1, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, residual=tp.x, dropout=d0,
        tile_n=DROP_TILE)
    ops.layernorm_fwd(tp.x1, vecs["ln2_g"], vecs["ln2_b"], tp.m, tp.mean2, tp.rstd2, flag)
    LY.ffn_up(W, vecs, tp.m, tp, probe="block_gemm")
    d1 = None if drop is None else (drop[0], drop[1], drop[2], n)
    _bg(tp.h1, W["w2"], b_mn=True, out=out, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=vecs["b2"], tile_n=DROP_TILE,
             residual=tp.x1, dropout=d1)


def xl_block_backward_ops(W, vecs, tp, R, g_out, g_x, G, drop, ws, rows_total=0):
    """g_out, g_x: [B*T, d] fp32.  No gradient flows into the memory rows;
    their LayerNorm / K / V contributions to the weight gradients do."""
    B, T, M, H, dh, Kl = tp.B, tp.T, tp.M, tp.H, tp.dh, tp.Kl
    d = H * dh
    f = tp.h1.shape[-1]
    Nt = B * T
    n = (rows_total or Nt) * d
    cdt = tp.xa.dtype
    scale = 1.0 / math.sqrt(dh)
    # feed-forward + LN2 (as the reference block)
    nbc = ops.colsum_blocks(Nt)
    g_h2 = ws.get_rows("g_h2", (Nt, d), cdt)
    nbm = ops.mask_grad_blocks(Nt, d, ops._pitch(g_h2))
    part = ws.get("colsum_part", (max(nbc, nbm), max(f, 3 * d)), torch.float32)
    pm = ws.get("mask_part", (nbm, d), torch.float32)
    ops.mask_grad(g_out, g_h2, n, drop, pm)
    _bg(tp.h1, g_h2, a_mn=True, b_mn=True, out=G["w2"])
    g_z1 = ws.get_rows("g_z1", (Nt, f), cdt)
    LY.ffn_act_grad(g_h2, W, tp, g_z1, probe="block_gemm")
    ops.colsum_partial(g_z1, part[:, :f])
    _bg(tp.m, g_z1, a_mn=True, b_mn=True, out=G["w1"])
    g_m = ws.get("g_m", (Nt, d), torch.float32)
    _bg(g_z1, W["w1"], out=g_m)
    nbl_cur = ops.layernorm_bwd_blocks(Nt)
    nbl_mem = ops.layernorm_bwd_blocks(B * M) if M else 0
    pg = ws.get("ln_pg", (nbl_cur + nbl_mem, d), torch.float32)
    pb = ws.get("ln_pb", (nbl_cur + nbl_mem, d), torch.float32)
    g_x1 = ws.get("g_x1", (Nt, d), torch.float32)
    g_proj = ws.get_rows("g_proj", (Nt, d), cdt)
    pg2 = ws.get("ln2_pg", (nbl_cur, d), torch.float32)
    pb2 = ws.get("ln2_pb", (nbl_cur, d), torch.float32)
    ops.layernorm_bwd(g_m, tp.x1, tp.mean2, tp.rstd2, vecs["ln2_g"], g_x1, pg2, pb2,
                      resid_grad=g_out, dx_masked=g_proj, dropout=drop)
    # relative-position attention
    _bg(tp.ctx, g_proj, a_mn=True, b_mn=True, out=G["wo"])
    g_ctx = ws.get_rows("g_ctx", (Nt, d), cdt)
    _bg(g_proj, W["wo"], out=g_ctx)
    g_ctx_h = ws.get_rows("xl_g_ctx_h", (H, Nt, dh), cdt)
    ops.xl_split_heads(g_ctx, g_ctx_h, H, dh)
    g3 = g_ctx_h.view(H * B, T, dh)
    g_ac = ws.get("xl_g_ac", (H * B, T, tp.ldk), cdt)
    g_bd = ws.get("xl_g_bd", (H, Nt, tp.ldk), cdt)
    # fp32 head-gradient rows at 16-byte pitches (head dim 41 -> 44): the GEMM
    # epilogues store them with vector stores
    f32r = lambda name, *s: ws.get(name, s[:-1] + (-(-s[-1] // 4) * 4,), torch.float32)[..., : s[-1]]  # noqa: E731
    g_qu = f32r("xl_g_qu", H, Nt, dh)
    g_qv = f32r("xl_g_qv", H, Nt, dh)
    dq_done = False
    bias_part = None
    kv = fused_kv_ok(tp)
    d_rows = ws.get("xl_d_rows", (H * B * T,), torch.float32) if kv else None
    # the persistent bwd_dq and bwd_kv write straight into the merged g_qkv rows
    # (no fp32 dQu / dQv, no merge pass)
    merged = kv and bool(N.lib().rp_xl_dq_persistent())
    g_qkv = ws.get_rows("xl_g_qkv", (B * Kl, 3 * d), cdt)
    if fused_dq_ok(tp):
        # dP, dS, dAC / dBD and dQu = dAC k, dQv = dBD r in one kernel (csrc/xl_attn.cu),
        # plus the per-CTA column sums of dQu / dQv for the u / v gradients; with
        # the key-major kernel below it leaves D per query row instead of dAC
        bias_part = ws.get("xl_dq_bias", (ops.xl_dq_bias_part_elems(H, B, T),), torch.float32)
        with ops.span("xl_attn_bwd"):
            ops.xl_attn_bwd_dq(g_ctx_h, tp.vh, tp.kh, tp.rh, tp.probs_buf, None if kv else g_ac, g_bd, g_ctx, tp.ctx,
                               None if merged else g_qu, None if merged else g_qv, B, T, M, tp.mem_len, scale,
                               bias_part=bias_part, d_rows=d_rows, g_qkv=g_qkv if merged else None)
        dq_done = True
    elif fused_bwd_ok(tp):
        # dP on the tensor cores, dS, dAC and the un-shifted dBD in one kernel (csrc/xl_attn.cu)
        with ops.span("xl_attn_bwd"):
            ops.xl_attn_bwd(g_ctx_h, tp.vh, tp.probs_buf, g_ac, g_bd, g_ctx, tp.ctx, B, T, M, tp.mem_len, scale)
    else:
        g_p = ws.get("xl_ac", (H * B, T, tp.ldk), torch.float32)[:, :, :Kl]
        ops.gemm(g3, tp.vh.view(H * B, Kl, dh), out=g_p, tile_n=SCORE_TILE)
        ops.xl_softmax_bwd(g_p, tp.probs_buf, g_ac, g_bd, T, M, tp.mem_len, scale)
    # dK / dV leave their GEMMs rounded to the compute dtype, as g_qkv holds them
    g_vh = ws.get_rows("xl_g_vh", (H * B, Kl, dh), cdt) if cdt == torch.bfloat16 else f32r("xl_g_vh", H * B, Kl, dh)
    # P^T and dAC^T are banded: key j sees queries i >= j - M (causal window),
    # so each key tile starts its K loop (over queries) at its first live block
    band = -M if BANDED else None
    g_kh = ws.get_rows("xl_g_kh", (H * B, Kl, dh), cdt) if cdt == torch.bfloat16 else f32r("xl_g_kh", H * B, Kl, dh)
    if kv:
        # dV = P^T dO and dK = dS^T (q+u) in one key-major kernel: bitwise the two
        # banded GEMMs below, without the dAC matrix
        with ops.span("xl_attn_bwd"):
            ops.xl_attn_bwd_kv(g3, tp.vh.view(H * B, Kl, dh), tp.qu.view(H * B, T, dh), tp.probs_buf, d_rows,
                               None if merged else g_kh, None if merged else g_vh, B, T, M, tp.mem_len, scale,
                               g_qkv=g_qkv if merged else None)
    else:
        ops.gemm(tp.probs, g3, a_mn=True, b_mn=True, out=g_vh, k_lo_off=band)
    g_ac, g_bd = g_ac[:, :, :Kl], g_bd[:, :, :Kl]
    g_rh = f32r("xl_g_rh", H, Kl, dh)
    if not dq_done:
        ops.gemm(g_ac, tp.kh.view(H * B, Kl, dh), b_mn=True, out=g_qu.view(H * B, T, dh))
    if not kv:
        ops.gemm(g_ac, tp.qu.view(H * B, T, dh), a_mn=True, b_mn=True, out=g_kh, k_lo_off=band)
    if not dq_done:
        ops.gemm(g_bd, tp.rh, b_mn=True, out=g_qv)
    ops.gemm(g_bd, tp.qv, a_mn=True, b_mn=True, out=g_rh)
    bias_jobs = []
    if bias_part is not None:
        # the fused backward's per-CTA dQu / dQv column sums: [B*nqt, H*64] per bias,
        # finished with the block's other column sums below
        pu, pv = bias_part.view(2, -1, H * dh)
        bias_jobs = [(pu, pu.shape[0], G["r_w_bias"]), (pv, pv.shape[0], G["r_r_bias"])]
    else:
        work = ws.get("xl_bias_ws", (N.lib().rp_xl_bias_grad_workspace_bytes(H, dh) // 4,), torch.float32)
        ops.xl_bias_grad(g_qu, g_qv, work, G["r_w_bias"], G["r_r_bias"], H, Nt, dh)
    g_r = ws.get_rows("xl_g_r", (Kl, d), cdt)
    ops.xl_merge_heads(g_rh, g_r, H, dh)
    _bg(R, g_r, a_mn=True, b_mn=True, out=G["wr"])
    if not merged:
        ops.xl_merge_grads(g_qu, g_qv, g_kh, g_vh, g_qkv, B, T, M, H, dh)
    _bg(tp.a, g_qkv, a_mn=True, b_mn=True, out=G["wqkv"])
    g_a = ws.get("xl_g_a", (B * Kl, d), torch.float32)
    _bg(g_qkv, W["wqkv"], out=g_a)
    # LN1 over both row blocks: memory rows add to the gain / bias sums only
    # (stop-gradient: no dx is written for them)
    BM = B * M
    if M:
        ops.layernorm_bwd(g_a[:BM], tp.xa[:BM], tp.mean1[:BM], tp.rstd1[:BM], vecs["ln1_g"], None,
                          pg[nbl_cur:], pb[nbl_cur:])
    ops.layernorm_bwd(g_a[BM:], tp.xa[BM:], tp.mean1[BM:], tp.rstd1[BM:], vecs["ln1_g"], g_x, pg[:nbl_cur],
                      pb[:nbl_cur], resid_grad=g_x1)
    # every bias / gain column sum of the block finished in one launch
    ops.colsum_finish_multi([(pm, nbm, G["b2"]), (part[:, :f], nbc, G["b1"]), (pg2, nbl_cur, G["ln2_g"]),
                             (pb2, nbl_cur, G["ln2_b"]), (pg, nbl_cur + nbl_mem, G["ln1_g"]),
                             (pb, nbl_cur + nbl_mem, G["ln1_b"])] + bias_jobs)


# ---------------------------------------------------------------------------
# the same block through the C ABI (rp_xl_block_forward / _backward,
# csrc/layers.cpp): one call per block for a non-Python host, bitwise equal
# to the op-by-op path above (tests/test_module_abi_gpu.py)


def fused_flags(tp):
    """The RP_XL_FUSED_* kernels this process's switches select for the tape."""
    f = 0
    if fused_pv_ok(tp):
        f |= N.XL_FUSED_PV
    elif fused_ok(tp):
        f |= N.XL_FUSED_FWD
    if fused_dq_ok(tp):
        f |= N.XL_FUSED_DQ
        if fused_kv_ok(tp):
            f |= N.XL_FUSED_KV
    elif fused_bwd_ok(tp):
        f |= N.XL_FUSED_BWD
    if BANDED:
        f |= N.XL_BANDED
    return f


def xl_desc(tp, drop, rows_total=0, max_ctas=0):
    from .rng import keep_threshold  # noqa: F401

    d = N.XlBlockDesc()
    d.B, d.T, d.M, d.d, d.f = tp.B, tp.T, tp.M, tp.H * tp.dh, tp.h1.shape[-1]
    d.H, d.dtype = tp.H, N.BF16 if tp.xa.dtype == torch.bfloat16 else N.F32
    d.activation = N.ACT_GELU if getattr(tp, "activation", "relu") == "gelu" else N.ACT_RELU
    d.max_ctas, d.mem_len = max_ctas, tp.mem_len
    if drop is not None:
        d.drop_enabled, d.drop_seed, d.drop_threshold, d.drop_scale = 1, drop[0], drop[1], drop[2]
    d.drop_rows_total = rows_total or 0
    d.ldk = tp.ldk
    d.fused = fused_flags(tp)
    d.score_tile = SCORE_TILE
    return d


def xl_weights(W):
    w = N.XlBlockWeights()
    for n in N.XL_W_MATS + N.XL_W_VECS:
        setattr(w, n, W[n].data_ptr())
    return w


def xl_tape(tp):
    t = N.XlBlockTape()
    for n in N.XL_TAPE:
        v = tp.probs_buf if n == "probs" else getattr(tp, n, None)
        setattr(t, n, None if v is None else v.data_ptr())
    return t


def xl_grads(G):
    g = N.XlBlockGrads()
    for n in ("wqkv", "wo", "w1", "w2", "wr", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b1", "b2", "r_w_bias", "r_r_bias"):
        setattr(g, n, G[n].data_ptr())
    return g


def _native_ws(ws, d):
    import ctypes

    nbytes = N.lib().rp_xl_block_workspace_bytes(ctypes.byref(d))
    return ws.get("xl_native_ws", (max(256, nbytes),), torch.uint8), nbytes


def xl_block_forward_native(W, vecs, out, tp, R, drop, ws, flag, rows_total=0):
    import ctypes

    d = xl_desc(tp, drop, rows_total)
    buf, nbytes = _native_ws(ws, d)
    ops._count(1)
    N.check(N.lib().rp_xl_block_forward(ctypes.byref(d), ctypes.byref(xl_weights(W)), R.data_ptr(), out.data_ptr(),
                                        ctypes.byref(xl_tape(tp)), buf.data_ptr(), nbytes,
                                        None if flag is None else flag.data_ptr(), ops._stream()), "xl_block_forward")


def xl_block_backward_native(W, vecs, tp, R, g_out, g_x, G, drop, ws, rows_total=0):
    import ctypes

    d = xl_desc(tp, drop, rows_total)
    buf, nbytes = _native_ws(ws, d)
    ops._count(1)
    N.check(N.lib().rp_xl_block_backward(ctypes.byref(d), ctypes.byref(xl_weights(W)), R.data_ptr(),
                                         ctypes.byref(xl_tape(tp)), g_out.data_ptr(), g_x.data_ptr(),
                                         ctypes.byref(xl_grads(G)), buf.data_ptr(), nbytes, ops._stream()),
            "xl_block_backward")

