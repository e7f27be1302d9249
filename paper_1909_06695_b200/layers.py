"""Device forward / hand-derived backward of the three layer kinds.

Same math and op order as the reference layer protocol (reference
pkg/src/ringpipe/layers.py): token+position embedding with dropout
(layers.py:114-136), the pre-LN single-head block (layers.py:168-253) and the
tied projection with its fused softmax cross-entropy head (layers.py:268-322).
Every op is one call into libringpipe_b200.so: tcgen05 GEMMs with fused
epilogues for all contractions, row kernels for LayerNorm / softmax /
dropout-masked gradients, a deterministic sorted scatter for the tied
embedding gradient.  Activations are stored in the compute dtype (bf16 or
fp32), every reduction and every gradient flowing along the residual stream
is fp32.

Dropout streams follow the reference exactly: the layer's seed is
mix64(dropout_seed, step, global_layer_idx) (model.py:218-219); the
embedding mask occupies stream positions [0, n); the block's attention mask
[0, n) and FFN mask [n, 2n) with n = B*T*d (layers.py:184-195, 209-212).
"""

import math

import torch

from . import _native as N
from . import ops
from .rng import keep_threshold

BLOCK_VEC = (("ln1_g", "d"), ("ln1_b", "d"), ("ln2_g", "d"), ("ln2_b", "d"), ("b1", "f"), ("b2", "d"))
BLOCK_MAT = (("wqkv", ("d", "3d")), ("wo", ("d", "d")), ("w1", ("d", "f")), ("w2", ("f", "d")))
# reference key order of a block's parameters (layers.py:153-166)
BLOCK_KEYS = ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2")


def _pad8(n):
    return (n + 7) // 8 * 8


_GOLDEN = 0x9E3779B97F4A7C15
_MASK64 = (1 << 64) - 1


class Dropout:
    """(seed, integer keep threshold, 1/(1-p)) of one layer stream, or None."""

    @staticmethod
    def make(seed, p, train):
        if not train or p <= 0.0:
            return None
        return (seed, keep_threshold(p), 1.0 / (1.0 - p))

    @staticmethod
    def shift(drop, positions):
        """The same stream `positions` further on: the mask draws
        splitmix64(seed + (pos + 1) * GOLDEN) (reference tensor.py:41-48,
        63-70), so position pos + k of `seed` is position pos of
        seed + k * GOLDEN (mod 2^64).  A row block starting at token row r0 of
        a [B, T, d] batch uses shift(drop, r0 * d)."""
        if drop is None or not positions:
            return drop
        return ((drop[0] + positions * _GOLDEN) & _MASK64,) + tuple(drop[1:])


def pad_cols(cols, dtype):
    """Row pitch of a [rows, cols] matrix: bf16 rows are padded to 16 bytes
    (the TMA row-pitch rule) when cols is not a multiple of 8 -- BASELINE
    configs[3]'s d 410, heads of 41 and d_ff 2100."""
    return _pad8(cols) if dtype == torch.bfloat16 and cols % 8 else cols


def empty_rows(*shape, dtype, device):
    """torch.empty(shape) whose last-dim rows sit at pad_cols pitch (a view)."""
    c = shape[-1]
    cp = pad_cols(c, dtype)
    t = torch.empty(*shape[:-1], cp, dtype=dtype, device=device)
    return t if cp == c else t[..., :c]


def copy_rows(dst, src):
    """dst.copy_(src) for row-major [..., rows, cols] tensors; when both share
    one padded row pitch the copy runs over the padded rows (one dense copy
    instead of a strided one; pad columns carry no data)."""
    ld = dst.stride(-2) if dst.dim() >= 2 else 0
    if (dst.shape == src.shape and dst.dim() >= 2 and dst.stride(-1) == 1 and src.stride(-1) == 1
            and ld != dst.shape[-1] and src.stride(-2) == ld and dst.dtype == src.dtype):
        shp = tuple(dst.shape[:-1]) + (ld,)
        dst.as_strided(shp, dst.stride()).copy_(src.as_strided(shp, src.stride()))
    else:
        dst.copy_(src)


class Workspace:
    """Named scratch buffers reused across calls (one per module and role)."""

    def __init__(self, device):
        self.device = device
        self._bufs = {}

    def get(self, name, shape, dtype):
        shape = tuple(int(s) for s in shape)
        t = self._bufs.get(name)
        if t is None or t.dtype != dtype or t.numel() < math.prod(shape):
            t = torch.empty(math.prod(shape), dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[: math.prod(shape)].view(shape)

    def get_rows(self, name, shape, dtype):
        """Like get, with the last-dim rows at pad_cols pitch."""
        c = shape[-1]
        cp = pad_cols(c, dtype)
        t = self.get(name, tuple(shape[:-1]) + (cp,), dtype)
        return t if cp == c else t[..., :c]

    def nbytes(self):
        return sum(t.numel() * t.element_size() for t in self._bufs.values())


class BlockTape:
    """Forward intermediates of one block for one stale slot (store-all)."""

    def __init__(self, B, T, d, f, dtype, device, activation="relu"):
        N = B * T
        Tp = _pad8(T)
        self.activation = activation
        e = lambda *s: torch.empty(s, dtype=dtype, device=device)  # noqa: E731
        f32 = lambda *s: torch.empty(s, dtype=torch.float32, device=device)  # noqa: E731
        self.a = e(N, d)
        self.qkv = e(B, T, 3 * d)
        self.probs_buf = e(B, T, Tp)
        self.probs = self.probs_buf[:, :, :T]
        self.ctx = e(B, T, d)
        self.x1 = e(N, d)
        self.m = e(N, d)
        self.h1 = e(N, f)
        self.z1 = e(N, f) if activation == "gelu" else None  # the GELU pre-activation (its gradient needs it)
        self.mean1, self.rstd1, self.mean2, self.rstd2 = f32(N), f32(N), f32(N), f32(N)

    def nbytes(self):
        return sum(t.numel() * t.element_size() for t in
                   (self.a, self.qkv, self.probs_buf, self.ctx, self.x1, self.m, self.h1, self.z1,
                    self.mean1, self.rstd1, self.mean2, self.rstd2) if t is not None)


ACTIVATIONS = ("relu", "gelu")


def ffn_up(W, vecs, m, tape, probe=None):
    """h1 = act(m w1 + b1) into tape.h1: ReLU fused in the GEMM epilogue
    (reference layers.py:190-191); GELU as z1 = m w1 + b1 (kept for the
    backward) and the vector GELU kernel."""
    if getattr(tape, "activation", "relu") == "gelu":
        ops.gemm(m, W["w1"], b_mn=True, out=tape.z1, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=vecs["b1"],
                 probe=probe)
        ops.gelu(tape.z1, tape.h1)
    else:
        ops.gemm(m, W["w1"], b_mn=True, out=tape.h1, epilogue=N.EPI_BIAS_RELU, bias=vecs["b1"], probe=probe)


def ffn_act_grad(g_h2, W, tape, g_z1, probe=None):
    """g_z1 = (g_h2 w2^T) * act'(z1) (reference layers.py:221 for ReLU)."""
    if getattr(tape, "activation", "relu") == "gelu":
        ops.gemm(g_h2, W["w2"], out=g_z1, epilogue=N.EPI_GELU_GRAD, residual=tape.z1, probe=probe)
    else:
        ops.gemm(g_h2, W["w2"], out=g_z1, epilogue=N.EPI_RELU_GRAD, residual=tape.h1, probe=probe)


# ---------------------------------------------------------------------------
# embedding (layers.py:114-136)


def embed_forward(tied_c, pos_c, tokens, out, vocab, drop, flag):
    ops.embed_fwd(tokens, tied_c, pos_c, out.view(tokens.shape[0], tokens.shape[1], -1), vocab, drop, flag)


def embed_backward(g, tokens, t_max, grad_pos, emb_grad, beta, ws, drop):
    """grad_pos fully written; emb_grad[tok] += beta * (scatter-sum of masked g)."""
    n = tokens.numel()
    nbytes = N.lib().rp_embed_bwd_workspace_bytes(n, g.shape[-1])
    work = ws.get("embed_ws", (max(256, nbytes),), torch.uint8)
    ops.embed_bwd(g, tokens, t_max, grad_pos, emb_grad, beta, work, drop)


# ---------------------------------------------------------------------------
# transformer block (layers.py:168-253)


def block_forward_ops(W, vecs, x, out, tape, B, T, drop, ws, flag):
    """x, out: [B*T, d] compute dtype.  W: compute-dtype matrices; vecs: fp32."""
    d = x.shape[-1]
    n = B * T * d
    ops.layernorm_fwd(x, vecs["ln1_g"], vecs["ln1_b"], tape.a, tape.mean1, tape.rstd1, flag)
    ops.gemm(tape.a, W["wqkv"], b_mn=True, out=tape.qkv.view(B * T, 3 * d))
    q, k, v = tape.qkv[..., :d], tape.qkv[..., d: 2 * d], tape.qkv[..., 2 * d:]
    Tp = tape.probs_buf.shape[-1]
    scores = ws.get("scores", (B, T, Tp), torch.float32)[:, :, :T]
    ops.gemm(q, k, alpha=1.0 / math.sqrt(d), out=scores)
    ops.softmax_causal(scores, tape.probs)
    ops.gemm(tape.probs, v, b_mn=True, out=tape.ctx)
    d0 = None if drop is None else (drop[0], drop[1], drop[2], 0)
    ops.gemm(tape.ctx.view(B * T, d), W["wo"], b_mn=True, out=tape.x1, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL,
             residual=x, dropout=d0)
    ops.layernorm_fwd(tape.x1, vecs["ln2_g"], vecs["ln2_b"], tape.m, tape.mean2, tape.rstd2, flag)
    with ops.span("ffn1_gemm"):
        ffn_up(W, vecs, tape.m, tape)
    d1 = None if drop is None else (drop[0], drop[1], drop[2], n)
    ops.gemm(tape.h1, W["w2"], b_mn=True, out=out, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=vecs["b2"],
             residual=tape.x1, dropout=d1)


def block_backward_ops(W, vecs, x, tape, g_out, g_x, G, B, T, drop, ws):
    """g_out, g_x: [B*T, d] fp32 (g_x may alias g_out).  G: fp32 grad views."""
    d = x.shape[-1]
    f = tape.h1.shape[-1]
    Nt = B * T
    n = Nt * d
    cdt = x.dtype
    inv = 1.0 / math.sqrt(d)
    nbc = ops.colsum_blocks(Nt)
    nbm = ops.mask_grad_blocks(Nt, d)
    part = ws.get("colsum_part", (max(nbc, nbm), max(f, 3 * d)), torch.float32)
    # feed-forward branch
    g_h2 = ws.get("g_h2", (Nt, d), cdt)
    pm = ws.get("mask_part", (nbm, d), torch.float32)
    ops.mask_grad(g_out, g_h2, n, drop, pm)
    ops.colsum_finish(pm, nbm, G["b2"])
    ops.gemm(tape.h1, g_h2, a_mn=True, b_mn=True, out=G["w2"])
    g_z1 = ws.get("g_z1", (Nt, f), cdt)
    ffn_act_grad(g_h2, W, tape, g_z1)
    ops.colsum_partial(g_z1, part[:, :f])
    ops.colsum_finish(part[:, :f], nbc, G["b1"])
    ops.gemm(tape.m, g_z1, a_mn=True, b_mn=True, out=G["w1"])
    g_m = ws.get("g_m", (Nt, d), torch.float32)
    ops.gemm(g_z1, W["w1"], out=g_m)
    nbl = ops.layernorm_bwd_blocks(Nt)
    pg = ws.get("ln_pg", (nbl, d), torch.float32)
    pb = ws.get("ln_pb", (nbl, d), torch.float32)
    g_x1 = ws.get("g_x1", (Nt, d), torch.float32)
    g_proj = ws.get("g_proj", (Nt, d), cdt)
    ops.layernorm_bwd(g_m, tape.x1, tape.mean2, tape.rstd2, vecs["ln2_g"], g_x1, pg, pb, resid_grad=g_out,
                      dx_masked=g_proj, dropout=drop)
    ops.colsum_finish(pg, nbl, G["ln2_g"])
    ops.colsum_finish(pb, nbl, G["ln2_b"])
    # attention branch
    ops.gemm(tape.ctx.view(Nt, d), g_proj, a_mn=True, b_mn=True, out=G["wo"])
    g_ctx = ws.get("g_ctx", (B, T, d), cdt)
    ops.gemm(g_proj, W["wo"], out=g_ctx.view(Nt, d))
    Tp = tape.probs_buf.shape[-1]
    g_p = ws.get("g_p", (B, T, Tp), torch.float32)[:, :, :T]
    q, k, v = tape.qkv[..., :d], tape.qkv[..., d: 2 * d], tape.qkv[..., 2 * d:]
    ops.gemm(g_ctx, v, out=g_p)
    g_qkv = ws.get("g_qkv", (B, T, 3 * d), cdt)
    ops.gemm(tape.probs, g_ctx, a_mn=True, b_mn=True, out=g_qkv[..., 2 * d:])
    g_s = ws.get("g_s", (B, T, Tp), cdt)[:, :, :T]
    ops.softmax_bwd(g_p, tape.probs, g_s, inv)
    ops.gemm(g_s, k, b_mn=True, out=g_qkv[..., :d])
    ops.gemm(g_s, q, a_mn=True, b_mn=True, out=g_qkv[..., d: 2 * d])
    g2 = g_qkv.view(Nt, 3 * d)
    ops.gemm(tape.a, g2, a_mn=True, b_mn=True, out=G["wqkv"])
    g_a = ws.get("g_a", (Nt, d), torch.float32)
    ops.gemm(g2, W["wqkv"], out=g_a)
    ops.layernorm_bwd(g_a, x, tape.mean1, tape.rstd1, vecs["ln1_g"], g_x, pg, pb, resid_grad=g_x1)
    ops.colsum_finish(pg, nbl, G["ln1_g"])
    ops.colsum_finish(pb, nbl, G["ln1_b"])


# ---------------------------------------------------------------------------
# tied head (layers.py:287-322)


class HeadState:
    """Per-slot head intermediates: row logsumexp and the loss."""

    def __init__(self, Nt, device):
        self.lse = torch.empty(Nt, dtype=torch.float32, device=device)
        self.loss = torch.empty((), dtype=torch.float32, device=device)
        self.loss64 = torch.empty((), dtype=torch.float64, device=device)


def head_forward_ops(h, tied_c, targets, vocab, hs, ws, flag):
    """Mean CE of h @ tied^T against targets without materialising logits."""
    Nt = h.shape[0]
    bn = ops.gemm_tile_n(vocab, Nt)
    nt = (vocab + bn - 1) // bn
    partial = ws.get("head_partial", (Nt, 2 * nt, 2), torch.float32)  # per tile and column half
    zy = ws.get("head_zy", (Nt,), torch.float32)
    rows_loss = ws.get("head_rows", (Nt,), torch.float32)
    with ops.span("head_gemm"):
        ops.gemm(h, tied_c, epilogue=N.EPI_LSE_PARTIAL, targets=targets, partial=partial, target_logit=zy)
    ops.ce_finish(partial, zy, targets, vocab, hs.lse, rows_loss, hs.loss, hs.loss64, flag)


def head_backward_ops(h, tied_c, targets, vocab, hs, g_h, vo_out, vo_alpha, ws, vo_accumulate=False):
    """g_h = dz @ tied (fp32); vo_out = vo_alpha * dz^T @ h when vo_out is given."""
    Nt, d = h.shape
    vp = _pad8(vocab)
    dz = ws.get("head_dz", (Nt, vp), h.dtype)[:, :vocab]
    with ops.span("head_gemm"):
        ops.gemm(h, tied_c, epilogue=N.EPI_CE_GRAD, targets=targets, lse=hs.lse, ce_scale=1.0 / Nt, out=dz)
    with ops.span("head_gemm"):
        ops.gemm(dz, tied_c, b_mn=True, out=g_h)
    if vo_out is not None:
        with ops.span("head_gemm"):
            if vo_accumulate:
                ops.gemm(dz, h, a_mn=True, b_mn=True, out=vo_out, alpha=vo_alpha,
                         epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, residual=vo_out)
            else:
                ops.gemm(dz, h, a_mn=True, b_mn=True, out=vo_out, alpha=vo_alpha)


# ---------------------------------------------------------------------------
# native composites (csrc/layers.cpp): one C-ABI call per layer.  The *_ops
# functions above are the same sequence issued op by op from Python and are
# kept as a cross-check (tests/test_layers_gpu.py asserts bitwise equality).

import ctypes  # noqa: E402


def _p(t):
    return None if t is None else t.data_ptr()


# SM budget for the block GEMMs issued from the current thread (0 = whole GPU);
# the concurrent engine lowers it for work off the critical path.
CTA_BUDGET = {"value": 0}


def _block_desc(x, f, B, T, drop, rows_total=0, activation="relu"):
    dsc = N.BlockDesc()
    dsc.drop_rows_total = rows_total or 0
    dsc.activation = N.ACT_GELU if activation == "gelu" else N.ACT_RELU
    dsc.max_ctas = CTA_BUDGET["value"]
    dsc.B, dsc.T, dsc.d, dsc.f = B, T, x.shape[-1], f
    dsc.dtype = N.BF16 if x.dtype == torch.bfloat16 else N.F32
    if drop is not None:
        dsc.drop_enabled, dsc.drop_seed, dsc.drop_threshold, dsc.drop_scale = 1, drop[0], drop[1], drop[2]
    return dsc


def _weights(W):
    w = N.BlockWeights()
    for n in ("wqkv", "wo", "w1", "w2", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b1", "b2"):
        setattr(w, n, W[n].data_ptr())
    return w


def _tape(tp):
    t = N.BlockTape()
    t.a, t.qkv, t.probs, t.ctx = _p(tp.a), _p(tp.qkv), _p(tp.probs_buf), _p(tp.ctx)
    t.x1, t.m, t.h1 = _p(tp.x1), _p(tp.m), _p(tp.h1)
    t.z1 = _p(getattr(tp, "z1", None))
    t.mean1, t.rstd1, t.mean2, t.rstd2 = _p(tp.mean1), _p(tp.rstd1), _p(tp.mean2), _p(tp.rstd2)
    return t


def _ws_bytes(ws, name, nbytes):
    buf = ws.get(name, (int(nbytes),), torch.uint8)
    return buf


def block_forward(W, vecs, x, out, tape, B, T, drop, ws, flag, rows_total=0):
    """rows_total: token rows of the whole batch when this is one row block of
    it (micro-batched relay; the caller shifts `drop` to the block's rows)."""
    f = tape.h1.shape[-1]
    dsc = _block_desc(x, f, B, T, drop, rows_total, getattr(tape, "activation", "relu"))
    nbytes = N.lib().rp_block_workspace_bytes(ctypes.byref(dsc))
    buf = _ws_bytes(ws, "block_ws", nbytes)
    ops._count(13 if getattr(tape, "activation", "relu") == "gelu" else 12)
    N.check(N.lib().rp_block_forward(ctypes.byref(dsc), ctypes.byref(_weights(W)), _p(x), _p(out),
                                     ctypes.byref(_tape(tape)), _p(buf), nbytes, _p(flag), ops._stream()),
            "block_forward")


def block_backward(W, vecs, x, tape, g_out, g_x, G, B, T, drop, ws, rows_total=0):
    f = tape.h1.shape[-1]
    dsc = _block_desc(x, f, B, T, drop, rows_total, getattr(tape, "activation", "relu"))
    nbytes = N.lib().rp_block_workspace_bytes(ctypes.byref(dsc))
    buf = _ws_bytes(ws, "block_ws", nbytes)
    g = N.BlockGrads()
    for n in ("wqkv", "wo", "w1", "w2", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b1", "b2"):
        setattr(g, n, G[n].data_ptr())
    ops._count(27)
    N.check(N.lib().rp_block_backward(ctypes.byref(dsc), ctypes.byref(_weights(W)), _p(x), ctypes.byref(_tape(tape)),
                                      _p(g_out), _p(g_x), ctypes.byref(g), _p(buf), nbytes, ops._stream()),
            "block_backward")


def _head_desc(h, vocab, rows_total=0):
    hd = N.HeadDesc()
    hd.rows, hd.d, hd.vocab = h.shape[0], h.shape[1], vocab
    hd.rows_total = rows_total or 0
    hd.dtype = N.BF16 if h.dtype == torch.bfloat16 else N.F32
    return hd


def head_forward(h, tied_c, targets, vocab, hs, ws, flag):
    hd = _head_desc(h, vocab)
    nbytes = N.lib().rp_head_workspace_bytes(ctypes.byref(hd))
    buf = _ws_bytes(ws, "head_ws", nbytes)
    ops._count(3)
    with ops.span("head_gemm"):
        N.check(N.lib().rp_head_forward(ctypes.byref(hd), _p(h), _p(tied_c), _p(targets), _p(hs.lse), _p(hs.loss),
                                        _p(hs.loss64), _p(buf), nbytes, _p(flag), ops._stream()), "head_forward")


def head_backward(h, tied_c, targets, vocab, hs, g_h, vo_out, vo_alpha, ws, vo_accumulate=False, rows_total=0):
    """rows_total: rows of the whole batch when h is one row block of it (the
    cross-entropy gradient is 1/rows_total, layers.py:319)."""
    hd = _head_desc(h, vocab, rows_total)
    nbytes = N.lib().rp_head_workspace_bytes(ctypes.byref(hd))
    buf = _ws_bytes(ws, "head_ws", nbytes)
    ops._count(3 if vo_out is not None else 2)
    with ops.span("head_gemm_bwd"):
        N.check(N.lib().rp_head_backward(ctypes.byref(hd), _p(h), _p(tied_c), _p(targets), _p(hs.lse), _p(g_h),
                                         _p(vo_out), vo_alpha, int(vo_accumulate), _p(buf), nbytes, ops._stream()),
                "head_backward")
