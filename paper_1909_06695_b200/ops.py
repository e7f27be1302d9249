"""Thin torch-facing wrappers over the C-ABI kernels of libringpipe_b200.so.

Each wrapper validates shapes/dtypes, extracts raw device pointers and the
current CUDA stream, and calls one `rp_*` entry point.  Tensors are borrowed;
outputs are allocated with torch (PyTorch is the device-memory plumbing).
There is deliberately no CPU path: calling these on CPU tensors raises.
"""

import ctypes
import math

import torch

from . import _native as N
from .errors import DimensionError

_DT = {torch.float32: N.F32, torch.bfloat16: N.BF16}


class Probe:
    """Optional instrumentation used by bench.py: counts native kernel launches
    and records CUDA events around tagged GEMMs on the stream they run on."""

    def __init__(self):
        self.launches = 0
        self.events = {}  # tag -> list of (start, end)
        self.flops = {}  # tag -> list of algorithmic FLOPs per span (tagged GEMMs)

    def span(self, tag, flops=None):
        return _Span(self, tag, flops)

    def achieved(self, tag):
        """(total FLOPs, total ms, spans) of the tagged GEMM spans (synchronize first)."""
        ev = self.events.get(tag, [])
        fl = self.flops.get(tag, [])
        return float(sum(fl)), float(sum(s.elapsed_time(e) for s, e in ev)), len(ev)


class _Span:
    def __init__(self, probe, tag, flops=None):
        self.probe, self.tag, self.flops_ = probe, tag, flops

    def __enter__(self):
        if self.probe is not None:
            self.s = torch.cuda.Event(enable_timing=True)
            self.s.record()

    def __exit__(self, *exc):
        if self.probe is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.probe.events.setdefault(self.tag, []).append((self.s, e))
            if self.flops_ is not None:
                self.probe.flops.setdefault(self.tag, []).append(self.flops_)


PROBE = None  # set to a Probe() to instrument


def _count(n=1):
    if PROBE is not None:
        PROBE.launches += n


def span(tag, flops=None):
    return _Span(PROBE, tag, flops)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise DimensionError("ringpipe-b200 kernels take CUDA tensors only (no CPU fallback)")


def _mat3(t, name):
    """View a 2-d or 3-d tensor as (batch, rows, cols, ld, batch_stride)."""
    if t.dim() == 2:
        if t.stride(1) != 1:
            raise DimensionError(f"{name}: innermost dim must be contiguous")
        return 1, t.shape[0], t.shape[1], t.stride(0), t.shape[0] * t.stride(0)
    if t.dim() == 3:
        if t.stride(2) != 1:
            raise DimensionError(f"{name}: innermost dim must be contiguous")
        return t.shape[0], t.shape[1], t.shape[2], t.stride(1), t.stride(0)
    raise DimensionError(f"{name}: rank must be 2 or 3")


def tf32_split(x):
    """(hi, lo): x rounded to tf32 and the tf32-rounded remainder (both fp32).

    Outputs keep x's shape but with rows padded to 16 bytes so that TMA can
    address them whatever the logical width."""
    _require_cuda(x)
    if x.dtype != torch.float32:
        raise DimensionError("tf32_split takes fp32")
    if x.stride(-1) != 1 or (x.dim() == 3 and x.stride(0) != x.shape[1] * x.stride(1)):
        x = x.contiguous()
    cols = x.shape[-1]
    rows = x.numel() // max(cols, 1)
    ld_dst = (cols + 3) // 4 * 4
    shape = tuple(x.shape[:-1]) + (ld_dst,)
    hi = torch.empty(shape, dtype=torch.float32, device=x.device)
    lo = torch.empty_like(hi)
    ld = x.stride(-2) if x.dim() >= 2 else cols
    _count(1)
    N.check(N.lib().rp_tf32_split(_ptr(x), _ptr(hi), _ptr(lo), rows, cols, ld, ld_dst, _stream()), "tf32_split")
    return hi[..., :cols], lo[..., :cols]


def gemm(
    a,
    b,
    *,
    a_mn=False,
    b_mn=False,
    out=None,
    out_dtype=None,
    math=None,
    epilogue=N.EPI_STORE,
    alpha=1.0,
    bias=None,
    residual=None,
    dropout=None,
    targets=None,
    lse=None,
    partial=None,
    target_logit=None,
    ce_scale=0.0,
    a_lo=None,
    b_lo=None,
    tile_n=0,
    probe=None,
    k_lo_off=None,
):
    """C = epilogue(alpha * opA(a) @ opB(b)) on the tcgen05 GEMM.

    a: [M,K] (a_mn=False) or [K,M] (a_mn=True), optionally with a leading
    batch dim.  b: [N,K] (b_mn=False, "B transposed") or [K,N] (b_mn=True).
    bf16 operands run on kind::f16; fp32 operands run the 3-pass tf32 path
    unless math=MATH_TF32.  probe: a Probe tag -- with ops.PROBE set, the
    launch (and its split-K reduce) is bracketed by CUDA events and counted
    as 2*M*N*K*batch algorithmic FLOPs.  k_lo_off: op(A) is banded -- row m
    is zero for k < m + k_lo_off -- and tiles skip those k-blocks.
    """
    _require_cuda(a, b)
    if a.dtype != b.dtype or a.dtype not in _DT:
        raise DimensionError("GEMM operands must share dtype fp32 or bf16")
    ba, ra, ca, lda, sa = _mat3(a, "A")
    bb, rb, cb, ldb, sb = _mat3(b, "B")
    M, K = (ca, ra) if a_mn else (ra, ca)
    Nn, Kb = (cb, rb) if b_mn else (rb, cb)
    if K != Kb:
        raise DimensionError(f"inner dims disagree: K={K} vs {Kb}")
    batch = max(ba, bb)
    if ba != bb:
        if ba == 1 and a.dim() == 2:
            sa = 0
        elif bb == 1 and b.dim() == 2:
            sb = 0
        else:
            raise DimensionError("batch dims disagree")
    if math is None:
        math = N.MATH_BF16 if a.dtype == torch.bfloat16 else N.MATH_TF32X3
    if math == N.MATH_TF32X3 and (a_lo is None or b_lo is None):
        if a_lo is None:
            a, a_lo = tf32_split(a)
            ba, ra, ca, lda, sa = _mat3(a, "A")
        if b_lo is None:
            b, b_lo = tf32_split(b)
            bb, rb, cb, ldb, sb = _mat3(b, "B")
        if ba != bb:
            sa = 0 if ba == 1 else sa
            sb = 0 if bb == 1 else sb
    if out is None and epilogue != N.EPI_LSE_PARTIAL:
        odt = out_dtype or (torch.float32 if a.dtype == torch.float32 else torch.bfloat16)
        shape = (batch, M, Nn) if (a.dim() == 3 or b.dim() == 3) else (M, Nn)
        out = torch.empty(shape, dtype=odt, device=a.device)
    args = N.GemmArgs()
    args.math = math
    args.a_mn_major = int(a_mn)
    args.b_mn_major = int(b_mn)
    args.M, args.N, args.K, args.batch = M, Nn, K, batch
    args.A, args.A_lo, args.lda, args.stride_a = a.data_ptr(), (a_lo.data_ptr() if a_lo is not None else None), lda, sa
    args.B, args.B_lo, args.ldb, args.stride_b = b.data_ptr(), (b_lo.data_ptr() if b_lo is not None else None), ldb, sb
    if out is not None:
        _require_cuda(out)
        bo, ro, co, ldc, sc = _mat3(out, "C")
        if (ro, co) != (M, Nn):
            raise DimensionError(f"out shape {tuple(out.shape)} != ({M},{Nn})")
        args.out_dtype = _DT[out.dtype]
        args.C, args.ldc, args.stride_c = out.data_ptr(), ldc, sc
    else:
        args.out_dtype = N.F32
    args.epilogue = epilogue
    args.tile_n = tile_n
    if k_lo_off is not None:
        args.k_lo_sign, args.k_lo_off = 1, int(k_lo_off)
    args.alpha = alpha
    if bias is not None:
        args.bias = bias.data_ptr()
    if residual is not None:
        _, _, _, ldr, sr = _mat3(residual, "residual")
        args.residual, args.ld_residual, args.stride_residual = residual.data_ptr(), ldr, sr
    if dropout is not None:
        seed, thr, scale, pos0 = dropout
        args.drop_enabled = 1
        args.drop_seed, args.drop_threshold, args.drop_scale, args.drop_pos0 = seed, thr, scale, pos0
    if targets is not None:
        args.targets = targets.data_ptr()
    if lse is not None:
        args.lse = lse.data_ptr()
    if partial is not None:
        args.partial = partial.data_ptr()
    if target_logit is not None:
        args.target_logit = target_logit.data_ptr()
    args.ce_scale = ce_scale
    splits = 1
    rows_fold = batch == 1 or (out is not None and args.stride_c == M * args.ldc)
    if (out is not None and out.dtype == torch.float32 and epilogue == N.EPI_STORE and rows_fold
            and k_lo_off is None):
        # deterministic split-K for weight-gradient shapes (few tiles, long K;
        # batched: the XL dR GEMM, 8 heads x 8 key tiles), the same rule and
        # scratch size as the native composites (layers.cpp)
        splits = N.lib().rp_gemm_choose_splits(M, Nn, K, batch, SPLITK_CAP)
    if splits > 1:
        part = _splitk_scratch(out.device)
        args.k_splits = splits
        args.C, args.ldc, args.stride_c = part.data_ptr(), Nn, M * Nn
    with _Span(PROBE if probe else None, probe, 2.0 * M * Nn * K * batch):
        _count(1)
        N.check(N.lib().rp_gemm(ctypes.byref(args), _stream()), "gemm")
        if splits > 1:
            _count(1)
            N.check(N.lib().rp_splitk_reduce(_ptr(part), splits, batch * M, Nn, _ptr(out), out.stride(-2), _stream()),
                    "splitk_reduce")
    return out


SPLITK_CAP = 296 * 128 * 256 * 4  # bytes of split-K partials (= layers.cpp kBlockSplitK)
_SPLITK = {}


def _splitk_scratch(device):
    """Split-K partials, one buffer per (device, stream): GEMMs on one stream
    run in order, so they can share it; streams never do."""
    key = (device, torch.cuda.current_stream().cuda_stream)
    buf = _SPLITK.get(key)
    if buf is None:
        buf = _SPLITK[key] = torch.empty(SPLITK_CAP // 4, dtype=torch.float32, device=device)
    return buf


def gemm_tile_n(n, m=8192, batch=1):
    return N.lib().rp_gemm_tile_n(m, n, batch)


# ---------------------------------------------------------------------------
# row kernels


def _dtc(t):
    return _DT[t.dtype]


def _pitch(t):
    """Row pitch (elements) of a row-major matrix view whose rows may be padded
    (d not a multiple of 8: 16-byte bf16 rows); checks the layout the kernels assume."""
    if t is None:
        return 0
    if t.dim() >= 2 and t.stride(-1) == 1:
        ld = t.stride(-2)
        # leading dims must fold onto rows: stride(i) == size(i+1) * stride(i+1)
        for i in range(t.dim() - 2):
            if t.stride(i) != t.shape[i + 1] * t.stride(i + 1):
                raise DimensionError("row-padded tensors must be dense above the row dimension")
        return ld
    if t.is_contiguous():
        return t.shape[-1]
    raise DimensionError("kernels take row-major tensors (unit column stride)")


def _rows(t):
    return t.numel() // t.shape[-1]


def layernorm_fwd(x, gain, bias, y, mean, rstd, flag=None):
    rows, d = _rows(x), x.shape[-1]
    _count(1)
    N.check(N.lib().rp_layernorm_fwd(_dtc(x), _ptr(x), _ptr(gain), _ptr(bias), _ptr(y), _ptr(mean), _ptr(rstd),
                                     rows, d, _pitch(x), _pitch(y), _ptr(flag), _stream()), "layernorm_fwd")


def layernorm_bwd_blocks(rows):
    return N.lib().rp_layernorm_bwd_blocks(rows)


def layernorm_bwd(dy, x, mean, rstd, gain, dx, part_g, part_b, resid_grad=None, dx_masked=None, dropout=None):
    rows, d = _rows(x), x.shape[-1]
    for t in (dy, dx, resid_grad):
        if t is not None and not t.is_contiguous():
            raise DimensionError("layernorm_bwd: fp32 rows must be contiguous")
    seed, thr, scale = dropout if dropout is not None else (0, 0, 1.0)
    _count(1)
    N.check(N.lib().rp_layernorm_bwd(_dtc(x), _ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(gain),
                                     _ptr(resid_grad), _ptr(dx), _ptr(dx_masked), seed, thr, scale,
                                     int(dropout is not None), _ptr(part_g), _ptr(part_b), rows, d, _pitch(x),
                                     _pitch(dx_masked), _stream()),
            "layernorm_bwd")


def colsum_blocks(rows):
    return N.lib().rp_colsum_blocks(rows)


def mask_grad_blocks(rows, d, ld_out=0):
    return N.lib().rp_mask_grad_blocks_ld(rows, d, ld_out)


def colsum_partial(x, part):
    cols = x.shape[-1]
    rows = x.numel() // cols
    _count(1)
    N.check(N.lib().rp_colsum_partial(_dtc(x), _ptr(x), rows, cols, x.stride(-2), _ptr(part), _stream()),
            "colsum_partial")


def colsum_finish_multi(jobs):
    """jobs: up to 8 (part, nblk, out) triples finished in one launch."""
    n = len(jobs)
    parts = (ctypes.c_void_p * n)(*[j[0].data_ptr() for j in jobs])
    nblk = (ctypes.c_int32 * n)(*[j[1] for j in jobs])
    cols = (ctypes.c_int64 * n)(*[j[2].numel() for j in jobs])
    outs = (ctypes.c_void_p * n)(*[j[2].data_ptr() for j in jobs])
    _count(1)
    N.check(N.lib().rp_colsum_finish_multi(parts, nblk, cols, outs, n, _stream()), "colsum_finish_multi")


def colsum_finish(part, nblk, out):
    _count(1)
    N.check(N.lib().rp_colsum_finish(_ptr(part), nblk, out.numel(), _ptr(out), _stream()), "colsum_finish")


def mask_grad(g, out, pos0, dropout, part):
    rows, d = _rows(g), g.shape[-1]
    seed, thr, scale = dropout if dropout is not None else (0, 0, 1.0)
    _count(1)
    N.check(N.lib().rp_mask_grad(_dtc(out), _ptr(g), _ptr(out), rows, d, seed, pos0, thr, scale,
                                 int(dropout is not None), _ptr(part), _pitch(out), _stream()), "mask_grad")


def softmax_causal(scores, probs):
    """scores fp32 [B,T,>=T] view -> probs [B,T,T] view (row stride from probs)."""
    B, T = scores.shape[0], scores.shape[1]
    if scores.stride(1) != probs.stride(1):
        raise DimensionError("scores/probs row strides differ")
    _count(1)
    N.check(N.lib().rp_softmax_causal(_dtc(probs), _ptr(scores), _ptr(probs), B * T, T, probs.stride(1), _stream()),
            "softmax_causal")


def softmax_bwd(grad_probs, probs, grad_scores, scale):
    B, T = probs.shape[0], probs.shape[1]
    _count(1)
    N.check(N.lib().rp_softmax_bwd(_dtc(probs), _ptr(grad_probs), _ptr(probs), _ptr(grad_scores), scale, B * T, T,
                                   probs.stride(1), _stream()), "softmax_bwd")


# ---------------------------------------------------------------------------
# Transformer-XL attention glue (csrc/xl.cu)


def xl_split_qkv(qkv, u, v, qu, qv, kh, vh, B, T, M, H, dh):
    _require_cuda(qkv, u, v, qu, qv, kh, vh)
    ldh = _pitch(qu)
    if any(_pitch(t) != ldh for t in (qv, kh, vh)):
        raise DimensionError("xl_split_qkv: the head tensors share one row pitch")
    _count(1)
    N.check(N.lib().rp_xl_split_qkv(_dtc(qkv), _ptr(qkv), _ptr(u), _ptr(v), _ptr(qu), _ptr(qv), _ptr(kh), _ptr(vh),
                                    B, T, M, H, dh, _pitch(qkv), ldh, _stream()), "xl_split_qkv")


def xl_split_heads(src, dst, H, dh):
    """src [rows, >= H*dh] (row stride src.stride(0)) -> dst [H, rows, dh]."""
    rows = src.shape[0]
    _count(1)
    N.check(N.lib().rp_xl_split_heads(_dtc(src), _ptr(src), src.stride(0), _dtc(dst), _ptr(dst), rows, H, dh,
                                      _pitch(dst), _stream()), "xl_split_heads")


def xl_merge_heads(src, dst, H, dh):
    """src [H, rows, dh] -> dst [rows, H*dh] (row stride dst.stride(0))."""
    rows = dst.shape[0]
    _count(1)
    N.check(N.lib().rp_xl_merge_heads(_dtc(src), _ptr(src), _dtc(dst), _ptr(dst), dst.stride(0), rows, H, dh,
                                      _pitch(src), _stream()), "xl_merge_heads")


def xl_merge_grads(g_qu, g_qv, g_kh, g_vh, g_qkv, B, T, M, H, dh):
    """Head-major gradients -> g_qkv rows: dQu, dQv fp32 (one row pitch),
    dK, dV in g_qkv's dtype (one row pitch)."""
    ldg, ldkv = _pitch(g_qu), _pitch(g_kh)
    if _pitch(g_qv) != ldg or _pitch(g_vh) != ldkv:
        raise DimensionError("xl_merge_grads: dQu / dQv and dK / dV each share one row pitch")
    if g_qu.dtype != torch.float32 or g_qv.dtype != torch.float32 or g_kh.dtype != g_qkv.dtype or \
            g_vh.dtype != g_qkv.dtype:
        raise DimensionError("xl_merge_grads: dQu / dQv fp32, dK / dV in the dtype of g_qkv")
    _count(1)
    N.check(N.lib().rp_xl_merge_grads(_dtc(g_qkv), _ptr(g_qu), _ptr(g_qv), _ptr(g_kh), _ptr(g_vh), _ptr(g_qkv), B, T,
                                      M, H, dh, _pitch(g_qkv), ldg, ldkv, _stream()), "xl_merge_grads")


def xl_softmax_fwd(ac, bd, probs, T, M, mem_len, scale):
    """ac, bd fp32 [rows, lds]; probs [rows, ldp]; rows = H*B*T."""
    _count(1)
    rows = math.prod(probs.shape[:-1])
    N.check(N.lib().rp_xl_softmax_fwd(_dtc(probs), _ptr(ac), _ptr(bd), ac.stride(-2), _ptr(probs), probs.stride(-2),
                                      rows, T, M, mem_len, scale, _stream()), "xl_softmax_fwd")


def xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, mem_len, scale):
    """Fused scores + softmax (bf16, dh = 64): qu, qv [H*B*T, dh] head-major,
    kh [H*B*Kl, dh], rh [H*Kl, dh]; probs [H*B, T, ldp]."""
    _require_cuda(qu, qv, kh, rh, probs)
    for t in (qu, qv, kh, rh, probs):
        if t.dtype != torch.bfloat16:
            raise DimensionError("xl_attn_fwd takes bf16 tensors")
    for t in (qu, qv, kh, rh):
        if not t.is_contiguous():
            raise DimensionError("xl_attn_fwd operands must be contiguous")
    H, dh = rh.shape[0], rh.shape[-1]
    _count(1)
    N.check(N.lib().rp_xl_attn_fwd(_ptr(qu), _ptr(qv), _ptr(kh), _ptr(rh), _ptr(probs), probs.stride(-2), B, T, M,
                                   H, dh, mem_len, scale, _stream()), "xl_attn_fwd")


def xl_attn_bwd(g_ctx_h, vh, probs, g_ac, g_bd, g_ctx, ctx, B, T, M, mem_len, scale):
    """Fused softmax backward (bf16, dh = 64): g_ctx_h [H*B*T, dh] head-major,
    vh [H*B*Kl, dh], probs / g_ac / g_bd [H*B, T, ldp]; g_ctx, ctx merged
    [B*T, H*dh] rows (D_i = <g_ctx_i, ctx_i>)."""
    _require_cuda(g_ctx_h, vh, probs, g_ac, g_bd, g_ctx, ctx)
    for t in (g_ctx_h, vh, probs, g_ac, g_bd, g_ctx, ctx):
        if t.dtype != torch.bfloat16:
            raise DimensionError("xl_attn_bwd takes bf16 tensors")
    for t in (g_ctx_h, vh, g_ctx, ctx):
        if not t.is_contiguous():
            raise DimensionError("xl_attn_bwd operands must be contiguous")
    ldp = probs.stride(-2)
    if g_ac.stride(-2) != ldp or g_bd.stride(-2) != ldp:
        raise DimensionError("xl_attn_bwd: P, dAC and dBD must share the row pitch")
    H, dh = g_ctx.shape[-1] // vh.shape[-1], vh.shape[-1]
    _count(1)
    N.check(N.lib().rp_xl_attn_bwd(_ptr(g_ctx_h), _ptr(vh), _ptr(probs), _ptr(g_ac), _ptr(g_bd), ldp, _ptr(g_ctx),
                                   _ptr(ctx), B, T, M, H, dh, mem_len, scale, _stream()), "xl_attn_bwd")


def padded(t):
    """The view of a row-pitched tensor over its full pitch (pad columns included)."""
    ld = _pitch(t)
    if ld == t.shape[-1]:
        return t
    return t.as_strided(tuple(t.shape[:-1]) + (ld,), t.stride())


def xl_attn_fwd_pv(qu, qv, kh, vh, rh, probs, ctx, B, T, M, mem_len, scale):
    """xl_attn_fwd plus ctx = P v: qu / qv [H*B*T, dh], kh / vh [H*B*(M+T),
    dh], rh [H, M+T, dh] head-major; probs [H*B, T, ldp]; ctx the merged
    [B*T, H*dh] rows.  The kernel's head dim is 64: a smaller model head dim
    rides in rows pitched at 64 whose pad columns are zero (XLTape)."""
    _require_cuda(qu, qv, kh, vh, rh, probs, ctx)
    for t in (qu, qv, kh, vh, rh, probs, ctx):
        if t.dtype != torch.bfloat16:
            raise DimensionError("xl_attn_fwd_pv takes bf16 tensors")
    H, dh = rh.shape[0], rh.shape[-1]
    ops_in = [padded(t) for t in (qu, qv, kh, vh, rh)]
    for t in ops_in:
        if not t.is_contiguous() or t.shape[-1] != 64:
            raise DimensionError("xl_attn_fwd_pv operands: contiguous rows of 64 (head dims < 64 zero-padded)")
    _count(1)
    N.check(N.lib().rp_xl_attn_fwd_pv(*[_ptr(t) for t in ops_in], _ptr(probs), probs.stride(-2), _ptr(ctx), B, T, M, H,
                                      64, mem_len, scale, dh, _pitch(ctx), _stream()), "xl_attn_fwd_pv")


def xl_attn_bwd_dq(g_ctx_h, vh, kh, rh, probs, g_ac, g_bd, g_ctx, ctx, g_qu, g_qv, B, T, M, mem_len, scale,
                   bias_part=None, d_rows=None, g_qkv=None):
    """xl_attn_bwd plus the query gradients on the tensor cores (dh = 64,
    T % 128 == 0): g_qu = dAC kh, g_qv = dBD r_h written as fp32 [H*B*T, dh].
    g_ac None: dAC is not written (xl_attn_bwd_kv forms dK itself); d_rows:
    fp32 [H*B*T] receives D_i = <g_ctx_i, ctx_i> for xl_attn_bwd_kv.  g_qkv
    (with g_ac None and d_rows): bf16(dQu + dQv) straight into the merged
    [B*(M+T), 3d] query-gradient columns instead of g_qu / g_qv (then None)."""
    _require_cuda(g_ctx_h, vh, kh, rh, probs, g_bd, g_ctx, ctx)
    if g_qkv is not None:
        _require_cuda(g_qkv)
        if g_qkv.dtype != torch.bfloat16 or not g_qkv.is_contiguous():
            raise DimensionError("xl_attn_bwd_dq: g_qkv is contiguous bf16 [B*(M+T), 3d]")
    else:
        _require_cuda(g_qu, g_qv)
    if d_rows is not None and (d_rows.dtype != torch.float32 or d_rows.numel() < g_ctx_h.shape[0] * g_ctx_h.shape[1]
                               or not d_rows.is_contiguous()):
        raise DimensionError("xl_attn_bwd_dq: d_rows is a contiguous fp32 [H*B*T] buffer")
    for t in (g_ctx_h, vh, kh, rh, probs, g_bd, g_ctx, ctx) + ((g_ac,) if g_ac is not None else ()):
        if t.dtype != torch.bfloat16:
            raise DimensionError("xl_attn_bwd_dq takes bf16 operands")
    for t in (g_qu, g_qv):
        if t is not None and (t.dtype != torch.float32 or not t.is_contiguous()):
            raise DimensionError("xl_attn_bwd_dq writes contiguous fp32 query gradients")
    for t in (g_ctx_h, vh, kh, rh, g_ctx, ctx):
        if not t.is_contiguous():
            raise DimensionError("xl_attn_bwd_dq operands must be contiguous")
    ldp = probs.stride(-2)
    if (g_ac is not None and g_ac.stride(-2) != ldp) or g_bd.stride(-2) != ldp:
        raise DimensionError("xl_attn_bwd_dq: P, dAC and dBD must share the row pitch")
    H, dh = g_ctx.shape[-1] // vh.shape[-1], vh.shape[-1]
    _count(2 if d_rows is not None and g_ac is None and N.lib().rp_xl_dq_persistent() else 1)  # + the D-rows kernel
    N.check(N.lib().rp_xl_attn_bwd_dq(_ptr(g_ctx_h), _ptr(vh), _ptr(kh), _ptr(rh), _ptr(probs), _ptr(g_ac),
                                      _ptr(g_bd), ldp, _ptr(g_ctx), _ptr(ctx), _ptr(g_qu), _ptr(g_qv), B, T, M, H, dh,
                                      mem_len, scale, _ptr(bias_part), _ptr(d_rows), _ptr(g_qkv), _stream()),
            "xl_attn_bwd_dq")


def xl_attn_bwd_kv(g_ctx_h, vh, qu, probs, d_rows, g_kh, g_vh, B, T, M, mem_len, scale, g_qkv=None):
    """Key-major dK / dV (dh = 64, T % 128 == 0; after xl_attn_bwd_dq with
    d_rows): g_vh = P^T g_ctx_h and g_kh = dS^T qu as bf16 [H*B, M+T, dh],
    bitwise the banded GEMMs over P and dAC.  g_qkv: into the merged
    [B*(M+T), 3d] key / value columns instead (g_kh / g_vh None), the memory
    rows' query columns zeroed."""
    outs = (g_qkv,) if g_qkv is not None else (g_kh, g_vh)
    _require_cuda(g_ctx_h, vh, qu, probs, d_rows, *outs)
    for t in (g_ctx_h, vh, qu, probs) + outs:
        if t.dtype != torch.bfloat16:
            raise DimensionError("xl_attn_bwd_kv takes bf16 operands")
    for t in (g_ctx_h, vh, qu, d_rows) + outs:
        if not t.is_contiguous():
            raise DimensionError("xl_attn_bwd_kv operands must be contiguous")
    if d_rows.dtype != torch.float32:
        raise DimensionError("xl_attn_bwd_kv: d_rows is fp32")
    dh = vh.shape[-1]
    H = vh.numel() // (B * (M + T) * dh)
    _count(1)
    N.check(N.lib().rp_xl_attn_bwd_kv(_ptr(g_ctx_h), _ptr(vh), _ptr(qu), _ptr(probs), probs.stride(-2), _ptr(d_rows),
                                      _ptr(g_kh), _ptr(g_vh), B, T, M, H, dh, mem_len, scale, _ptr(g_qkv), _stream()),
            "xl_attn_bwd_kv")


def xl_dq_bias_part_elems(H, B, T):
    return N.lib().rp_xl_dq_bias_part_bytes(H, B, T) // 4


def xl_dq_bias_finish(part, g_u, g_v, H, B, T):
    """r_w_bias / r_r_bias gradients from xl_attn_bwd_dq's per-CTA column sums."""
    _count(1)
    N.check(N.lib().rp_xl_dq_bias_finish(_ptr(part), _ptr(g_u), _ptr(g_v), H, B, T, _stream()), "xl_dq_bias_finish")


def gelu(z, y):
    """y = GELU(z) = 0.5 z (1 + erf(z / sqrt 2)) (same dtype and size)."""
    _require_cuda(z, y)
    if z.dtype != y.dtype or z.shape != y.shape or _pitch(z) != _pitch(y):
        raise DimensionError("gelu takes two tensors of one dtype, shape and row pitch")
    # pitched rows (pad_cols): the elementwise pass runs over the padded extent
    # (pad columns are never read by the GEMMs)
    n = _rows(z) * _pitch(z) if z.dim() >= 2 else z.numel()
    _count(1)
    N.check(N.lib().rp_gelu_fwd(_dtc(z), _ptr(z), _ptr(y), n, _stream()), "gelu")


def axpy(y, x, alpha=1.0):
    """y += alpha * x (fp32, same element count)."""
    _require_cuda(y, x)
    if y.dtype != torch.float32 or x.dtype != torch.float32 or y.numel() != x.numel():
        raise DimensionError("axpy takes two fp32 tensors of one size")
    _count(1)
    N.check(N.lib().rp_axpy(_ptr(y), _ptr(x), alpha, y.numel(), _stream()), "axpy")


def rows_copy(src, dst, cols=None, val=None, val_const=0.0, aug=False):
    """dst[r, :cols] = src[r, :cols]; with aug, dst[r, cols] = val[r] (or val_const); zeros to dst's width."""
    _require_cuda(src, dst)
    rows = dst.shape[0]
    cols = src.shape[-1] if cols is None else cols
    if src.shape[0] != rows:
        raise DimensionError("rows_copy: row counts differ")
    _count(1)
    N.check(N.lib().rp_rows_copy(_dtc(src), _ptr(src), src.stride(0), rows, cols, _ptr(val), val_const, int(aug),
                                 _dtc(dst), _ptr(dst), dst.stride(0), _stream()), "rows_copy")


def rows_gather(src, idx, dst):
    _require_cuda(src, idx, dst)
    _count(1)
    N.check(N.lib().rp_rows_gather(_dtc(src), _ptr(src), src.stride(0), _ptr(idx), idx.numel(), src.shape[-1],
                                   _ptr(dst), dst.stride(0), _stream()), "rows_gather")


def rows_scatter_add(src, idx, dst):
    _require_cuda(src, idx, dst)
    _count(1)
    N.check(N.lib().rp_rows_scatter_add(_ptr(src), src.stride(0), _ptr(idx), idx.numel(), src.shape[-1], _ptr(dst),
                                        dst.stride(0), _stream()), "rows_scatter_add")


def xl_softmax_bwd(g_p, probs, g_ac, g_bd, T, M, mem_len, scale):
    _count(1)
    rows = math.prod(probs.shape[:-1])
    N.check(N.lib().rp_xl_softmax_bwd(_dtc(probs), _ptr(g_p), g_p.stride(-2), _ptr(probs), probs.stride(-2),
                                      _ptr(g_ac), _ptr(g_bd), rows, T, M, mem_len, scale, _stream()),
            "xl_softmax_bwd")


def xl_bias_grad(g_qu, g_qv, work, g_u, g_v, H, rows, dh):
    ldg = _pitch(g_qu)
    if _pitch(g_qv) != ldg:
        raise DimensionError("xl_bias_grad: dQu and dQv share one row pitch")
    _count(2)
    N.check(N.lib().rp_xl_bias_grad(_ptr(g_qu), _ptr(g_qv), _ptr(work), _ptr(g_u), _ptr(g_v), H, rows, dh, ldg,
                                    _stream()), "xl_bias_grad")


def embed_fwd(tokens, tied, pos, out, vocab, dropout=None, flag=None):
    B, T = tokens.shape
    d = tied.shape[1]
    seed, thr, scale = dropout if dropout is not None else (0, 0, 1.0)
    _count(1)
    ld = _pitch(out)
    if _pitch(tied) != ld or _pitch(pos) != ld:
        raise DimensionError("embed_fwd: V, the position table and the output share one row pitch")
    N.check(N.lib().rp_embed_fwd(_dtc(out), _ptr(tokens), _ptr(tied), _ptr(pos), _ptr(out), B, T, d, vocab, seed,
                                 thr, scale, int(dropout is not None), _ptr(flag), ld, _stream()), "embed_fwd")


def embed_bwd(grad, tokens, t_max, grad_pos, emb_grad, beta, work, dropout=None):
    B, T = tokens.shape
    d = grad.shape[-1]
    seed, thr, scale = dropout if dropout is not None else (0, 0, 1.0)
    # ids outside [0, vocab) are skipped by the scatter (the forward flagged them)
    vocab = emb_grad.shape[0] if emb_grad is not None else 1
    if not grad.is_contiguous():
        raise DimensionError("embed_bwd: the gradient rows must be contiguous")
    ld = _pitch(grad_pos) if grad_pos is not None else _pitch(emb_grad)
    if emb_grad is not None and grad_pos is not None and _pitch(emb_grad) != ld:
        raise DimensionError("embed_bwd: the position and tied gradients share one row pitch")
    _count(4)
    N.check(N.lib().rp_embed_bwd(_ptr(grad), _ptr(tokens), B, T, t_max, d, vocab, seed, thr, scale,
                                 int(dropout is not None), _ptr(grad_pos), _ptr(emb_grad), beta, _ptr(work),
                                 ld, _stream()), "embed_bwd")


def ce_finish(partial, target_logit, targets, vocab, lse, loss_rows, loss, loss64=None, flag=None):
    rows, ntiles = partial.shape[0], partial.shape[1]
    _count(2)
    N.check(N.lib().rp_ce_finish(_ptr(partial), ntiles, _ptr(target_logit), _ptr(targets), vocab, rows, _ptr(lse),
                                 _ptr(loss_rows), _ptr(loss), _ptr(loss64), _ptr(flag), _stream()), "ce_finish")


def adam_step(w, g, m, v, copy, n, lr, b1, b2, eps, c1, c2, flag=None):
    cd = _dtc(copy) if copy is not None else N.F32
    _count(1)
    N.check(N.lib().rp_adam_step(_ptr(w), _ptr(g), _ptr(m), _ptr(v), _ptr(copy), cd, n, lr, b1, b2, eps, c1, c2,
                                 _ptr(flag), _stream()), "adam_step")


def sgd_step(w, g, copy, n, lr, flag=None):
    cd = _dtc(copy) if copy is not None else N.F32
    _count(1)
    N.check(N.lib().rp_sgd_step(_ptr(w), _ptr(g), _ptr(copy), cd, n, lr, _ptr(flag), _stream()), "sgd_step")


def init_uniform(out, seed, pos0, scale):
    _count(1)
    N.check(N.lib().rp_init_uniform(_ptr(out), out.numel(), seed & ((1 << 64) - 1), pos0, float(scale), _stream()),
            "init_uniform")


def cast(src, dst):
    _count(1)
    N.check(N.lib().rp_cast(_ptr(src), _dtc(src), _ptr(dst), _dtc(dst), src.numel(), _stream()), "cast")


def sq_norm(x, part, out, accumulate=False):
    _count(2)
    N.check(N.lib().rp_sq_norm(_ptr(x), x.numel(), _ptr(part), _ptr(out), int(accumulate), _stream()), "sq_norm")
