"""Thin torch-facing wrappers over the C-ABI kernels of libringpipe_b200.so.

Each wrapper validates shapes/dtypes, extracts raw device pointers and the
current CUDA stream, and calls one `rp_*` entry point.  Tensors are borrowed;
outputs are allocated with torch (PyTorch is the device-memory plumbing).
There is deliberately no CPU path: calling these on CPU tensors raises.
"""

import ctypes

import torch

from . import _native as N
from .errors import DimensionError

_DT = {torch.float32: N.F32, torch.bfloat16: N.BF16}


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
    """(hi, lo) with hi = x truncated to tf32, lo = x - hi (both fp32)."""
    _require_cuda(x)
    if x.dtype != torch.float32:
        raise DimensionError("tf32_split takes fp32")
    hi = torch.empty_like(x, memory_format=torch.contiguous_format)
    lo = torch.empty_like(hi)
    cols = x.shape[-1]
    rows = x.numel() // max(cols, 1)
    if x.stride(-1) != 1 or (x.dim() == 3 and x.stride(0) != x.shape[1] * x.stride(1)):
        x = x.contiguous()
    ld = x.stride(-2) if x.dim() >= 2 else cols
    N.check(N.lib().rp_tf32_split(_ptr(x), _ptr(hi), _ptr(lo), rows, cols, ld, cols, _stream()), "tf32_split")
    return hi, lo


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
):
    """C = epilogue(alpha * opA(a) @ opB(b)) on the tcgen05 GEMM.

    a: [M,K] (a_mn=False) or [K,M] (a_mn=True), optionally with a leading
    batch dim.  b: [N,K] (b_mn=False, "B transposed") or [K,N] (b_mn=True).
    bf16 operands run on kind::f16; fp32 operands run the 3-pass tf32 path
    unless math=MATH_TF32.
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
    N.check(N.lib().rp_gemm(ctypes.byref(args), _stream()), "gemm")
    return out


def gemm_tile_n(n):
    return N.lib().rp_gemm_tile_n(n)
