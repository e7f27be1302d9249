"""tcgen05 GEMM parity: every operand major-ness, both arithmetic modes, ragged
shapes, batching and each fused epilogue, against fp64 torch references.

The contraction replaces reference kernels.mm/bmm (kernels.py:68-81); the
epilogues restate layers.py:184-195 (bias/dropout/residual, bias/ReLU) and
layers.py:310-319 (logsumexp and softmax-CE gradient)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.rng import dropout_scale_mask, keep_threshold  # noqa: E402


def _ops():
    from paper_1909_06695_b200 import ops

    return ops


def _mk(shape, dtype, dev, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).to(dev)


def _ref(a, b, a_mn, b_mn):
    a64 = a.double()
    b64 = b.double()
    A = a64.transpose(-1, -2) if a_mn else a64
    B = b64 if b_mn else b64.transpose(-1, -2)
    return A @ B


def _rel(x, y):
    return (x.double() - y.double()).norm().item() / max(y.double().norm().item(), 1e-30)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(256, 512, 512), (200, 136, 72), (128, 64, 1024), (8, 8, 8)])
def test_gemm_majors(dev, dtype, a_mn, b_mn, shape):
    ops = _ops()
    M, Nn, K = shape
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    a = _mk((K, M) if a_mn else (M, K), dt, dev, 1)
    b = _mk((K, Nn) if b_mn else (Nn, K), dt, dev, 2)
    c = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, out_dtype=torch.float32)
    ref = _ref(a, b, a_mn, b_mn)
    # bf16: exact products, fp32 accumulation.  tf32x3: ~fp32 operands; the
    # tensor-core accumulation error grows with K (measured 6e-6 @512, 1.1e-5 @1024)
    tol = 1e-5 if dtype == "bf16" else max(2e-6, 2e-5 * K / 1024)
    assert _rel(c, ref) < tol


@pytest.mark.parametrize("tile_n", [64, 128, 256])
def test_gemm_batched_tiles(dev, tile_n):
    ops = _ops()
    a = _mk((3, 300, 160), torch.bfloat16, dev, 3)
    b = _mk((3, 260, 160), torch.bfloat16, dev, 4)
    c = ops.gemm(a, b, out_dtype=torch.float32, tile_n=tile_n)
    assert _rel(c, _ref(a, b, False, False)) < 1e-5


def test_gemm_strided_views(dev):
    # q/k/v are column slices of one [N, 3d] projection buffer
    ops = _ops()
    qkv = _mk((2, 64, 3 * 96), torch.float32, dev, 5)
    q, k = qkv[..., :96], qkv[..., 96:192]
    s = ops.gemm(q, k, alpha=0.25)
    ref = 0.25 * (q.double() @ k.double().transpose(-1, -2))
    assert _rel(s, ref) < 2e-6


def test_bf16_out(dev):
    ops = _ops()
    a = _mk((512, 256), torch.bfloat16, dev, 6)
    b = _mk((384, 256), torch.bfloat16, dev, 7)
    c = ops.gemm(a, b)
    assert c.dtype == torch.bfloat16
    assert _rel(c, _ref(a, b, False, False)) < 5e-3


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_bias_relu(dev, dtype):
    ops = _ops()
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    a = _mk((300, 128), dt, dev, 8)
    w = _mk((128, 520), dt, dev, 9)  # [K, N] as stored by the reference (w1)
    bias = _mk((520,), torch.float32, dev, 10)
    from paper_1909_06695_b200 import _native as N

    out = ops.gemm(a, w, b_mn=True, epilogue=N.EPI_BIAS_RELU, bias=bias, out_dtype=torch.float32)
    ref = torch.clamp(_ref(a, w, False, True) + bias.double(), min=0)
    assert _rel(out, ref) < (1e-5 if dtype == "bf16" else 2e-6)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_bias_dropout_residual(dev, dtype):
    ops = _ops()
    from paper_1909_06695_b200 import _native as N

    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    M, K, Nn, p, seed, pos0 = 4 * 33, 96, 160, 0.2, 0xDEADBEEF12345, 777
    a = _mk((M, K), dt, dev, 11)
    w = _mk((K, Nn), dt, dev, 12)
    bias = _mk((Nn,), torch.float32, dev, 13)
    resid = _mk((M, Nn), dt, dev, 14)
    out = ops.gemm(
        a, w, b_mn=True, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=bias, residual=resid,
        dropout=(seed, keep_threshold(p), 1.0 / (1.0 - p), pos0), out_dtype=dt,
    )
    mask = torch.from_numpy(dropout_scale_mask(seed, pos0, (M, Nn), p)).to(dev)
    ref = resid.double() + (_ref(a, w, False, True) + bias.double()) * mask
    # exact zeros where the mask drops
    dropped = mask == 0
    assert torch.all(out.double()[dropped] == resid.double()[dropped])
    assert _rel(out, ref) < (5e-3 if dtype == "bf16" else 2e-6)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_lse_partial_and_ce_grad(dev, dtype):
    ops = _ops()
    from paper_1909_06695_b200 import _native as N

    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    M, d, V = 200, 64, 1000
    h = _mk((M, d), dt, dev, 15) * 3
    tied = _mk((V, d), dt, dev, 16)
    y = torch.randint(0, V, (M,), device=dev, generator=None)
    bn = ops.gemm_tile_n(V, M)
    nt = (V + bn - 1) // bn
    partial = torch.empty((M, 2 * nt, 2), dtype=torch.float32, device=dev)  # per tile and column half
    zy = torch.empty((M,), dtype=torch.float32, device=dev)
    ops.gemm(h, tied, epilogue=N.EPI_LSE_PARTIAL, targets=y, partial=partial, target_logit=zy)
    mx = partial[..., 0].max(dim=1).values
    lse = mx + torch.log((partial[..., 1] * torch.exp(partial[..., 0] - mx[:, None])).sum(dim=1))
    z = _ref(h, tied, False, False)
    lse_ref = torch.logsumexp(z, dim=1)
    assert (lse.double() - lse_ref).abs().max().item() < 1e-4
    assert (zy.double() - z[torch.arange(M), y]).abs().max().item() < 1e-4
    dz = ops.gemm(h, tied, epilogue=N.EPI_CE_GRAD, targets=y, lse=lse, ce_scale=1.0 / M, out_dtype=torch.float32)
    p = torch.softmax(z, dim=1)
    p[torch.arange(M), y] -= 1.0
    assert _rel(dz, p / M) < 1e-4


@pytest.mark.parametrize("off", [-512, -300, 0, 200])
def test_banded_a_skips_zero_k_blocks_bitwise(off):
    """k_lo_off: op(A) row m is zero for k < m + off (the causal window of the
    XL attention matrices); tiles skip those k-blocks -- the result is bitwise
    the dense GEMM's (the skipped products are exact zeros)."""
    from paper_1909_06695_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(9)
    HB, Kl, T, dh = 6, 1024, 512, 64
    P = torch.rand(HB, T, Kl, device="cuda", generator=g).to(torch.bfloat16)
    i = torch.arange(T, device="cuda")[:, None]
    j = torch.arange(Kl, device="cuda")[None, :]
    P = P.masked_fill(i < j + off, 0)  # A = P^T: row j is zero for k = i < j + off
    G = (torch.randn(HB, T, dh, device="cuda", generator=g)).to(torch.bfloat16)
    dense = ops.gemm(P, G, a_mn=True, b_mn=True, out_dtype=torch.float32)
    band = ops.gemm(P, G, a_mn=True, b_mn=True, out_dtype=torch.float32, k_lo_off=off)
    assert torch.equal(dense, band)
    want = P.float().transpose(1, 2) @ G.float()
    assert float((band - want).norm() / want.norm()) <= 1e-5


def test_batched_split_k_matches_dense_and_is_deterministic():
    """Split-K over a batch of matrices (the XL dR GEMM: 8 heads x 8 key tiles,
    K = 11264 queries): partials [split][matrix], one fixed-order reduce over
    batch*M rows; equal to fp64 within the bf16-operand GEMM tolerance and
    bitwise reproducible."""
    import torch

    from paper_1909_06695_b200 import _native as N
    from paper_1909_06695_b200 import ops

    H, Kl, R, dh = 8, 1024, 11264, 64
    g = torch.Generator(device="cuda").manual_seed(3)
    a = (torch.randn(H, R, Kl, device="cuda", generator=g) * 0.3).bfloat16()
    b = (torch.randn(H, R, dh, device="cuda", generator=g) * 0.3).bfloat16()
    assert N.lib().rp_gemm_choose_splits(Kl, dh, R, H, ops.SPLITK_CAP) > 1
    out = torch.empty(H, Kl, dh, device="cuda")
    ops.gemm(a, b, a_mn=True, b_mn=True, out=out)
    out2 = torch.empty_like(out)
    ops.gemm(a, b, a_mn=True, b_mn=True, out=out2)
    ref = torch.einsum("hrk,hrn->hkn", a.double(), b.double())
    err = ((out.double() - ref).norm() / ref.norm()).item()
    assert err <= 1e-5, err
    assert torch.equal(out, out2)
