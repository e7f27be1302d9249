"""LayerNorm forward / backward kernels (reference layers.py:62-79) at every
model width the BASELINE configs use (d = 128 .. 1024, plus ragged 410 / 640 / 1000)
against fp64 torch: fp32 rel-L2 <= 2e-6, bf16 inputs (fp32 math) <= 2e-6
against fp64 evaluated on the same bf16 inputs."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))


@pytest.mark.parametrize("d", [64, 128, 400, 410, 512, 640, 1000, 1024])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_layernorm_fwd_bwd_matches_fp64(d, dtype):
    from paper_1909_06695_b200 import ops

    rows = 1000 + d % 7  # ragged row tails (the d > 512 kernel pairs warps per row)
    g = torch.Generator(device="cuda").manual_seed(d)
    x = (torch.randn(rows, d, device="cuda", generator=g) * 2 + 0.5).to(dtype)
    gain = 1 + 0.1 * torch.randn(d, device="cuda", generator=g)
    bias = 0.1 * torch.randn(d, device="cuda", generator=g)
    dy = torch.randn(rows, d, device="cuda", generator=g)
    res = torch.randn(rows, d, device="cuda", generator=g)
    y = torch.empty(rows, d, device="cuda", dtype=dtype)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    ops.layernorm_fwd(x, gain, bias, y, mean, rstd)
    nb = ops.layernorm_bwd_blocks(rows)
    pg = torch.empty(nb, d, device="cuda")
    pb = torch.empty(nb, d, device="cuda")
    dx = torch.empty(rows, d, device="cuda")
    ops.layernorm_bwd(dy, x, mean, rstd, gain, dx, pg, pb, resid_grad=res)
    dg = torch.empty(d, device="cuda")
    db = torch.empty(d, device="cuda")
    ops.colsum_finish(pg, nb, dg)
    ops.colsum_finish(pb, nb, db)
    torch.cuda.synchronize()
    # fp64 reference (layers.py:62-79: biased variance, eps 1e-5)
    X = x.double()
    mu = X.mean(-1, keepdim=True)
    var = ((X - mu) ** 2).mean(-1, keepdim=True)
    rs = 1.0 / torch.sqrt(var + 1e-5)
    xh = (X - mu) * rs
    Y = xh * gain.double() + bias.double()
    tol = 2e-6 if dtype == torch.float32 else 4e-3  # bf16 output rounding
    assert rel(y.float(), Y) <= tol
    DY = dy.double()
    dxh = DY * gain.double()
    DX = rs * (dxh - dxh.mean(-1, keepdim=True) - xh * (dxh * xh).mean(-1, keepdim=True)) + res.double()
    assert rel(dx, DX) <= 2e-6
    assert rel(dg, (DY * xh).sum(0)) <= 2e-6
    assert rel(db, DY.sum(0)) <= 2e-6
