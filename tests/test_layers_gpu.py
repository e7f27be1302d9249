"""Native layer composites (csrc/layers.cpp) vs the same op sequence issued
from Python (layers.*_ops): bitwise equal outputs, tapes and gradients, for
both arithmetic modes, with dropout on and off.  Plus the block/head against
fp64 torch autograd-free references built from the oracle."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import layers as OL  # noqa: E402


def _setup(dtype, B=2, T=24, d=64, f=128, seed=0):
    from paper_1909_06695_b200 import layers as LY

    g = torch.Generator().manual_seed(seed)
    dev = "cuda"
    cdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    r = lambda *s, sc=0.2: (torch.rand(*s, generator=g, dtype=torch.float64) * 2 - 1).mul(sc)  # noqa: E731
    W = {"wqkv": r(d, 3 * d), "wo": r(d, d), "w1": r(d, f), "w2": r(f, d)}
    V = {"ln1_g": 1 + r(d), "ln1_b": r(d), "ln2_g": 1 + r(d), "ln2_b": r(d), "b1": r(f), "b2": r(d)}
    x = r(B * T, d, sc=1.0)
    Wd = {k: v.to(cdt).to(dev).contiguous() for k, v in W.items()}
    Wd.update({k: v.float().to(dev) for k, v in V.items()})
    xd = x.to(cdt).to(dev)
    return LY, Wd, xd, (W, V, x), B, T, d, f, cdt


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("train", [True, False])
def test_native_block_equals_op_sequence(dtype, train):
    LY, W, x, _, B, T, d, f, cdt = _setup(dtype)
    drop = LY.Dropout.make(0xABCDEF, 0.2, train)
    outs = []
    for fwd, bwd in ((LY.block_forward, LY.block_backward), (LY.block_forward_ops, LY.block_backward_ops)):
        ws = LY.Workspace(x.device)
        tape = LY.BlockTape(B, T, d, f, cdt, x.device)
        out = torch.empty_like(x)
        fwd(W, W, x, out, tape, B, T, drop, ws, None)
        g_out = torch.linspace(-1, 1, x.numel(), device=x.device).view_as(x).float()
        g_x = torch.empty_like(g_out)
        G = {k: torch.empty(v.shape, dtype=torch.float32, device=x.device) for k, v in W.items()}
        bwd(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
        torch.cuda.synchronize()
        outs.append((out.clone(), tape.h1.clone(), g_x.clone(), {k: v.clone() for k, v in G.items()}))
    a, b = outs
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    for k in a[3]:
        assert torch.equal(a[3][k], b[3][k]), k


def test_native_block_fp32_vs_oracle():
    LY, W, x, (W64, V64, x64), B, T, d, f, cdt = _setup("fp32", B=2, T=20, d=32, f=64, seed=3)
    seed, p = 1234567, 0.15
    drop = LY.Dropout.make(seed, p, True)
    ws = LY.Workspace(x.device)
    tape = LY.BlockTape(B, T, d, f, cdt, x.device)
    out = torch.empty_like(x)
    LY.block_forward(W, W, x, out, tape, B, T, drop, ws, None)
    g_out = torch.linspace(-1, 1, x.numel(), device=x.device).view_as(x).float()
    g_x = torch.empty_like(g_out)
    G = {k: torch.empty(v.shape, dtype=torch.float32, device=x.device) for k, v in W.items()}
    LY.block_backward(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
    P = dict(V64)
    P = {k: v.numpy() for k, v in P.items()}
    w = W64["wqkv"].numpy()
    P.update(wq=w[:, :d], wk=w[:, d:2 * d], wv=w[:, 2 * d:], wo=W64["wo"].numpy(), w1=W64["w1"].numpy(),
             w2=W64["w2"].numpy())
    xo = x64.numpy().reshape(B, T, d).astype(np.float32).astype(np.float64)
    ro, c = OL.block_fwd(P, xo, seed, p, True)
    rgx, RG = OL.block_bwd(P, c, g_out.double().cpu().numpy().reshape(B, T, d))
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)  # noqa: E731
    assert rel(out.double().cpu().numpy().reshape(B, T, d), ro) < 2e-6
    assert rel(g_x.double().cpu().numpy().reshape(B, T, d), rgx) < 2e-5
    gw = G["wqkv"].double().cpu().numpy()
    for name, ref in (("wq", RG["wq"]), ("wk", RG["wk"]), ("wv", RG["wv"])):
        off = {"wq": 0, "wk": d, "wv": 2 * d}[name]
        assert rel(gw[:, off:off + d], ref) < 2e-5, name
    for name in ("wo", "w1", "w2", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"):
        assert rel(G[name].double().cpu().numpy(), RG[name]) < 2e-5, name


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_native_head_equals_ops_and_oracle(dtype):
    from paper_1909_06695_b200 import layers as LY

    g = torch.Generator().manual_seed(7)
    Nt, d, V = 96, 32, 1003  # odd vocab exercises the padded dz rows
    cdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    h64 = torch.rand(Nt, d, generator=g, dtype=torch.float64) * 2 - 1
    t64 = torch.rand(V, d, generator=g, dtype=torch.float64) * 2 - 1
    y = torch.randint(0, V, (Nt,), generator=g)
    h, tied, yd = h64.to(cdt).cuda(), t64.to(cdt).cuda(), y.cuda()
    res = []
    for fwd, bwd in ((LY.head_forward, LY.head_backward), (LY.head_forward_ops, LY.head_backward_ops)):
        ws = LY.Workspace(h.device)
        hs = LY.HeadState(Nt, h.device)
        fwd(h, tied, yd, V, hs, ws, None)
        gh = torch.empty(Nt, d, dtype=torch.float32, device=h.device)
        vo = torch.empty(V, d, dtype=torch.float32, device=h.device)
        bwd(h, tied, yd, V, hs, gh, vo, 0.5, ws)
        torch.cuda.synchronize()
        res.append((hs.loss.item(), gh.clone(), vo.clone()))
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1]) and torch.equal(res[0][2], res[1][2])
    loss, rgh, rgv = OL.head_loss_grad(h.double().cpu().numpy()[None], tied.double().cpu().numpy(), y.numpy()[None])
    tol = 2e-3 if dtype == "bf16" else 2e-5
    assert abs(res[0][0] - loss) <= tol * abs(loss)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(res[0][1].double().cpu().numpy(), rgh[0]) < (1e-2 if dtype == "bf16" else 2e-5)
    assert rel(res[0][2].double().cpu().numpy(), 0.5 * rgv) < (1e-2 if dtype == "bf16" else 2e-5)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_gelu_block_native_equals_ops_and_oracle(dtype):
    """The GELU FFN option (north_star's memory-bound GELU kernel + the
    GELU-gradient GEMM epilogue): the native composite is bitwise the op
    sequence, and both match the fp64 block with the exact erf GELU
    (fp32: <= 2e-6 forward, <= 2e-5 gradients; bf16 <= 1e-2 / 3e-2)."""
    LY, W, x, (W64, V64, x64), B, T, d, f, cdt = _setup(dtype, B=2, T=20, d=32, f=64, seed=5)
    seed, p = 7654321, 0.15
    drop = LY.Dropout.make(seed, p, True)
    outs = []
    for fwd, bwd in ((LY.block_forward, LY.block_backward), (LY.block_forward_ops, LY.block_backward_ops)):
        ws = LY.Workspace(x.device)
        tape = LY.BlockTape(B, T, d, f, cdt, x.device, activation="gelu")
        out = torch.empty_like(x)
        fwd(W, W, x, out, tape, B, T, drop, ws, None)
        g_out = torch.linspace(-1, 1, x.numel(), device=x.device).view_as(x).float()
        g_x = torch.empty_like(g_out)
        G = {k: torch.empty(v.shape, dtype=torch.float32, device=x.device) for k, v in W.items()}
        bwd(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
        torch.cuda.synchronize()
        outs.append((out.clone(), g_x.clone(), {k: v.clone() for k, v in G.items()}, g_out))
    a, b = outs
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    for k in a[2]:
        assert torch.equal(a[2][k], b[2][k]), k
    P = {k: v.numpy() for k, v in V64.items()}
    w = W64["wqkv"].to(cdt).double().numpy()
    P.update(wq=w[:, :d], wk=w[:, d:2 * d], wv=w[:, 2 * d:], wo=W64["wo"].to(cdt).double().numpy(),
             w1=W64["w1"].to(cdt).double().numpy(), w2=W64["w2"].to(cdt).double().numpy())
    xo = x.double().cpu().numpy().reshape(B, T, d)
    ro, c = OL.block_fwd(P, xo, seed, p, True, act="gelu")
    rgx, RG = OL.block_bwd(P, c, a[3].double().cpu().numpy().reshape(B, T, d))
    rel = lambda u, v: np.linalg.norm(u - v) / max(np.linalg.norm(v), 1e-30)  # noqa: E731
    tf, tg = (2e-6, 2e-5) if dtype == "fp32" else (1e-2, 3e-2)
    assert rel(a[0].double().cpu().numpy().reshape(B, T, d), ro) < tf
    assert rel(a[1].double().cpu().numpy().reshape(B, T, d), rgx) < tg
    for name in ("wo", "w1", "w2", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"):
        assert rel(a[2][name].double().cpu().numpy(), RG[name]) < tg, name


def test_gelu_kernel_matches_torch():
    from paper_1909_06695_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(2)
    for dt, n, tol in ((torch.bfloat16, 3 * 4096 + 5, 8e-3), (torch.float32, 10001, 1e-6)):
        z = (torch.randn(n, device="cuda", generator=g) * 3).to(dt)
        y = torch.empty_like(z)
        ops.gelu(z, y)
        want = torch.nn.functional.gelu(z.double())
        err = float((y.double() - want).abs().max() / want.abs().max())
        assert err <= tol, (dt, err)
