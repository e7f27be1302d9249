"""Widths that are not multiples of 8 -- BASELINE.json configs[3]'s d 410 =
10 heads x 41 and d_ff 2100 -- on the device.  bf16 rows of those widths are
not 16-byte multiples, so every bf16 matrix keeps its rows at a padded pitch
(layers.pad_cols); the kernels take the pitch.  Checked against the fp64
restatements (oracle/xl.py, oracle/adaptive.py) with the tolerances of
tests/test_xl_gpu.py / tests/test_adaptive_gpu.py: fp32 check mode rel-L2
<= 2e-5 (block), bf16 <= 1e-2 (forward) / 3e-2 (gradients)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import adaptive as A  # noqa: E402
from oracle import xl as X  # noqa: E402
from oracle.rng import Stream  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def host(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_c4_shape_xl_block_matches_restatement(dtype):
    """One XL block at the published configs[3] widths (d 410, 10 x 41, d_ff
    2100), memory full, dropout on."""
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD

    B, T, M, H, d, f = 2, 24, 24, 10, 410, 2100
    stack = MD.build_xl_stack(64, d, f, 1, T, 0.1, 3, H, M, dtype=dtype, cutoffs=[16, 40])
    st = stack.storage[1]
    st.configure_ring(1)
    st.ensure(0)
    W = st.weights(0)
    cdt = stack.cdtype
    if cdt == torch.bfloat16:
        assert W["wqkv"].stride(0) == 1232 and W["w1"].stride(0) == 2104 and W["w2"].stride(0) == 416
    P = {k: host(v) for k, v in st._public(W).items()}
    rs = Stream(17)
    x = torch.from_numpy(rs.uniform_signed((B, T, d), 1.0)).to(cdt).double().numpy()
    mem = torch.from_numpy(rs.uniform_signed((B, M, d), 1.0)).to(cdt).double().numpy()
    gout = rs.uniform_signed((B, T, d), 1.0)
    dev = stack.runtime.device
    tp = XD.XLTape(B, T, M, d, f, H, cdt, dev)
    tp.mem.copy_(torch.from_numpy(mem.reshape(B * M, d)))
    tp.x.copy_(torch.from_numpy(x.reshape(B * T, d)))
    tp.mem_len = M
    R = XD.sinusoid(M + T, d, cdt, dev)
    ws = LY.Workspace(dev)
    drop = LY.Dropout.make(1234, 0.1, True)
    out = LY.empty_rows(B * T, d, dtype=cdt, device=dev)
    XD.xl_block_forward(W, W, out, tp, R, drop, ws, stack.runtime.flag)
    g = torch.from_numpy(gout.reshape(B * T, d)).float().to(dev)
    gx = torch.empty_like(g)
    XD.xl_block_backward(W, W, tp, R, g, gx, st.G, drop, ws)
    torch.cuda.synchronize()
    ref, cache = X.xl_block_fwd(P, x, mem, M, H, 1234, 0.1, True)
    if cdt == torch.bfloat16:
        # ReLU kinks: a bf16 pre-activation within rounding of 0 flips the
        # mask, and each flip moves a whole d_ff gradient entry (rel-L2 ~
        # sqrt(flip fraction), ~4% here).  The gradients are compared with the
        # device's mask forced onto the restatement (as tests/test_production_gpu.py)
        on = host(tp.h1).reshape(B, T, f) > 0.0
        z1 = np.abs(cache["z1"]) + 1e-300
        cache["z1"] = np.where(on, z1, -z1)
    rgx, RG = X.xl_block_bwd(P, cache, gout)
    tf, tg = (2e-5, 1e-4) if dtype == "fp32" else (1e-2, 3e-2)
    assert rel(host(out).reshape(B, T, d), ref) <= tf
    assert rel(host(gx).reshape(B, T, d), rgx) <= tg
    grads = {k: host(v) for k, v in st.grads.items()}
    for k, want in RG.items():
        assert rel(grads[k], want) <= tg, (k, rel(grads[k], want))
    # the pad columns of the gradient buffer are never written
    if cdt == torch.bfloat16:
        flat = st.flat_grad[st.n_vec:]
        for _, off, r, c, pc in st.mat_blocks():
            assert not flat[off: off + r * pc].view(r, pc)[:, c:].any()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_adaptive_head_at_d410_matches_restatement(dtype):
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200.adaptive import AdaptiveHead

    N, d, vocab, cutoffs = 300, 410, 1200, [200, 520, 1000]
    r = np.random.default_rng(7)
    h = r.normal(size=(N, d)) * 0.5
    V = r.normal(size=(vocab, d)) * 0.3
    n = len(A.clusters(cutoffs, vocab))
    Wc, bc = r.normal(size=(n, d)) * 0.3, r.normal(size=n) * 0.2
    y = np.minimum((r.pareto(1.2, size=N) * cutoffs[0] / 4).astype(np.int64), vocab - 1)
    y[0] = vocab - 1
    cdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    dev = "cuda"
    hd = LY.empty_rows(N, d, dtype=cdt, device=dev)
    hd.copy_(torch.from_numpy(h))
    Vd = LY.empty_rows(vocab, d, dtype=cdt, device=dev)
    Vd.copy_(torch.from_numpy(V))
    Wm = LY.empty_rows(n, d, dtype=cdt, device=dev)
    Wm.copy_(torch.from_numpy(Wc))
    bm = torch.from_numpy(bc).float().to(dev)
    head = AdaptiveHead(vocab, d, cutoffs, dev, cdt)
    loss = head.forward(hd, Vd, Wm, bm, y)
    g_h = torch.empty(N, d, device=dev)
    g_V = torch.full((vocab, d), float("nan"), device=dev)
    g_W = torch.empty(n, d, device=dev)
    g_b = torch.empty_like(bm)
    head.backward(g_h, g_V, g_W, g_b)
    torch.cuda.synchronize()
    rl, rgh, rgV, rgW, rgb = A.adaptive_loss_grad(host(hd), host(Vd), host(Wm), host(bm.to(cdt)), y, cutoffs)
    tl, tg = (1e-5, 1e-4) if dtype == "fp32" else (1e-2, 3e-2)
    assert abs(float(loss) - rl) <= tl * abs(rl), (float(loss), rl)
    assert torch.isfinite(g_V).all()
    for got, want, name in ((g_h, rgh, "h"), (g_V, rgV, "V"), (g_W, rgW, "Wc"), (g_b, rgb, "bc")):
        assert rel(host(got), want) <= tg, (name, rel(host(got), want))


def _pads_zero(stack):
    for st in stack.storage:
        flat = st.flat_master[st.n_vec:]
        for _, off, r, c, pc in st.mat_blocks():
            if pc != c and flat[off: off + r * pc].view(r, pc)[:, c:].any():
                return False
    t = stack.tied_store
    return t.pitch == t.d or not t.flat_master.view(t.vocab, t.pitch)[:, t.d:].any()


@pytest.mark.parametrize("K", [1, 3])
def test_pitched_xl_ouroboros_tracks_restatement(K):
    """Ouroboros steps of an XL model with the adaptive head at widths that
    are not multiples of 8 (d 82 = 2 heads x 41, d_ff 100): fp32 check mode
    against the fp64 restatement (loss rel <= 2e-5, packet rel-L2 <= 2e-4),
    bf16 (pitched rows) tracking it (loss rel <= 2e-2), the concurrent
    executor bitwise equal to the reference executor in bf16, and the pad
    columns of every master staying zero under Adam.

    The trajectories use SGD: Adam's first updates are lr * g / (|g| + eps),
    so a gradient entry that is ~0 relative to its tensor moves by a full
    +-lr on whichever side of zero rounding puts it, and a multi-step
    comparison then measures that amplification, not the kernels (measured:
    Adam trajectories drift to 5e-2 by step 2 at d 32 and d 82 alike while
    lr 1e-9 or SGD stay at 1e-5; tests/test_teacher_forced_gpu.py covers Adam
    one step at a time)."""
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200.data import SegmentStream
    from oracle import ouroboros as OO

    vocab, d, f, blocks, T, M, H, B, p, cut = 96, 82, 100, 3, 16, 16, 2, 2, 0.1, [24, 56]
    lr = 0.05
    toks = (Stream(2).uniform((B * 8 * T + 4,)) * vocab).astype(np.int64)
    src = SegmentStream(toks, T, B)

    def make(dtype, concurrent=False, opt="sgd"):
        stack = MD.build_xl_stack(vocab, d, f, blocks, T, p, 5, H, M, dtype=dtype, cutoffs=cut)
        cls = E.ConcurrentPipelineEngine if concurrent and K > 1 else E.PipelineEngine
        return stack, cls(stack, MD.partition(stack.num_layers, K), 9), O.make_optimizer(
            opt, O.LrSchedule(lr if opt == "sgd" else 2e-3, "fixed"))

    V, layers = X.init_xl_params(vocab, d, f, blocks, T, H, 5, cutoffs=cut)
    ora = X.XLOuroborosOracle(V, layers, K, 9, p, H, M, B, OO.Sgd(lambda t: lr), cutoffs=cut)
    s32, e32, o32 = make("fp32")
    s16, e16, o16 = make("bf16")
    sc, ec, oc = make("bf16", concurrent=True)
    sa, ea, oa = make("bf16", opt="adam")
    assert s16.tied_store.pitch == 88
    for t in range(5):
        b = src.batch_at(t)
        packet, loss = e32.step(t, b, o32)
        got = packet.cpu()
        oloss, opk = ora.step(t, b.x, b.y)
        assert abs(loss - oloss) <= 2e-5 * abs(oloss), (t, loss, oloss)
        for k in range(K):
            for key, want in opk["module_grads"][k].items():
                g = got.module_grads[k][key]
                if np.any(want):
                    assert rel(g, want) <= 2e-4, (t, k, key, rel(g, want))
        if np.any(opk["emb_grad"]):
            assert rel(got.emb_grad, opk["emb_grad"]) <= 2e-4
        p16, l16 = e16.step(t, b, o16)
        c16 = p16.cpu()
        pc, lc = ec.step(t, b, oc)
        assert l16 == lc, (t, l16, lc)
        assert np.array_equal(c16.emb_grad, pc.cpu().emb_grad)
        assert abs(l16 - oloss) <= 2e-2 * abs(oloss), (t, l16, oloss)
        _, la = ea.step(t, b, oa)
        assert np.isfinite(la)
    torch.cuda.synchronize()
    assert _pads_zero(s16) and _pads_zero(sc) and _pads_zero(sa)


def test_dense_row_composites_reject_pitched_widths():
    """The C-ABI composites (one call per block / module) take dense bf16 rows
    and say so; the pitched widths run through the op-level entry points."""
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD
    from paper_1909_06695_b200.errors import DimensionError

    B, T, M, H, d, f = 1, 16, 16, 2, 82, 100
    stack = MD.build_xl_stack(64, d, f, 1, T, 0.1, 3, H, M, dtype="bf16", cutoffs=[16, 40])
    st = stack.storage[1]
    st.configure_ring(1)
    st.ensure(0)
    W = st.weights(0)
    dev = stack.runtime.device
    tp = XD.XLTape(B, T, M, d, f, H, torch.bfloat16, dev)
    tp.xa.zero_()
    out = LY.empty_rows(B * T, d, dtype=torch.bfloat16, device=dev)
    with pytest.raises(DimensionError, match="dense bf16 rows"):
        XD.xl_block_forward_native(W, W, out, tp, XD.sinusoid(M + T, d, torch.bfloat16, dev), None,
                                   LY.Workspace(dev), stack.runtime.flag)
    with pytest.raises(DimensionError, match="adaptive head"):
        MD.build_xl_stack(64, d, f, 1, T, 0.1, 3, H, M, dtype="bf16")


def test_fused_forward_takes_zero_padded_head_dims():
    """Head dim 41 rides zero-padded to 64 through xl_attn_fwd_pv: P and
    ctx = P v equal the unfused GEMM + softmax path within one bf16 rounding,
    and the block output within the bf16 tolerance."""
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD

    B, T, M, H, d, f = 2, 150, 150, 10, 410, 2100
    stack = MD.build_xl_stack(64, d, f, 1, T, 0.1, 3, H, M, dtype="bf16", cutoffs=[16, 40])
    st = stack.storage[1]
    st.configure_ring(1)
    st.ensure(0)
    W = st.weights(0)
    dev = stack.runtime.device
    g = torch.Generator(device=dev).manual_seed(4)
    xa = (torch.rand(B * (M + T), d, device=dev, generator=g) * 2 - 1).bfloat16()
    R = XD.sinusoid(M + T, d, torch.bfloat16, dev)
    drop = LY.Dropout.make(99, 0.1, True)
    res = []
    saved = XD.FUSED_PV
    try:
        for fused in (False, True):
            XD.FUSED_PV = fused
            tp = XD.XLTape(B, T, M, d, f, H, torch.bfloat16, dev)
            assert tp.dhp == 64 and XD.fused_pv_ok(tp) == fused
            LY.copy_rows(tp.xa, xa)
            tp.mem_len = M - 30
            out = LY.empty_rows(B * T, d, dtype=torch.bfloat16, device=dev)
            XD.xl_block_forward_ops(W, W, out, tp, R, drop, LY.Workspace(dev), stack.runtime.flag)
            torch.cuda.synchronize()
            res.append((tp.probs.float().clone(), tp.ctx.float().clone(), out.float().clone()))
    finally:
        XD.FUSED_PV = saved
    (p0, c0, o0), (p1, c1, o1) = res
    assert (p1 - p0).abs().max().item() <= 2 ** -8 * max(p0.abs().max().item(), 1e-3)
    assert ((c1 - c0).norm() / c0.norm()).item() <= 1e-2
    assert ((o1 - o0).norm() / o0.norm()).item() <= 1e-2
