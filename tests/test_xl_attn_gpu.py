"""Fused Transformer-XL attention kernels (csrc/xl_attn.cu) on the device.

Kernel level: P from the fused tcgen05 scores + relative shift + masked
softmax against an fp32 torch evaluation of the same bf16 operands
(oracle/xl.py's score formula): rel-L2 <= 4e-3 (bf16 output rounding is
2^-9 relative), zeros outside the causal / memory-validity window and in the
row padding.  Block level: the bf16 XL block with the fused kernels against
the unfused bf16 path (AC / BD GEMMs + softmax kernels): outputs and every
gradient rel-L2 <= 1e-2; against the fp64 restatement no worse than the
unfused bf16 path (rel-L2 <= max(1.25 x unfused, 3e-2))."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import xl as X  # noqa: E402
from oracle.rng import Stream  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def _pad8(n):
    return (n + 7) // 8 * 8


def ref_probs(qu, qv, kh, rh, B, T, M, mem_len, scale):
    """fp32 P [HB, T, Kl] from bf16 head-major operands."""
    H, Kl, dh = rh.shape
    HB = H * B
    qu, qv = qu.float().view(HB, T, dh), qv.float().view(HB, T, dh)
    kh = kh.float().view(HB, Kl, dh)
    rr = rh.float().repeat_interleave(B, dim=0)  # [HB, Kl, dh]
    ac = qu @ kh.transpose(1, 2)
    bdf = qv @ rr.transpose(1, 2)  # [HB, T, Kl] unshifted
    i = torch.arange(T, device=qu.device)[:, None]
    j = torch.arange(Kl, device=qu.device)[None, :]
    pidx = (T - 1 - i + j).clamp(0, Kl - 1).expand(T, Kl)
    bd = torch.gather(bdf, 2, pidx.unsqueeze(0).expand(HB, T, Kl))
    s = (ac + bd) * scale
    valid = (j >= M - mem_len) & (j <= M + i)
    s = s.masked_fill(~valid, float("-inf"))
    return torch.softmax(s, dim=-1), valid


@pytest.mark.parametrize("dh", [64, 128])
@pytest.mark.parametrize("B,H,T,M,mem_len", [(2, 2, 128, 128, 128), (1, 3, 200, 72, 50), (2, 1, 64, 0, 0),
                                             (1, 2, 256, 256, 100), (2, 8, 512, 512, 512), (1, 2, 100, 28, 28)])
def test_fused_scores_softmax_matches_fp32(B, H, T, M, mem_len, dh):
    from paper_1909_06695_b200 import ops

    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(T + M)
    Kl = M + T
    ldp = _pad8(Kl)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
    qu, qv = mk(H, B * T, dh), mk(H, B * T, dh)
    kh, rh = mk(H, B * Kl, dh), mk(H, Kl, dh)
    probs = torch.full((H * B, T, ldp), float("nan"), device=dev, dtype=torch.bfloat16)
    scale = 1.0 / math.sqrt(dh)
    ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, mem_len, scale)
    torch.cuda.synchronize()
    want, valid = ref_probs(qu, qv, kh, rh, B, T, M, mem_len, scale)
    got = probs[:, :, :Kl].float()
    assert torch.isfinite(probs.float()).all()
    assert rel(got.cpu(), want.cpu()) <= 4e-3
    assert (got[:, ~valid] == 0).all()
    assert (probs[:, :, Kl:] == 0).all()
    # every row sums to 1 up to bf16 rounding
    assert (got.sum(-1) - 1).abs().max().item() <= 2e-2


def test_fused_equals_unfused_softmax_path():
    """Same P as the GEMM (fp32 AC / BD) + rp_xl_softmax_fwd path up to bf16 rounding."""
    from paper_1909_06695_b200 import ops

    dev = "cuda"
    B, H, T, M, mem_len, dh = 2, 4, 256, 256, 200, 64
    g = torch.Generator(device=dev).manual_seed(3)
    Kl, ldp = M + T, _pad8(M + T)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
    qu, qv = mk(H, B * T, dh), mk(H, B * T, dh)
    kh, rh = mk(H, B * Kl, dh), mk(H, Kl, dh)
    scale = 1.0 / math.sqrt(dh)
    p1 = torch.empty(H * B, T, ldp, device=dev, dtype=torch.bfloat16)
    ops.xl_attn_fwd(qu, qv, kh, rh, p1, B, T, M, mem_len, scale)
    ac = torch.empty(H * B, T, ldp, device=dev)[:, :, :Kl]
    bd = torch.empty(H, B * T, ldp, device=dev)[:, :, :Kl]
    ops.gemm(qu.view(H * B, T, dh), kh.view(H * B, Kl, dh), out=ac)
    ops.gemm(qv, rh, out=bd)
    p2 = torch.empty_like(p1)
    ops.xl_softmax_fwd(ac, bd, p2, T, M, mem_len, scale)
    torch.cuda.synchronize()
    d = (p1.float() - p2.float()).abs()
    assert d.max().item() <= 2 ** -7
    assert rel(p1.float().cpu(), p2.float().cpu()) <= 4e-3


def _block(H, T, M, mem_len, fused, monkeypatch, dh=64):
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD

    monkeypatch.setattr(XD, "FUSED", fused)
    B, d, f = 2, dh * H, 128
    stack = MD.build_xl_stack(40, d, f, 1, T, 0.1, 3, H, M, dtype="bf16")
    st = stack.storage[1]
    from paper_1909_06695_b200 import ops

    mat = torch.empty(st.n_mat, dtype=torch.bfloat16, device=st.master.device)
    ops.cast(st.master[st.n_vec:], mat)
    W = st._carve(None, None, None, st.master[: st.n_vec], mat)
    P = {k: v.detach().double().cpu().numpy() for k, v in st.params.items()}
    rs = Stream(17)
    x = rs.uniform_signed((B, T, d), 1.0)
    mem = rs.uniform_signed((B, M, d), 1.0)
    gout = rs.uniform_signed((B, T, d), 1.0)
    dev = stack.runtime.device
    tp = XD.XLTape(B, T, M, d, f, H, torch.bfloat16, dev)
    tp.mem.copy_(torch.from_numpy(mem.reshape(B * M, d)))
    tp.x.copy_(torch.from_numpy(x.reshape(B * T, d)))
    tp.mem_len = mem_len
    R = XD.sinusoid(M + T, d, torch.bfloat16, dev)
    ws = LY.Workspace(dev)
    drop = LY.Dropout.make(1234, 0.1, True)
    out = torch.empty(B * T, d, device=dev, dtype=torch.bfloat16)
    assert XD.fused_ok(tp) == fused
    XD.xl_block_forward(W, W, out, tp, R, drop, ws, stack.runtime.flag)
    g = torch.from_numpy(gout.reshape(B * T, d)).float().to(dev)
    gx = torch.empty_like(g)
    XD.xl_block_backward(W, W, tp, R, g, gx, st.G, drop, ws)
    torch.cuda.synchronize()
    res = {"out": out.float().cpu().numpy().reshape(B, T, d), "gx": gx.cpu().numpy().reshape(B, T, d)}
    res.update({k: v.detach().double().cpu().numpy() for k, v in st.grads.items()})
    return res, (P, x, mem, gout)


@pytest.mark.parametrize("H,T,M,mem_len,dh", [(2, 128, 128, 128, 64), (2, 192, 64, 40, 64), (2, 100, 36, 36, 64),
                                              (2, 128, 128, 100, 128)])
def test_fused_block_tracks_unfused_and_restatement(H, T, M, mem_len, dh, monkeypatch):
    a, (P, x, mem, gout) = _block(H, T, M, mem_len, True, monkeypatch, dh)
    b, _ = _block(H, T, M, mem_len, False, monkeypatch, dh)
    for k in b:
        assert rel(a[k], b[k]) <= 1e-2, (k, rel(a[k], b[k]))
    # against fp64: no worse than the unfused bf16 path (bf16 rounding of the
    # weights / activations dominates both)
    ref, cache = X.xl_block_fwd(P, x, mem, mem_len, H, 1234, 0.1, True)
    rgx, RG = X.xl_block_bwd(P, cache, gout)
    RG = dict(RG, out=ref, gx=rgx)
    for k, want in RG.items():
        ea, eb = rel(a[k], want), rel(b[k], want)
        assert ea <= max(1.25 * eb, 3e-2), (k, ea, eb)


def ref_bwd(probs, g3, vh, gctx, ctx, B, T, M, mem_len, scale, H, dh):
    """fp32 dAC and un-shifted dBD from the same bf16 inputs, D from <g_ctx, ctx>."""
    HB, Kl = H * B, M + T
    P = probs[:, :, :Kl].float()
    dP = g3.float().view(HB, T, dh) @ vh.float().view(HB, Kl, dh).transpose(1, 2)
    D = (gctx.float() * ctx.float()).view(B, T, H, dh).sum(-1).permute(2, 0, 1).reshape(HB, T, 1)
    dS = P * (dP - D) * scale
    i = torch.arange(T, device=P.device)[:, None]
    j = torch.arange(Kl, device=P.device)[None, :]
    dS = dS.masked_fill(~((j >= M - mem_len) & (j <= M + i)), 0.0)
    jj = (j - (T - 1 - i)).expand(T, Kl)  # key index j for every (i, p)
    dBD = torch.gather(dS, 2, jj.clamp(0, Kl - 1).unsqueeze(0).expand(HB, T, Kl))
    dBD = dBD.masked_fill(((jj < 0) | (jj >= Kl)).unsqueeze(0), 0.0)
    return dS, dBD


@pytest.mark.parametrize("dh", [64, 128])
@pytest.mark.parametrize("B,H,T,M,mem_len", [(2, 2, 128, 128, 128), (1, 3, 200, 72, 50), (2, 1, 64, 0, 0),
                                             (1, 2, 256, 256, 100), (2, 8, 512, 512, 512)])
def test_fused_softmax_backward_matches_fp32(B, H, T, M, mem_len, dh):
    from paper_1909_06695_b200 import ops

    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(7 * T + M)
    Kl = M + T
    ldp = _pad8(Kl)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
    qu, qv = mk(H, B * T, dh), mk(H, B * T, dh)
    kh, rh, vh = mk(H, B * Kl, dh), mk(H, Kl, dh), mk(H, B * Kl, dh)
    scale = 1.0 / math.sqrt(dh)
    probs = torch.empty(H * B, T, ldp, device=dev, dtype=torch.bfloat16)
    ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, mem_len, scale)
    g3 = mk(H, B * T, dh)
    gctx = g3.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh).contiguous()
    # ctx = P v (bf16-rounded, as the forward's merged tape row)
    ctx_h = (probs[:, :, :Kl].float() @ vh.float().view(H * B, Kl, dh)).to(torch.bfloat16)
    ctx = ctx_h.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh).contiguous()
    gac = torch.full((H * B, T, ldp), float("nan"), device=dev, dtype=torch.bfloat16)
    gbd = torch.full((H, B * T, ldp), float("nan"), device=dev, dtype=torch.bfloat16)
    ops.xl_attn_bwd(g3, vh, probs, gac, gbd, gctx, ctx, B, T, M, mem_len, scale)
    torch.cuda.synchronize()
    want_ac, want_bd = ref_bwd(probs, g3, vh, gctx, ctx, B, T, M, mem_len, scale, H, dh)
    assert torch.isfinite(gac.float()).all() and torch.isfinite(gbd.float()).all()
    assert rel(gac[:, :, :Kl].float().cpu(), want_ac.cpu()) <= 4e-3
    assert rel(gbd.view(H * B, T, ldp)[:, :, :Kl].float().cpu(), want_bd.cpu()) <= 4e-3
    assert (gac[:, :, Kl:] == 0).all() and (gbd[:, :, Kl:] == 0).all()
    # dBD is a permutation of dAC's row entries (plus zeros)
    assert torch.equal(gac.float().sum(-1), gbd.view(H * B, T, ldp).float().sum(-1)) or \
        rel(gac.float().sum(-1).cpu(), gbd.view(H * B, T, ldp).float().sum(-1).cpu()) <= 1e-5


def test_fused_xl_engine_tracks_restatement():
    """Ouroboros K=2 over segment streams with memory, bf16, head dim 64 (the
    fused kernels run in every block): loss within the bf16 production
    tolerance of the fp64 restatement, and the multi-stream executor stays
    bitwise equal to the single-stream one."""
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200 import xl as XD
    from paper_1909_06695_b200.data import SegmentStream
    from oracle import ouroboros as OO

    vocab, d, f, blocks, T, M, H, B, p = 64, 128, 256, 2, 16, 16, 2, 2, 0.1
    lr = 2e-3

    def make(concurrent):
        stack = MD.build_xl_stack(vocab, d, f, blocks, T, p, 5, H, M, dtype="bf16")
        eng = (E.ConcurrentPipelineEngine if concurrent else E.PipelineEngine)(stack, MD.partition(stack.num_layers, 2), 9)
        return stack, eng, O.make_optimizer("adam", O.LrSchedule(lr, "fixed"))

    s1, e1, o1 = make(False)
    s2, e2, o2 = make(True)
    V, layers = X.init_xl_params(vocab, d, f, blocks, T, H, 5)
    ora = X.XLOuroborosOracle(V, layers, 2, 9, p, H, M, B, OO.Adam(lambda t: lr))
    toks = (Stream(2).uniform((B * 8 * T + 4,)) * vocab).astype(np.int64)
    src = SegmentStream(toks, T, B)
    assert XD.FUSED
    for t in range(6):
        b = src.batch_at(t)
        p1, l1 = e1.step(t, b, o1)
        c1 = p1.cpu()
        p2, l2 = e2.step(t, b, o2)
        c2 = p2.cpu()
        assert l1 == l2
        assert np.array_equal(c1.emb_grad, c2.emb_grad)
        oloss, _ = ora.step(t, b.x, b.y)
        assert abs(l1 - oloss) <= 2e-2 * abs(oloss), (t, l1, oloss)


def test_fused_backward_rejects_unaligned_segment_length():
    """T % 8 != 0 would put dBD chunk stores off 16-byte alignment: the C ABI
    refuses (DimensionError) and the block falls back to the unfused backward."""
    from paper_1909_06695_b200 import ops
    from paper_1909_06695_b200.errors import DimensionError

    B, H, T, M, dh = 1, 1, 100, 28, 64
    Kl, dev = M + T, "cuda"
    ldp = _pad8(Kl)
    z = lambda *s: torch.zeros(*s, device=dev, dtype=torch.bfloat16)  # noqa: E731
    with pytest.raises(DimensionError):
        ops.xl_attn_bwd(z(H, B * T, dh), z(H, B * Kl, dh), z(H * B, T, ldp), z(H * B, T, ldp), z(H, B * T, ldp),
                        z(B * T, H * dh), z(B * T, H * dh), B, T, M, M, dh ** -0.5)


@pytest.mark.parametrize("B,H,T,M,mem_len", [(2, 2, 128, 128, 128), (1, 2, 256, 256, 100), (2, 1, 128, 0, 0),
                                             (1, 3, 384, 128, 60), (2, 8, 512, 512, 512)])
def test_fused_dq_backward_equals_fused_backward_plus_gemms(B, H, T, M, mem_len):
    """xl_attn_bwd_dq: dAC / dBD bitwise equal to xl_attn_bwd's, and the
    in-kernel query gradients dQu = dAC k, dQv = dBD r (tcgen05, dS kept in
    shared memory) against fp32 torch products of the same bf16 matrices
    (exact bf16 products, fp32 sums: rel-L2 <= 1e-5)."""
    from paper_1909_06695_b200 import ops

    dev, dh = "cuda", 64
    g = torch.Generator(device=dev).manual_seed(11 * T + M + mem_len)
    Kl = M + T
    ldp = _pad8(Kl)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
    qu, qv = mk(H, B * T, dh), mk(H, B * T, dh)
    kh, rh, vh = mk(H, B * Kl, dh), mk(H, Kl, dh), mk(H, B * Kl, dh)
    scale = 1.0 / math.sqrt(dh)
    probs = torch.empty(H * B, T, ldp, device=dev, dtype=torch.bfloat16)
    ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, mem_len, scale)
    g3 = mk(H, B * T, dh)
    gctx = g3.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh).contiguous()
    ctx_h = (probs[:, :, :Kl].float() @ vh.float().view(H * B, Kl, dh)).to(torch.bfloat16)
    ctx = ctx_h.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh).contiguous()
    nan = lambda *s: torch.full(s, float("nan"), device=dev, dtype=torch.bfloat16)  # noqa: E731
    gac1, gbd1 = nan(H * B, T, ldp), nan(H, B * T, ldp)
    gac2, gbd2 = nan(H * B, T, ldp), nan(H, B * T, ldp)
    gqu = torch.full((H, B * T, dh), float("nan"), device=dev)
    gqv = torch.full((H, B * T, dh), float("nan"), device=dev)
    ops.xl_attn_bwd(g3, vh, probs, gac1, gbd1, gctx, ctx, B, T, M, mem_len, scale)
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, gac2, gbd2, gctx, ctx, gqu, gqv, B, T, M, mem_len, scale)
    torch.cuda.synchronize()
    assert torch.equal(gac1, gac2)
    assert torch.equal(gbd1, gbd2)
    want_qu = gac2[:, :, :Kl].float() @ kh.view(H * B, Kl, dh).float()
    want_qv = gbd2.view(H, B * T, ldp)[:, :, :Kl].float() @ rh.float()
    assert rel(gqu.view(H * B, T, dh).cpu(), want_qu.cpu()) <= 1e-5
    assert rel(gqv.cpu(), want_qv.cpu()) <= 1e-5


@pytest.mark.parametrize("B,H,T,M,mem_len", [(2, 2, 128, 128, 128), (1, 3, 200, 72, 50), (2, 1, 64, 0, 0),
                                             (1, 2, 256, 256, 100), (2, 8, 512, 512, 512), (1, 2, 100, 28, 28)])
def test_fused_pv_forward_equals_fused_forward_plus_gemm(B, H, T, M, mem_len):
    """xl_attn_fwd_pv: P bitwise equal to xl_attn_fwd's, and ctx = P v from the
    in-kernel tcgen05 MMA (P tile kept in shared memory) against fp32 torch
    products of the same bf16 P and v, merged to [B*T, H*dh] rows
    (exact bf16 products, fp32 sums, one bf16 rounding: rel-L2 <= 4e-3)."""
    from paper_1909_06695_b200 import ops

    dev, dh = "cuda", 64
    g = torch.Generator(device=dev).manual_seed(3 * T + M + mem_len)
    Kl = M + T
    ldp = _pad8(Kl)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
    qu, qv = mk(H, B * T, dh), mk(H, B * T, dh)
    kh, rh, vh = mk(H, B * Kl, dh), mk(H, Kl, dh), mk(H, B * Kl, dh)
    scale = 1.0 / math.sqrt(dh)
    p1 = torch.full((H * B, T, ldp), float("nan"), device=dev, dtype=torch.bfloat16)
    p2 = torch.full((H * B, T, ldp), float("nan"), device=dev, dtype=torch.bfloat16)
    ctx = torch.full((B * T, H * dh), float("nan"), device=dev, dtype=torch.bfloat16)
    ops.xl_attn_fwd(qu, qv, kh, rh, p1, B, T, M, mem_len, scale)
    ops.xl_attn_fwd_pv(qu, qv, kh, vh, rh, p2, ctx, B, T, M, mem_len, scale)
    torch.cuda.synchronize()
    assert torch.equal(p1, p2)
    want_h = p2[:, :, :Kl].float() @ vh.view(H * B, Kl, dh).float()  # [HB, T, dh]
    want = want_h.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh)
    assert torch.isfinite(ctx.float()).all()
    assert rel(ctx.float().cpu(), want.cpu()) <= 4e-3


@pytest.mark.parametrize("ctas", [0, 3])
@pytest.mark.parametrize("B,H,T,M,mem_len", [(2, 2, 128, 128, 128), (1, 2, 256, 256, 100), (2, 1, 128, 0, 0),
                                             (1, 3, 384, 128, 60), (2, 8, 512, 512, 512), (1, 2, 256, 200, 150)])
def test_fused_kv_backward_equals_banded_gemms(B, H, T, M, mem_len, ctas, monkeypatch):
    """xl_attn_bwd_kv: dV = P^T dO and dK = dS^T (q+u), key-major with dS
    recomputed from P, dP and xl_attn_bwd_dq's D rows, bitwise equal to the
    banded dV / dK GEMMs over P and dAC (the same K = 16 MMA sequence); and
    xl_attn_bwd_dq without dAC leaves dBD / dQu / dQv bitwise unchanged.
    ctas = 3: the persistent kernels (xl_attn_bwd_kv, and xl_attn_bwd_dq
    without dAC) on 3 CTAs, each walking many items with its pipelines
    running across item boundaries -- the no-dAC dq outputs are then those of
    the persistent dq kernel against the one-item kernel's."""
    from paper_1909_06695_b200 import ops

    if ctas:
        monkeypatch.setenv("RP_XL_KV_CTAS", str(ctas))
        monkeypatch.setenv("RP_XL_DQ_CTAS", str(ctas))

    dev, dh = "cuda", 64
    g = torch.Generator(device=dev).manual_seed(7 * T + M + mem_len)
    Kl = M + T
    ldp = _pad8(Kl)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
    qu, qv = mk(H, B * T, dh), mk(H, B * T, dh)
    kh, rh, vh = mk(H, B * Kl, dh), mk(H, Kl, dh), mk(H, B * Kl, dh)
    scale = 1.0 / math.sqrt(dh)
    probs = torch.empty(H * B, T, ldp, device=dev, dtype=torch.bfloat16)
    ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, mem_len, scale)
    g3 = mk(H, B * T, dh)
    gctx = g3.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh).contiguous()
    ctx_h = (probs[:, :, :Kl].float() @ vh.float().view(H * B, Kl, dh)).to(torch.bfloat16)
    ctx = ctx_h.view(H, B * T, dh).permute(1, 0, 2).reshape(B * T, H * dh).contiguous()
    nan = lambda *s: torch.full(s, float("nan"), device=dev, dtype=torch.bfloat16)  # noqa: E731
    nanf = lambda *s: torch.full(s, float("nan"), device=dev)  # noqa: E731
    gac1, gbd1, gbd2 = nan(H * B, T, ldp), nan(H, B * T, ldp), nan(H, B * T, ldp)
    gqu1, gqv1, gqu2, gqv2 = (nanf(H, B * T, dh) for _ in range(4))
    d_rows = nanf(H * B * T)
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, gac1, gbd1, gctx, ctx, gqu1, gqv1, B, T, M, mem_len, scale)
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, None, gbd2, gctx, ctx, gqu2, gqv2, B, T, M, mem_len, scale,
                       d_rows=d_rows)
    gk, gv = nan(H * B, Kl, dh), nan(H * B, Kl, dh)
    g3h, quh = g3.view(H * B, T, dh), qu.view(H * B, T, dh)
    ops.xl_attn_bwd_kv(g3h, vh.view(H * B, Kl, dh), quh, probs, d_rows, gk, gv, B, T, M, mem_len, scale)
    want_v, want_k = nan(H * B, Kl, dh), nan(H * B, Kl, dh)
    ops.gemm(probs[:, :, :Kl], g3h, a_mn=True, b_mn=True, out=want_v, k_lo_off=-M)
    ops.gemm(gac1[:, :, :Kl], quh, a_mn=True, b_mn=True, out=want_k, k_lo_off=-M)
    torch.cuda.synchronize()
    assert torch.equal(gbd1, gbd2)
    assert torch.equal(gqu1, gqu2) and torch.equal(gqv1, gqv2)
    want_d = (gctx.float() * ctx.float()).view(B, T, H, dh).sum(-1).permute(2, 0, 1).reshape(-1)
    assert rel(d_rows.cpu(), want_d.cpu()) <= 1e-5
    assert torch.equal(gv, want_v), (gv.float() - want_v.float()).abs().max().item()
    assert torch.equal(gk, want_k), (gk.float() - want_k.float()).abs().max().item()
    # and against fp32 torch products of the same bf16 matrices (one bf16 rounding)
    fv = probs[:, :, :Kl].float().transpose(1, 2) @ g3h.float()
    fk = gac1[:, :, :Kl].float().transpose(1, 2) @ quh.float()
    assert rel(gv.float().cpu(), fv.cpu()) <= 4e-3
    assert rel(gk.float().cpu(), fk.cpu()) <= 4e-3


@pytest.mark.parametrize("H,T,M,mem_len", [(2, 128, 128, 128), (2, 256, 128, 100)])
def test_fused_kv_block_bitwise_equals_gemm_path(H, T, M, mem_len, monkeypatch):
    """A bf16 XL block with the key-major dK / dV kernel (RP_XL_FUSED_KV) is
    bitwise the block with the banded GEMMs over P and dAC."""
    from paper_1909_06695_b200 import xl as XD

    monkeypatch.setattr(XD, "FUSED_KV", True)
    a, _ = _block(H, T, M, mem_len, True, monkeypatch)
    monkeypatch.setattr(XD, "FUSED_KV", False)
    b, _ = _block(H, T, M, mem_len, True, monkeypatch)
    for k in b:
        assert np.array_equal(a[k], b[k]), (k, rel(a[k], b[k]))
