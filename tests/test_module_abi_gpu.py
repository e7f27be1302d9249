"""The module-level C ABI (rp_module_forward / rp_module_backward) against
the per-layer host loop the engines use: same kernels in the same order, so
activations, stale-slot tapes, the loss, every parameter gradient, the
boundary gradient and the tied gradient must agree bitwise."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VOCAB, D, F, BLOCKS, T, B = 96, 32, 64, 4, 16, 3


def build(dtype, K):
    from paper_1909_06695_b200 import model as M

    stack = M.build_stack(VOCAB, D, F, BLOCKS, T, 0.1, 5, dtype=dtype)
    part = M.partition(stack.num_layers, K)
    return stack, M.build_modules(stack, part, dropout_seed=9)


def clone_tape(arena):
    out = [t.clone() for t in arena.acts]
    for tp in arena.tapes:
        out += [tp.a.clone(), tp.qkv.clone(), tp.probs_buf.clone(), tp.ctx.clone(), tp.x1.clone(), tp.m.clone(),
                tp.h1.clone(), tp.mean1.clone(), tp.rstd1.clone(), tp.mean2.clone(), tp.rstd2.clone()]
    return out


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_module_abi_bitwise_equals_host_loop(dtype):
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import module_abi as MA
    from paper_1909_06695_b200.model import StaleSlot, _Arena

    stack, mods = build(dtype, 3)
    dev = stack.runtime.device
    g = torch.Generator(device=dev).manual_seed(3)
    tokens = torch.randint(0, VOCAB, (B, T), device=dev, generator=g)
    targets = torch.randint(0, VOCAB, (B * T,), device=dev, generator=g)
    step = 4
    for m in mods:
        m.snapshot(step)
        seeds = [m._layer_seed(step, i) for i in range(len(m.layers))]
        arenas = [_Arena(m, B, T), _Arena(m, B, T)]
        outs = [None, None]
        for a in arenas:
            if m.has_embedding:
                a.tokens.copy_(tokens)
            else:
                a.acts[0].copy_((torch.rand(B * T, D, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
                                 * 2 - 1).to(a.acts[0].dtype))
            if m.has_projection:
                a.targets.copy_(targets)
        if not m.has_projection:
            outs = [torch.empty(B * T, D, dtype=stack.cdtype, device=dev) for _ in range(2)]
        ws = [LY.Workspace(dev), LY.Workspace(dev)]
        r0 = m._run_forward(step, arenas[0], seeds, True, outs[0], ws[0], live=False)
        r1 = MA.forward(m, arenas[1], step, seeds, True, outs[1], ws[1])
        assert torch.equal(r0, r1), m.index
        for x, y in zip(clone_tape(arenas[0]), clone_tape(arenas[1])):
            assert torch.equal(x, y), m.index
        # delayed backward: boundary gradient in, parameter / boundary / tied gradients out
        g_out = None if m.has_projection else torch.rand(B * T, D, device=dev, generator=g) - 0.5
        alpha = 0.5 if m.has_projection else 0.0
        beta = 0.5 if m.has_embedding else 0.0
        results = []
        for path in range(2):
            tied = torch.full((VOCAB, D), 0.25, device=dev)
            g_in = None if m.has_embedding else torch.empty(B * T, D, device=dev)
            m.zero_grads()
            if path == 0:
                slot = StaleSlot(step, step, None, None, seeds, arenas[0])
                m.recompute_backward(slot, g_out, "snapshot", True, g_in=g_in, emb=(alpha, beta, tied))
            else:
                MA.backward(m, arenas[1], step, seeds, True, g_out, g_in, tied, alpha, beta, True, ws[1])
            grads = {k: v.clone() for k, v in m.grad_views.items()}
            results.append((grads, tied.clone(), None if g_in is None else g_in.clone()))
        (ga, ta, ia), (gb, tb, ib) = results
        for k in ga:
            assert torch.equal(ga[k], gb[k]), (m.index, k)
        assert torch.equal(ta, tb), m.index
        if ia is not None:
            assert torch.equal(ia, ib), m.index


def test_module_abi_rejects_bad_descriptors():
    from paper_1909_06695_b200 import _native as N

    dsc = N.ModuleDesc()
    dsc.B, dsc.T, dsc.d, dsc.n_heads, dsc.M, dsc.mem_len = 1, 1, 8, 3, 4, 0  # heads do not divide d
    assert N.lib().rp_module_forward(dsc, None, None, None, None, 0, None, None) != 0
    dsc = N.ModuleDesc()
    dsc.B, dsc.T, dsc.d = 1, 1, 8
    assert N.lib().rp_module_forward(dsc, None, None, None, None, 0, None, None) != 0
    assert np.isscalar(N.lib().rp_module_workspace_bytes(dsc))


def test_embedding_gradient_kernel_matches_reference_rule():
    """rp_embedding_gradient vs the reference rule (engine.py:54-69)."""
    from paper_1909_06695_b200.engine import embedding_gradient
    from paper_1909_06695_b200.errors import ScheduleViolation

    dev = torch.device("cuda")
    vo = torch.rand(7, 8, device=dev) - 0.5
    vi = torch.rand(7, 8, device=dev) - 0.5
    for conv, c in (("half_avg", 0.5), ("sum", 1.0)):
        got = embedding_gradient(5, 3, vo, vi, conv)
        assert torch.equal(got, c * vo + c * vi)
        host = embedding_gradient(5, 3, vo.cpu().numpy(), vi.cpu().numpy(), conv)
        np.testing.assert_array_equal(got.cpu().numpy(), host)
    assert not embedding_gradient(0, 3, vo, None).any()
    with pytest.raises(ScheduleViolation):
        embedding_gradient(0, 3, vo, vi)
    with pytest.raises(ScheduleViolation):
        embedding_gradient(4, 3, vo, None)


def _xl_tape_tensors(tp):
    out = []
    for n in ("xa", "a", "qkv", "qu", "qv", "kh", "vh", "rh", "probs_buf", "ctx", "x1", "m", "h1", "z1", "mean1",
              "rstd1", "mean2", "rstd2"):
        v = getattr(tp, n, None)
        if v is not None:
            out.append(v.clone())
    return out


@pytest.mark.parametrize("dtype,act", [("fp32", "relu"), ("bf16", "relu"), ("bf16", "gelu")])
def test_xl_block_abi_bitwise_equals_host_loop(dtype, act):
    """rp_xl_block_forward / _backward (one C call per Transformer-XL block)
    against the op-by-op host path of xl.py: bitwise equal outputs, tapes and
    gradients -- bf16 at head dim 64 and T % 128 == 0 runs the fused
    forward-with-P.V and backward-with-dQ kernels, fp32 the GEMM + softmax path."""
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD

    B_, T_, M_, H, d, f = 2, 128, 128, 2, 128, 256
    stack = MD.build_xl_stack(64, d, f, 1, T_, 0.1, 3, H, M_, dtype=dtype, activation=act)
    st = stack.storage[1]
    st.configure_ring(1)
    st.ensure(0)
    W = st.weights(0)
    dev = stack.runtime.device
    cdt = stack.cdtype
    g = torch.Generator(device=dev).manual_seed(5)
    xa = ((torch.rand(B_ * (M_ + T_), d, device=dev, generator=g) * 2 - 1)).to(cdt)
    g_out = torch.rand(B_ * T_, d, device=dev, generator=g) - 0.5
    R = XD.sinusoid(M_ + T_, d, cdt, dev)
    drop = LY.Dropout.make(4321, 0.1, True)
    res = []
    for native in (False, True):
        tp = XD.XLTape(B_, T_, M_, d, f, H, cdt, dev, act)
        tp.xa.copy_(xa)
        tp.mem_len = M_ - 20
        ws = LY.Workspace(dev)
        out = torch.empty(B_ * T_, d, dtype=cdt, device=dev)
        gx = torch.empty(B_ * T_, d, device=dev)
        st.grad.zero_()
        if native:
            XD.xl_block_forward_native(W, W, out, tp, R, drop, ws, stack.runtime.flag)
            XD.xl_block_backward_native(W, W, tp, R, g_out, gx, st.G, drop, ws)
        else:
            XD.xl_block_forward_ops(W, W, out, tp, R, drop, ws, stack.runtime.flag)
            XD.xl_block_backward_ops(W, W, tp, R, g_out, gx, st.G, drop, ws)
        torch.cuda.synchronize()
        res.append((out.clone(), gx.clone(), st.grad.clone(), _xl_tape_tensors(tp)))
    a, b = res
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    for u, v in zip(a[3], b[3]):
        assert torch.equal(u, v)
    if dtype == "bf16":
        assert XD.fused_flags(tp) & 15 == 12  # the P.V-fused forward and the dQ-fused backward ran
        assert XD.fused_flags(tp) & XD.N.XL_FUSED_KV  # and the key-major dK / dV kernel


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_xl_module_abi_bitwise_equals_host_loop(dtype):
    """rp_module_forward / rp_module_backward over Transformer-XL modules
    (memory loaded / stored by the host around the call) against the per-layer
    host loop: bitwise equal losses, activations, tapes, memory and gradients."""
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import module_abi as MA
    from paper_1909_06695_b200.model import StaleSlot, _Arena

    V, d, f, nb, T_, M_, H, B_ = 64, 128, 256, 3, 128, 128, 2, 2
    runs = []
    for path in range(2):
        stack = MD.build_xl_stack(V, d, f, nb, T_, 0.1, 5, H, M_, dtype=dtype)
        mods = MD.build_modules(stack, MD.partition(stack.num_layers, 2), dropout_seed=9)
        dev = stack.runtime.device
        g = torch.Generator(device=dev).manual_seed(3)
        rec = []
        for step in range(2):  # the second step sees the first one's memory
            tokens = torch.randint(0, V, (B_, T_), device=dev, generator=g)
            targets = torch.randint(0, V, (B_ * T_,), device=dev, generator=g)
            x_next = None
            for m in mods:
                m.snapshot(step)
                seeds = [m._layer_seed(step, i) for i in range(len(m.layers))]
                a = _Arena(m, B_, T_)
                if m.has_embedding:
                    a.tokens.copy_(tokens)
                else:
                    a.acts[0].copy_(x_next)
                if m.has_projection:
                    a.targets.copy_(targets)
                out = None if m.has_projection else torch.empty(B_ * T_, d, dtype=stack.cdtype, device=dev)
                ws = LY.Workspace(dev)
                if path == 0:
                    r = m._run_forward(step, a, seeds, True, out, ws, live=True)
                else:
                    r = MA.forward(m, a, step, seeds, True, out, ws, live=True)
                x_next = out
                rec += [r.clone()] + [t.clone() for t in a.acts] + [t.clone() for tp in a.tapes
                                                                   for t in _xl_tape_tensors(tp)]
                rec += [v.clone() for v in m.mem.values()]
                g_out = None if m.has_projection else torch.linspace(-1, 1, B_ * T_ * d, device=dev).view(-1, d)
                g_in = None if m.has_embedding else torch.empty(B_ * T_, d, device=dev)
                tied = torch.zeros(V, d, device=dev)
                m.zero_grads()
                if path == 0:
                    m.recompute_backward(StaleSlot(step, step, None, None, seeds, a), g_out, "snapshot", True,
                                         g_in=g_in, emb=(0.5, 0.5, tied))
                else:
                    MA.backward(m, a, step, seeds, True, g_out, g_in, tied, 0.5 if m.has_projection else 0.0,
                                0.5 if m.has_embedding else 0.0, True, ws)
                rec += [v.clone() for v in m.grad_views.values()] + [tied.clone()]
                if g_in is not None:
                    rec.append(g_in.clone())
        torch.cuda.synchronize()
        runs.append(rec)
    assert len(runs[0]) == len(runs[1])
    for i, (u, v) in enumerate(zip(*runs)):
        assert torch.equal(u, v), i
