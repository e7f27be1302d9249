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


def test_module_abi_rejects_xl_and_empty():
    from paper_1909_06695_b200 import _native as N
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import module_abi as MA

    stack = M.build_xl_stack(VOCAB, D, F, 2, T, 0.1, 5, 2, 8, dtype="fp32")
    (m,) = M.build_modules(stack, M.partition(stack.num_layers, 1), dropout_seed=9)
    with pytest.raises(ValueError):
        MA.describe(m, B, T, [0] * 4, True)
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
