"""Transformer-XL blocks on the device against the fp64 restatement
(oracle/xl.py; parity unpinned at the reference, which has no XL path).

fp32 check mode, stated tolerances: block outputs / gradients rel-L2 <= 2e-5
(layer level, one call); Ouroboros free run over segment streams with
memory: loss rel <= 2e-5, packet tensors rel-L2 <= 2e-4 (as the reference
model's parity test, tests/test_engine_gpu.py)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ouroboros as OO  # noqa: E402
from oracle import xl as X  # noqa: E402
from oracle.rng import Stream  # noqa: E402

CFG = dict(vocab=64, d=32, f=64, blocks=2, seq=8, mem=8, heads=4, batch=2, p=0.1, init_seed=5, dseed=9)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def host(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("T,M,mem_len,H,d", [(8, 8, 8, 4, 32), (8, 8, 0, 4, 32), (12, 6, 6, 2, 32), (8, 8, 5, 1, 32),
                                             (10, 6, 6, 2, 80)])
def test_xl_block_matches_restatement(T, M, mem_len, H, d):
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD

    B, f = 2, 48
    stack = MD.build_xl_stack(40, d, f, 1, T, 0.2, 3, H, M, dtype="fp32")
    st = stack.storage[1]
    W = st._carve(None, None, None, st.master[: st.n_vec], st.master[st.n_vec:])
    P = {k: host(v) for k, v in st.params.items()}
    rs = Stream(17)
    x = rs.uniform_signed((B, T, d), 1.0)
    mem = rs.uniform_signed((B, M, d), 1.0)
    gout = rs.uniform_signed((B, T, d), 1.0)
    dev = stack.runtime.device
    tp = XD.XLTape(B, T, M, d, f, H, torch.float32, dev)
    tp.mem.copy_(torch.from_numpy(mem.reshape(B * M, d)))
    tp.x.copy_(torch.from_numpy(x.reshape(B * T, d)))
    tp.mem_len = mem_len
    R = XD.sinusoid(M + T, d, torch.float32, dev)
    ws = LY.Workspace(dev)
    drop = LY.Dropout.make(1234, 0.2, True)
    out = torch.empty(B * T, d, device=dev)
    XD.xl_block_forward(W, W, out, tp, R, drop, ws, stack.runtime.flag)
    ref, cache = X.xl_block_fwd(P, x, mem, mem_len, H, 1234, 0.2, True)
    assert rel(host(out).reshape(B, T, d), ref) <= 2e-5
    g = torch.from_numpy(gout.reshape(B * T, d)).float().to(dev)
    gx = torch.empty_like(g)
    XD.xl_block_backward(W, W, tp, R, g, gx, st.G, drop, ws)
    rgx, RG = X.xl_block_bwd(P, cache, gout)
    assert rel(host(gx).reshape(B, T, d), rgx) <= 2e-5
    grads = {k: host(v) for k, v in st.grads.items()}
    for k, want in RG.items():
        assert rel(grads[k], want) <= 2e-5, (k, rel(grads[k], want))


def make_pair(K, lr, dtype="fp32", concurrent=False):
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import optim as O

    c = CFG
    stack = MD.build_xl_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], c["init_seed"], c["heads"],
                              c["mem"], dtype=dtype)
    part = MD.partition(stack.num_layers, K)
    eng = (E.ConcurrentPipelineEngine if concurrent else E.PipelineEngine)(stack, part, c["dseed"])
    gopt = O.make_optimizer("adam", O.LrSchedule(lr, "fixed"))
    V, layers = X.init_xl_params(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["heads"], c["init_seed"])
    ora = X.XLOuroborosOracle(V, layers, K, c["dseed"], c["p"], c["heads"], c["mem"], c["batch"],
                              OO.Adam(lambda t: lr))
    return stack, eng, gopt, ora


def segments(n):
    from paper_1909_06695_b200.data import SegmentStream

    c = CFG
    toks = (Stream(2).uniform((c["batch"] * (n + 1) * c["seq"] + 4,)) * c["vocab"]).astype(np.int64)
    return SegmentStream(toks, c["seq"], c["batch"])


def test_init_matches_restatement():
    c = CFG
    stack, _, _, ora = make_pair(2, 1e-3)
    assert rel(host(stack.tied), ora.V) <= 1e-7  # fp32 masters of the fp64 draw
    for idx, P in enumerate(ora.layers):
        for k, want in P.items():
            assert rel(host(stack.params[idx][k]), want) <= 1e-7, (idx, k)


@pytest.mark.parametrize("K", [1, 2, 4])
def test_xl_ouroboros_free_run_matches_restatement(K):
    stack, eng, gopt, ora = make_pair(K, 2e-3)
    src = segments(6)
    for t in range(6):
        b = src.batch_at(t)
        packet, loss = eng.step(t, b, gopt)
        got = packet.cpu()
        oloss, opk = ora.step(t, b.x, b.y)
        assert abs(loss - oloss) <= 2e-5 * abs(oloss), (t, loss, oloss)
        for k in range(K):
            for key, want in opk["module_grads"][k].items():
                g = got.module_grads[k][key]
                if not np.any(want):
                    assert not np.any(g), (t, k, key)
                else:
                    assert rel(g, want) <= 2e-4, (t, k, key, rel(g, want))
        if np.any(opk["emb_grad"]):
            assert rel(got.emb_grad, opk["emb_grad"]) <= 2e-4


def test_xl_concurrent_bitwise_equals_reference_executor_and_bf16_tracks():
    from paper_1909_06695_b200.engine import BatchSample  # noqa: F401

    _, e1, o1, _ = make_pair(3, 2e-3, dtype="bf16")
    _, e2, o2, ora = make_pair(3, 2e-3, dtype="bf16", concurrent=True)
    src = segments(8)
    for t in range(8):
        b = src.batch_at(t)
        p1, l1 = e1.step(t, b, o1)
        c1 = p1.cpu()
        p2, l2 = e2.step(t, b, o2)
        c2 = p2.cpu()
        assert l1 == l2
        assert np.array_equal(c1.emb_grad, c2.emb_grad)
        oloss, _ = ora.step(t, b.x, b.y)
        assert abs(l1 - oloss) <= 2e-2 * abs(oloss)


def test_by_cost_times_xl_blocks_and_the_adaptive_head():
    """measure_layer_costs times Transformer-XL blocks as XL blocks
    (attention over a full memory) and the adaptive head as the adaptive head,
    so by_cost partitions of the XL configs balance real costs."""
    from paper_1909_06695_b200 import model as MD

    stack = MD.build_xl_stack(2000, 64, 128, 4, 32, 0.1, 3, 4, 32, dtype="bf16", cutoffs=[104, 504])
    x = (Stream(1).uniform((4, 32)) * 2000).astype(np.int64)
    costs = MD.measure_layer_costs(stack, x, dropout_seed=3)
    assert len(costs) == stack.num_layers and all(c > 0 for c in costs)
    blocks = costs[1:-1]
    # the four XL blocks are the same work: within 2x of each other
    assert max(blocks) <= 2.0 * min(blocks)
    part = MD.partition(stack.num_layers, 3, "by_cost", costs)
    assert sum(hi - lo for lo, hi in part.groups) == stack.num_layers


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_xl_block_gelu_matches_restatement(dtype):
    """XL block with the GELU FFN option vs the fp64 restatement."""
    from paper_1909_06695_b200 import layers as LY
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import xl as XD

    B, T, M, H, d, f = 2, 128, 128, 2, 128, 256
    stack = MD.build_xl_stack(40, d, f, 1, T, 0.2, 3, H, M, dtype=dtype, activation="gelu")
    st = stack.storage[1]
    st.configure_ring(1)
    st.ensure(0)
    W = st.weights(0)
    P = {k: host(v) for k, v in st._public(W).items()}
    rs = Stream(17)
    x = rs.uniform_signed((B, T, d), 1.0)
    mem = rs.uniform_signed((B, M, d), 1.0)
    gout = rs.uniform_signed((B, T, d), 1.0)
    cdt = stack.cdtype
    x = torch.from_numpy(x).to(cdt).double().numpy()
    mem = torch.from_numpy(mem).to(cdt).double().numpy()
    dev = stack.runtime.device
    tp = XD.XLTape(B, T, M, d, f, H, cdt, dev, activation="gelu")
    tp.mem.copy_(torch.from_numpy(mem.reshape(B * M, d)))
    tp.x.copy_(torch.from_numpy(x.reshape(B * T, d)))
    tp.mem_len = M
    R = XD.sinusoid(M + T, d, cdt, dev)
    ws = LY.Workspace(dev)
    drop = LY.Dropout.make(1234, 0.2, True)
    out = torch.empty(B * T, d, device=dev, dtype=cdt)
    XD.xl_block_forward(W, W, out, tp, R, drop, ws, stack.runtime.flag)
    g = torch.from_numpy(gout.reshape(B * T, d)).float().to(dev)
    gx = torch.empty_like(g)
    XD.xl_block_backward(W, W, tp, R, g, gx, st.G, drop, ws)
    torch.cuda.synchronize()
    ref, cache = X.xl_block_fwd(P, x, mem, M, H, 1234, 0.2, True, act="gelu")
    rgx, RG = X.xl_block_bwd(P, cache, gout)
    tf, tg = (2e-5, 1e-4) if dtype == "fp32" else (1e-2, 3e-2)
    assert rel(host(out).reshape(B, T, d), ref) <= tf
    assert rel(host(gx).reshape(B, T, d), rgx) <= tg
    grads = {k: host(v) for k, v in st.grads.items()}
    for k, want in RG.items():
        assert rel(grads[k], want) <= tg, (k, rel(grads[k], want))
