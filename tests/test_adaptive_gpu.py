"""Adaptive tied softmax head on the device (paper_1909_06695_b200/adaptive.py)
against the fp64 restatement (oracle/adaptive.py; parity unpinned at the
reference, which has no adaptive softmax).  fp32 check mode (3-pass tf32
GEMMs): loss rel <= 1e-5, every gradient rel-L2 <= 1e-4.  bf16 production:
loss rel <= 1e-2, gradients rel-L2 <= 3e-2 (inputs rounded to bf16 first).
Covers several tails, an empty tail cluster and a cutoff at the vocabulary end."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import adaptive as A  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def _case(N, d, vocab, cutoffs, seed, empty=None):
    r = np.random.default_rng(seed)
    h = r.normal(size=(N, d)) * 0.5
    V = r.normal(size=(vocab, d)) * 0.3
    n = len(A.clusters(cutoffs, vocab))
    Wc = r.normal(size=(n, d)) * 0.3
    bc = r.normal(size=n) * 0.2
    # Zipf-like ids: the head is common, the tails rarer
    y = np.minimum((r.pareto(1.2, size=N) * cutoffs[0] / 4).astype(np.int64), vocab - 1)
    if empty is not None:
        lo, hi = A.clusters(cutoffs, vocab)[empty]
        y[(y >= lo) & (y < hi)] = 0
    y[0] = vocab - 1
    return h, V, Wc, bc, y


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("N,d,vocab,cutoffs,empty", [(256, 64, 1000, [200, 500, 800], None),
                                                     (300, 128, 2048, [512, 1024], 0),
                                                     (128, 64, 600, [96], None)])
def test_adaptive_head_matches_restatement(dtype, N, d, vocab, cutoffs, empty):
    from paper_1909_06695_b200.adaptive import AdaptiveHead

    h, V, Wc, bc, y = _case(N, d, vocab, cutoffs, seed=N + d, empty=empty)
    cdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    dev = "cuda"
    hd = torch.from_numpy(h).to(dev, cdt)
    Vd = torch.from_numpy(V).to(dev, cdt)
    Wm = torch.from_numpy(Wc).float().to(dev)
    bm = torch.from_numpy(bc).float().to(dev)
    head = AdaptiveHead(vocab, d, cutoffs, dev, cdt)
    loss = head.forward(hd, Vd, Wm, bm, y)
    g_h = torch.empty(N, d, device=dev)
    g_V = torch.full((vocab, d), float("nan"), device=dev)
    g_W = torch.empty_like(Wm)
    g_b = torch.empty_like(bm)
    head.backward(g_h, g_V, g_W, g_b)
    torch.cuda.synchronize()
    # reference on the inputs the device saw (bf16-rounded for bf16)
    hr, Vr = hd.double().cpu().numpy(), Vd.double().cpu().numpy()
    Wr = Wm.double().cpu().numpy() if dtype == "fp32" else Wm.bfloat16().double().cpu().numpy()
    br = bm.double().cpu().numpy() if dtype == "fp32" else bm.bfloat16().double().cpu().numpy()
    rl, rgh, rgV, rgW, rgb = A.adaptive_loss_grad(hr, Vr, Wr, br, y, cutoffs)
    tl, tg = (1e-5, 1e-4) if dtype == "fp32" else (1e-2, 3e-2)
    assert abs(float(loss) - rl) <= tl * abs(rl), (float(loss), rl)
    assert torch.isfinite(g_V).all()
    for got, want, name in ((g_h, rgh, "h"), (g_V, rgV, "V"), (g_W, rgW, "Wc"), (g_b, rgb, "bc")):
        assert rel(got.double().cpu().numpy(), want) <= tg, (name, rel(got.double().cpu().numpy(), want))


@pytest.mark.parametrize("K", [1, 2])
def test_xl_ouroboros_with_adaptive_head_matches_restatement(K):
    """Transformer-XL Ouroboros steps with the adaptive tied softmax as the
    projection (fp32 check mode) against the fp64 restatement: loss rel <=
    2e-5, every packet tensor (incl. the cluster weights / biases and the mixed
    tied gradient) rel-L2 <= 2e-4."""
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200.data import SegmentStream
    from oracle import ouroboros as OO
    from oracle import xl as X
    from oracle.rng import Stream

    vocab, d, f, blocks, T, M, H, B, p, cut = 64, 32, 64, 2, 8, 8, 4, 2, 0.1, [16, 40]
    lr = 2e-3
    stack = MD.build_xl_stack(vocab, d, f, blocks, T, p, 5, H, M, dtype="fp32", cutoffs=cut)
    eng = E.PipelineEngine(stack, MD.partition(stack.num_layers, K), 9)
    gopt = O.make_optimizer("adam", O.LrSchedule(lr, "fixed"))
    V, layers = X.init_xl_params(vocab, d, f, blocks, T, H, 5, cutoffs=cut)
    ora = X.XLOuroborosOracle(V, layers, K, 9, p, H, M, B, OO.Adam(lambda t: lr), cutoffs=cut)
    for k, want in layers[-1].items():
        assert rel(stack.params[-1][k].double().cpu().numpy(), want) <= 1e-7, k
    toks = (Stream(2).uniform((B * 8 * T + 4,)) * vocab).astype(np.int64)
    src = SegmentStream(toks, T, B)
    for t in range(5):
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


def test_device_batches_equal_host_batches_with_the_adaptive_head():
    """Device-resident targets reach the adaptive head's host bucketing
    through an early side-stream copy (adaptive.HostCopy), not a stream sync:
    the same losses and tied gradient as host batches, bitwise."""
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import optim as O
    from oracle.rng import Stream

    vocab, d, f, blocks, T, M, H, B, cut = 96, 64, 128, 2, 16, 16, 2, 2, [24, 56]
    toks = [((Stream(s).uniform((B, T)) * vocab).astype(np.int64), (Stream(s + 50).uniform((B, T)) * vocab).astype(np.int64))
            for s in range(4)]
    runs = []
    for device_batches in (False, True):
        stack = MD.build_xl_stack(vocab, d, f, blocks, T, 0.1, 5, H, M, dtype="bf16", cutoffs=cut)
        eng = E.ConcurrentPipelineEngine(stack, MD.partition(stack.num_layers, 2), 9)
        opt = O.make_optimizer("adam", O.LrSchedule(1e-3, "fixed"))
        losses = []
        for t, (x, y) in enumerate(toks):
            if device_batches:
                x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
            packet, loss = eng.step(t, E.BatchSample(x, y, t), opt)
            losses.append(loss)
        runs.append((losses, packet.cpu().emb_grad))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
