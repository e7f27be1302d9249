"""fp64 adaptive tied softmax restatement (oracle/adaptive.py; parity unpinned
at the reference, which has no adaptive softmax): reduction to the reference
tied head with no tail cluster, normalisation over the whole vocabulary, and
central finite differences of every input."""

import numpy as np

from oracle import adaptive as A
from oracle import layers as L


def _case(seed=0, N=12, d=8, vocab=40, cutoffs=(10, 25)):
    r = np.random.default_rng(seed)
    h = r.normal(size=(N, d))
    V = r.normal(size=(vocab, d)) * 0.5
    n = len(cutoffs)
    Wc = r.normal(size=(n, d)) * 0.5
    bc = r.normal(size=n) * 0.3
    y = r.integers(0, vocab, size=N)
    y[:3] = [0, cutoffs[0], vocab - 1]  # head, first tail, last tail
    return h, V, Wc, bc, y, list(cutoffs)


def test_no_tail_reduces_to_reference_head():
    h, V, _, _, y, _ = _case()
    loss, g_h, g_V, _, _ = A.adaptive_loss_grad(h, V, np.zeros((0, 8)), np.zeros(0), y, [V.shape[0]])
    rl, rgh, rgV = L.head_loss_grad(h, V, y)
    assert abs(loss - rl) <= 1e-12 * abs(rl)
    assert np.allclose(g_h, rgh, rtol=1e-12, atol=1e-14)
    assert np.allclose(g_V, rgV, rtol=1e-12, atol=1e-14)


def test_probabilities_sum_to_one_and_match_the_loss():
    h, V, Wc, bc, y, cut = _case(1)
    lp = A.adaptive_logprob(h, V, Wc, bc, cut)
    assert np.allclose(np.exp(lp).sum(axis=1), 1.0, atol=1e-12)
    loss = A.adaptive_loss_grad(h, V, Wc, bc, y, cut)[0]
    assert abs(loss + lp[np.arange(len(y)), y].mean()) <= 1e-12


def test_finite_differences_every_input():
    h, V, Wc, bc, y, cut = _case(2, N=6, d=5, vocab=17, cutoffs=(5, 11))
    loss, g_h, g_V, g_Wc, g_bc = A.adaptive_loss_grad(h, V, Wc, bc, y, cut)
    args = {"h": h, "V": V, "Wc": Wc, "bc": bc}
    grads = {"h": g_h, "V": g_V, "Wc": g_Wc, "bc": g_bc}
    eps = 1e-6
    for name, arr in args.items():
        for idx in np.ndindex(arr.shape):
            old = arr[idx]
            arr[idx] = old + eps
            lp = A.adaptive_loss_grad(h, V, Wc, bc, y, cut)[0]
            arr[idx] = old - eps
            lm = A.adaptive_loss_grad(h, V, Wc, bc, y, cut)[0]
            arr[idx] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - grads[name][idx]) <= 1e-7 + 1e-6 * abs(fd), (name, idx, fd, grads[name][idx])
