"""fp64 adaptive tied softmax head (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED AT THE REFERENCE: the reference has no adaptive softmax
(SURVEY.md 8(f) row 2 lists it for BASELINE
configs[3]).  This restates the published adaptive softmax (Grave et al.
2017, arXiv 1609.04309) in the form Transformer-XL trains WikiText-103 with
(ProjectedAdaptiveLogSoftmax, div_val = 1, tied output layers): vocabulary
cutoffs c_0 < c_1 < ... < c_{n-1} < V split the ids into a head [0, c_0) and
n tail clusters [c_k, c_{k+1}) (c_n = V).  The head scores the c_0 head ids against the tied
matrix rows and one "cluster" class per tail (own weight w_k and bias b_k):

    head logits   z = h V[:c_0]^T  ||  h W_c^T + b_c            [N, c_0 + n]
    tail k logits t = h V[c_k : c_{k+1}]^T                      (rows whose id is in cluster k)
    -log p(y) = -log softmax(z)[y]                               (y < c_0)
              = -log softmax(z)[c_0 + k] - log softmax(t)[y - c_k]   (y in cluster k)

The loss is the mean over the N rows.  Pinned by: a single cluster-free head
(n = 0) reduces to the reference tied head (oracle/layers.head_loss_grad,
itself pinned to the live reference), probabilities over the whole vocabulary
sum to 1, and central finite differences of every input.
"""

import numpy as np


def clusters(cutoffs, vocab):
    """Tail clusters [(c_k, c_{k+1})] for cutoffs [c_0, ..., c_{n-1}] and the
    vocabulary size: ids >= c_0 fall in n tails (the head holds [0, c_0))."""
    edges = list(cutoffs) + [vocab]
    return [(edges[k], edges[k + 1]) for k in range(len(cutoffs)) if edges[k] < edges[k + 1]]


def _log_softmax(z):
    m = z.max(axis=-1, keepdims=True)
    e = np.exp(z - m)
    s = e.sum(axis=-1, keepdims=True)
    return z - m - np.log(s), e / s


def adaptive_loss_grad(h, V, Wc, bc, y, cutoffs):
    """h [N, d], V [vocab, d] (tied), Wc [n, d], bc [n], y [N] ids.
    Returns (loss, g_h, g_V, g_Wc, g_bc)."""
    h = np.asarray(h, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    N = h.shape[0]
    c0 = cutoffs[0]
    tails = clusters(cutoffs, V.shape[0])
    n = len(tails)
    assert Wc.shape[0] == n and bc.shape[0] == n
    z = np.concatenate([h @ V[:c0].T, h @ Wc.T + bc[None, :]], axis=1)
    lp, p = _log_softmax(z)
    yh = y.copy()
    for k, (lo, hi) in enumerate(tails):
        yh[(y >= lo) & (y < hi)] = c0 + k
    loss = -lp[np.arange(N), yh].sum()
    dz = p.copy()
    dz[np.arange(N), yh] -= 1.0
    dz /= N
    g_h = dz[:, :c0] @ V[:c0] + dz[:, c0:] @ Wc
    g_V = np.zeros_like(V)
    g_V[:c0] = dz[:, :c0].T @ h
    g_Wc = dz[:, c0:].T @ h
    g_bc = dz[:, c0:].sum(axis=0)
    for k, (lo, hi) in enumerate(tails):
        rows = np.nonzero((y >= lo) & (y < hi))[0]
        if rows.size == 0:
            continue
        t = h[rows] @ V[lo:hi].T
        lpt, pt = _log_softmax(t)
        loss -= lpt[np.arange(rows.size), y[rows] - lo].sum()
        dt = pt.copy()
        dt[np.arange(rows.size), y[rows] - lo] -= 1.0
        dt /= N
        g_h[rows] += dt @ V[lo:hi]
        g_V[lo:hi] += dt.T @ h[rows]
    return loss / N, g_h, g_V, g_Wc, g_bc


def adaptive_logprob(h, V, Wc, bc, cutoffs):
    """log p(id) for every id of the vocabulary, [N, vocab] (small cases)."""
    h = np.asarray(h, dtype=np.float64)
    c0 = cutoffs[0]
    z = np.concatenate([h @ V[:c0].T, h @ Wc.T + bc[None, :]], axis=1)
    lp, _ = _log_softmax(z)
    out = np.empty((h.shape[0], V.shape[0]))
    out[:, :c0] = lp[:, :c0]
    for k, (lo, hi) in enumerate(clusters(cutoffs, V.shape[0])):
        lpt, _ = _log_softmax(h @ V[lo:hi].T)
        out[:, lo:hi] = lp[:, c0 + k][:, None] + lpt
    return out
