"""fp64 forward/backward of the three layer kinds (TEST INFRASTRUCTURE ONLY).

Restates reference layers.py: embedding (layers.py:114-136), pre-LN
single-head transformer block (layers.py:168-253), tied projection with the
fused softmax cross-entropy head (layers.py:268-322) and LayerNorm
(layers.py:62-79).  Contractions use numpy's BLAS matmul instead of the
reference's fixed-order loops (kernels.py:23-48); results agree to ~1e-13
relative, which the golden-fixture tests pin.

Each *_fwd returns (out, cache); each *_bwd consumes the cache.  Dropout
masks come from the splitmix64 stream at (seed, position) exactly as the
reference draws them: embedding positions [0, n); block mask0 [0, n) and
mask1 [n, 2n) with n = B*T*d (layers.py:184-195, 209-212).
"""

import math

import numpy as np
from scipy.special import erf as _erf

from .rng import dropout_scale_mask

EPS = 1e-5  # layers.py:25


class ShapeError(ValueError):
    pass


def ln_fwd(x, g, b):
    """layers.py:62-67 (biased variance, eps 1e-5)."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    rstd = 1.0 / np.sqrt((xc * xc).mean(axis=-1, keepdims=True) + EPS)
    xhat = xc * rstd
    return xhat * g + b, (xhat, rstd)


def ln_bwd(gy, g, cache):
    """layers.py:70-79."""
    xhat, rstd = cache
    red = tuple(range(gy.ndim - 1))
    dg = (gy * xhat).sum(axis=red)
    db = gy.sum(axis=red)
    gx = gy * g
    dx = rstd * (gx - gx.mean(axis=-1, keepdims=True) - xhat * (gx * xhat).mean(axis=-1, keepdims=True))
    return dx, dg, db


def _rows(x):
    return x.reshape(-1, x.shape[-1])


# ---------------------------------------------------------------------------
# embedding: layers.py:114-136


def embed_fwd(V, pos, tokens, seed, p, train, pos0=0):
    """pos0: first dropout position (a row block of a larger batch starts at
    its first row * d; the whole batch draws [0, N*d), layers.py:124)."""
    tokens = np.asarray(tokens)
    if tokens.size and tokens.max() >= V.shape[0]:
        raise ShapeError("token id out of vocabulary range")
    T = tokens.shape[-1]
    h = V[tokens] + pos[:T]
    mask = dropout_scale_mask(seed, pos0, h.shape, p) if train else None
    if mask is not None:
        h = h * mask
    return h, (tokens, mask)


def embed_bwd(g, cache, vocab, pos_shape):
    tokens, mask = cache
    if mask is not None:
        g = g * mask
    T = tokens.shape[-1]
    gpos = np.zeros(pos_shape)
    gpos[:T] = g.sum(axis=0)
    gV = np.zeros((vocab, g.shape[-1]))
    np.add.at(gV, tokens.reshape(-1), _rows(g))
    return gV, gpos


# ---------------------------------------------------------------------------
# transformer block: layers.py:168-253

BLOCK_KEYS = ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2")


def gelu(z):
    """Exact GELU 0.5 z (1 + erf(z / sqrt 2)) -- the FFN activation option
    of the device path (the reference FFN is ReLU, layers.py:191)."""
    return 0.5 * z * (1.0 + _erf(z / math.sqrt(2.0)))


def gelu_grad(z):
    return 0.5 * (1.0 + _erf(z / math.sqrt(2.0))) + z * np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)


def block_fwd(P, x, seed, p, train, pos0=0, n_total=None, act="relu"):
    """pos0 / n_total: a row block of a larger batch -- mask0 draws
    [pos0, pos0 + n), mask1 [n_total + pos0, ...) with n_total = N*d of the
    whole batch (layers.py:184-195).  act: "relu" (the reference) or "gelu"."""
    B, T, d = x.shape
    n = B * T * d
    n1 = n if n_total is None else n_total
    a, c1 = ln_fwd(x, P["ln1_g"], P["ln1_b"])
    ar = _rows(a)
    q = (ar @ P["wq"]).reshape(B, T, d)
    k = (ar @ P["wk"]).reshape(B, T, d)
    v = (ar @ P["wv"]).reshape(B, T, d)
    s = np.einsum("btd,bsd->bts", q, k) / math.sqrt(d)
    causal = np.tril(np.ones((T, T), dtype=bool))
    s = np.where(causal, s, -np.inf)
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    probs = e / e.sum(axis=-1, keepdims=True)
    ctx = probs @ v
    proj = (_rows(ctx) @ P["wo"]).reshape(B, T, d)
    m0 = dropout_scale_mask(seed, pos0, (B, T, d), p) if train else None
    if m0 is not None:
        proj = proj * m0
    x1 = x + proj
    m, c2 = ln_fwd(x1, P["ln2_g"], P["ln2_b"])
    z1 = _rows(m) @ P["w1"] + P["b1"]
    h1 = gelu(z1) if act == "gelu" else np.maximum(z1, 0.0)
    h2 = (h1 @ P["w2"] + P["b2"]).reshape(B, T, d)
    m1 = dropout_scale_mask(seed, n1 + pos0, (B, T, d), p) if train else None
    if m1 is not None:
        h2 = h2 * m1
    out = x1 + h2
    cache = dict(x=x, a=a, q=q, k=k, v=v, probs=probs, ctx=ctx, m=m, z1=z1, h1=h1, c1=c1, c2=c2, m0=m0, m1=m1,
                 act=act)
    return out, cache


def block_bwd(P, c, gout):
    B, T, d = gout.shape
    G = {}
    gh2 = gout * c["m1"] if c["m1"] is not None else gout
    gh2r = _rows(gh2)
    G["w2"] = c["h1"].T @ gh2r
    G["b2"] = gh2r.sum(axis=0)
    gz1 = (gh2r @ P["w2"].T) * (gelu_grad(c["z1"]) if c.get("act") == "gelu" else (c["z1"] > 0.0))
    G["w1"] = _rows(c["m"]).T @ gz1
    G["b1"] = gz1.sum(axis=0)
    gm = (gz1 @ P["w1"].T).reshape(B, T, d)
    gx1, G["ln2_g"], G["ln2_b"] = ln_bwd(gm, P["ln2_g"], c["c2"])
    gx1 = gx1 + gout
    gproj = gx1 * c["m0"] if c["m0"] is not None else gx1
    gpr = _rows(gproj)
    G["wo"] = _rows(c["ctx"]).T @ gpr
    gctx = (gpr @ P["wo"].T).reshape(B, T, d)
    pr = c["probs"]
    gprobs = gctx @ c["v"].transpose(0, 2, 1)
    gv = pr.transpose(0, 2, 1) @ gctx
    gs = (gprobs - (gprobs * pr).sum(axis=-1, keepdims=True)) * pr / math.sqrt(d)
    gq = gs @ c["k"]
    gk = gs.transpose(0, 2, 1) @ c["q"]
    ar = _rows(c["a"])
    G["wq"] = ar.T @ _rows(gq)
    G["wk"] = ar.T @ _rows(gk)
    G["wv"] = ar.T @ _rows(gv)
    ga = _rows(gq) @ P["wq"].T + _rows(gk) @ P["wk"].T + _rows(gv) @ P["wv"].T
    gx, G["ln1_g"], G["ln1_b"] = ln_bwd(ga.reshape(B, T, d), P["ln1_g"], c["c1"])
    return gx + gx1, G


# ---------------------------------------------------------------------------
# tied head: layers.py:287-322


def check_targets(y, vocab):
    y = np.asarray(y)
    if y.size and (y.max() >= vocab or y.min() < 0):
        raise ShapeError("target id out of range")
    return y


def head_loss_grad(h, V, y):
    """(loss, grad_h, grad_V_output_side) of mean CE over h @ V^T."""
    y = check_targets(y, V.shape[0]).reshape(-1)
    hr = _rows(h)
    z = hr @ V.T
    zmax = z.max(axis=1, keepdims=True)
    ez = np.exp(z - zmax)
    se = ez.sum(axis=1, keepdims=True)
    lse = zmax[:, 0] + np.log(se[:, 0])
    idx = np.arange(y.size)
    loss = float(np.mean(lse - z[idx, y]))
    dz = ez / se
    dz[idx, y] -= 1.0
    dz /= y.size
    return loss, (dz @ V).reshape(h.shape), dz.T @ hr


def head_loss(h, V, y):
    y = check_targets(y, V.shape[0]).reshape(-1)
    z = _rows(h) @ V.T
    zmax = z.max(axis=1)
    lse = zmax + np.log(np.exp(z - zmax[:, None]).sum(axis=1))
    return float(np.mean(lse - z[np.arange(y.size), y]))
