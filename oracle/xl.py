"""fp64 Transformer-XL block and model step (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED AT THE REFERENCE: the reference has no Transformer-XL path
(SPEC.md:13, SPEC.md:152 exclude it).  This file
restates the published Transformer-XL attention (Dai et al. 2019, arXiv
1901.02860, sec. 3.3: relative positional encodings with the global content
bias u and position bias v, and a segment-level recurrence whose memory is
the previous segment's layer input with gradients stopped) inside the
reference's pre-LN block (layers.py:168-253: same LayerNorm, dropout
positions, ReLU FFN and residuals).  It is pinned two ways instead:
  * with one head, no valid memory and u = v = wr = 0 it reduces to the
    reference block, which tests compare against oracle/layers.py (itself
    pinned to the live reference by tests/golden/);
  * central finite differences of the fp64 loss for every parameter,
    including u, v and wr, with memory present.

Shapes: x [B, T, d] the segment's layer input, mem [B, M, d] the previous
segment's layer input, of which the last `mem_len` rows are valid.  Keys run
over the concatenation [mem; x] (Kl = M + T rows).  Query i (position M + i)
sees key j iff M - mem_len <= j <= M + i.  The relative distance of (i, j) is
M + i - j; the sinusoid table R has row p for distance Kl - 1 - p (XL's
descending pos_seq), so the position term of (i, j) is row p = T - 1 - i + j
of (q_i + v) . (R wr)^T -- the "relative shift".
"""

import math

import numpy as np

from . import adaptive as A
from . import layers as L
from .ouroboros import OuroborosOracle
from .rng import Stream, hash64

XL_KEYS = ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "wr", "r_w_bias", "r_r_bias", "ln2_g", "ln2_b", "w1", "b1",
           "w2", "b2")


def sinusoid(Kl, d):
    """R [Kl, d]: row p encodes distance Kl-1-p as [sin(k w), cos(k w)]
    with w_c = 10000^(-2c/d) (XL's PositionalEmbedding)."""
    dist = np.arange(Kl - 1, -1, -1, dtype=np.float64)
    inv = 1.0 / (10000.0 ** (np.arange(0, d, 2, dtype=np.float64) / d))
    ang = dist[:, None] * inv[None, :]
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=1)


def _heads(x, H):
    B, n, d = x.shape
    return x.reshape(B, n, H, d // H).transpose(0, 2, 1, 3)  # [B, H, n, dh]


def _merge(x):
    B, H, n, dh = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B, n, H * dh)


def key_mask(T, M, mem_len):
    """[T, Kl] True where query i may attend key j."""
    i = np.arange(T)[:, None]
    j = np.arange(M + T)[None, :]
    return (j <= M + i) & (j >= M - mem_len)


def rel_shift(bdf, T):
    """bd[..., i, j] = bdf[..., i, T-1-i+j] (0 where that column is past the end)."""
    Kl = bdf.shape[-1]
    out = np.zeros(bdf.shape[:-2] + (T, Kl))
    for i in range(T):
        lo = T - 1 - i
        n = Kl - lo
        out[..., i, :n] = bdf[..., i, lo:]
    return out


def rel_shift_back(gbd, T):
    """Adjoint of rel_shift."""
    Kl = gbd.shape[-1]
    out = np.zeros(gbd.shape[:-2] + (T, Kl))
    for i in range(T):
        lo = T - 1 - i
        n = Kl - lo
        out[..., i, lo:] = gbd[..., i, :n]
    return out


def xl_block_fwd(P, x, mem, mem_len, H, seed, p, train, act="relu"):
    B, T, d = x.shape
    M = mem.shape[1]
    dh = d // H
    n = B * T * d
    xa = np.concatenate([mem, x], axis=1)
    a, c1 = L.ln_fwd(xa, P["ln1_g"], P["ln1_b"])
    q = a[:, M:] @ P["wq"]
    k = a @ P["wk"]
    v = a @ P["wv"]
    qh, kh, vh = _heads(q, H), _heads(k, H), _heads(v, H)
    R = sinusoid(M + T, d)
    r = R @ P["wr"]
    rh = r.reshape(M + T, H, dh).transpose(1, 0, 2)  # [H, Kl, dh]
    qu = qh + P["r_w_bias"][None, :, None, :]
    qv = qh + P["r_r_bias"][None, :, None, :]
    ac = qu @ kh.transpose(0, 1, 3, 2)
    bdf = np.einsum("bhid,hpd->bhip", qv, rh)
    s = (ac + rel_shift(bdf, T)) / math.sqrt(dh)
    s = np.where(key_mask(T, M, mem_len), s, -np.inf)
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    probs = e / e.sum(axis=-1, keepdims=True)
    ctx = _merge(probs @ vh)
    proj = ctx @ P["wo"]
    m0 = L.dropout_scale_mask(seed, 0, (B, T, d), p) if train else None
    if m0 is not None:
        proj = proj * m0
    x1 = x + proj
    m, c2 = L.ln_fwd(x1, P["ln2_g"], P["ln2_b"])
    z1 = m @ P["w1"] + P["b1"]
    h1 = L.gelu(z1) if act == "gelu" else np.maximum(z1, 0.0)
    h2 = h1 @ P["w2"] + P["b2"]
    m1 = L.dropout_scale_mask(seed, n, (B, T, d), p) if train else None
    if m1 is not None:
        h2 = h2 * m1
    out = x1 + h2
    cache = dict(M=M, H=H, R=R, a=a, qu=qu, qv=qv, kh=kh, vh=vh, rh=rh, probs=probs, ctx=ctx, m=m, z1=z1, h1=h1,
                 c1=c1, c2=c2, m0=m0, m1=m1, act=act)
    return out, cache


def xl_block_bwd(P, c, gout):
    """Returns (grad wrt x, grads by name); no gradient flows into mem."""
    B, T, d = gout.shape
    M, H = c["M"], c["H"]
    dh = d // H
    G = {}
    gh2 = gout * c["m1"] if c["m1"] is not None else gout
    G["w2"] = np.einsum("btf,btd->fd", c["h1"], gh2)
    G["b2"] = gh2.sum(axis=(0, 1))
    gz1 = (gh2 @ P["w2"].T) * (L.gelu_grad(c["z1"]) if c.get("act") == "gelu" else (c["z1"] > 0.0))
    G["w1"] = np.einsum("btd,btf->df", c["m"], gz1)
    G["b1"] = gz1.sum(axis=(0, 1))
    gm = gz1 @ P["w1"].T
    gx1, G["ln2_g"], G["ln2_b"] = L.ln_bwd(gm, P["ln2_g"], c["c2"])
    gx1 = gx1 + gout
    gproj = gx1 * c["m0"] if c["m0"] is not None else gx1
    G["wo"] = np.einsum("btd,bte->de", c["ctx"], gproj)
    gctx = _heads(gproj @ P["wo"].T, H)
    pr = c["probs"]
    gp = gctx @ c["vh"].transpose(0, 1, 3, 2)
    gvh = pr.transpose(0, 1, 3, 2) @ gctx
    gs = (gp - (gp * pr).sum(axis=-1, keepdims=True)) * pr / math.sqrt(dh)
    gbdf = rel_shift_back(gs, T)
    gqu = gs @ c["kh"]
    gkh = gs.transpose(0, 1, 3, 2) @ c["qu"]
    gqv = np.einsum("bhip,hpd->bhid", gbdf, c["rh"])
    grh = np.einsum("bhip,bhid->hpd", gbdf, c["qv"])
    G["r_w_bias"] = gqu.sum(axis=(0, 2))
    G["r_r_bias"] = gqv.sum(axis=(0, 2))
    gq = _merge(gqu + gqv)
    gr = grh.transpose(1, 0, 2).reshape(M + T, d)
    G["wr"] = c["R"].T @ gr
    a = c["a"]
    gk, gv = _merge(gkh), _merge(gvh)
    G["wq"] = np.einsum("btd,bte->de", a[:, M:], gq)
    G["wk"] = np.einsum("btd,bte->de", a, gk)
    G["wv"] = np.einsum("btd,bte->de", a, gv)
    ga = gk @ P["wk"].T + gv @ P["wv"].T
    ga[:, M:] += gq @ P["wq"].T
    gxa, G["ln1_g"], G["ln1_b"] = L.ln_bwd(ga, P["ln1_g"], c["c1"])
    return gxa[:, M:] + gx1, G


# ---------------------------------------------------------------------------
# the XL language model: reference embedding + XL blocks + tied head


def init_xl_params(vocab, d, f, n_blocks, seq_len, H, init_seed, cutoffs=None):
    """Draw order: V, the embedding's position table, then per block wq, wk,
    wv, wo, wr (+-1/sqrt d), r_w_bias, r_r_bias (+-1/sqrt d), w1 (+-1/sqrt d),
    w2 (+-1/sqrt f); LayerNorm gains 1, biases 0.  With adaptive-softmax
    cutoffs the projection layer last draws its cluster weights (+-1/sqrt d);
    cluster biases 0."""
    rs = Stream(hash64(init_seed))
    sd, sf = 1.0 / math.sqrt(d), 1.0 / math.sqrt(f)
    V = rs.uniform_signed((vocab, d), sd)
    layers = [{"pos": rs.uniform_signed((seq_len, d), sd)}]
    for _ in range(n_blocks):
        P = {"ln1_g": np.ones(d), "ln1_b": np.zeros(d)}
        for w in ("wq", "wk", "wv", "wo", "wr"):
            P[w] = rs.uniform_signed((d, d), sd)
        P["r_w_bias"] = rs.uniform_signed((H, d // H), sd)
        P["r_r_bias"] = rs.uniform_signed((H, d // H), sd)
        P["ln2_g"], P["ln2_b"] = np.ones(d), np.zeros(d)
        P["w1"] = rs.uniform_signed((d, f), sd)
        P["b1"] = np.zeros(f)
        P["w2"] = rs.uniform_signed((f, d), sf)
        P["b2"] = np.zeros(d)
        layers.append(P)
    proj = {}
    if cutoffs:
        n = len(A.clusters(cutoffs, vocab))
        proj = {"cluster_weight": rs.uniform_signed((n, d), sd), "cluster_bias": np.zeros(n)}
    layers.append(proj)
    return V, layers


def _head(h, V, y, P, cutoffs):
    """(loss, g_h, dVo, projection grads): the tied head, or the adaptive
    tied softmax (oracle/adaptive.py) when the projection has cluster params."""
    if not cutoffs:
        loss, g, dVo = L.head_loss_grad(h, V, y)
        return loss, g, dVo, {}
    d = h.shape[-1]
    loss, g, dVo, gW, gb = A.adaptive_loss_grad(h.reshape(-1, d), V, P["cluster_weight"], P["cluster_bias"],
                                                np.asarray(y).reshape(-1), cutoffs)
    return loss, g.reshape(h.shape), dVo, {"cluster_weight": gW, "cluster_bias": gb}


def xl_full_grads(V, layers, x, y, dropout_seed, step, p, mems, mem_len, H, train=True, cutoffs=None):
    """K=1 backprop of one segment.  mems: per block [B, M, d] (layer inputs
    of the previous segment).  Returns (grads, dVi, dVo, loss, new_mems)."""
    nl = len(layers)
    h, ce = L.embed_fwd(V, layers[0]["pos"], x, hash64(dropout_seed, step, 0), p, train)
    caches, new_mems = [], []
    for i in range(1, nl - 1):
        M = mems[i - 1].shape[1]
        new_mems.append(h[:, h.shape[1] - M:].copy())
        h, c = xl_block_fwd(layers[i], h, mems[i - 1], mem_len, H, hash64(dropout_seed, step, i), p, train)
        caches.append(c)
    loss, g, dVo, Gp = _head(h, V, y, layers[-1], cutoffs)
    G = {f"L{nl - 1}.{n}": a for n, a in Gp.items()}
    for i in range(nl - 2, 0, -1):
        g, Gi = xl_block_bwd(layers[i], caches[i - 1], g)
        for n, a in Gi.items():
            G[f"L{i}.{n}"] = a
    dVi, gpos = L.embed_bwd(g, ce, V.shape[0], layers[0]["pos"].shape)
    G["L0.pos"] = gpos
    return G, dVi, dVo, loss, new_mems


def xl_forward_loss(V, layers, x, y, dropout_seed, step, p, mems, mem_len, H, train=True):
    nl = len(layers)
    h, _ = L.embed_fwd(V, layers[0]["pos"], x, hash64(dropout_seed, step, 0), p, train)
    for i in range(1, nl - 1):
        h, _ = xl_block_fwd(layers[i], h, mems[i - 1], mem_len, H, hash64(dropout_seed, step, i), p, train)
    return L.head_loss(h, V, y)


class XLOuroborosOracle(OuroborosOracle):
    """The Ouroboros schedule over the XL model (fp64).  Memory is data, not a
    parameter: the forward of segment t runs at the live weights w^t in both
    the pipeline and plain backprop, so module k's stale gradient of sample s
    is the K=1 gradient of segment s given the memory segment s-1 left --
    exactly what `xl_full_grads` computes at step s."""

    def __init__(self, V, layers, K, dropout_seed, p, H, mem_len, batch, optimizer=None, cutoffs=None, **kw):
        super().__init__(V, layers, K, dropout_seed, p, optimizer, **kw)
        self.H, self.M = H, mem_len
        self.cutoffs = cutoffs
        d = V.shape[1]
        self.mems = [np.zeros((batch, mem_len, d)) for _ in range(len(layers) - 2)]
        self.mem_valid = 0

    def _full_grads(self, t, x, y):
        G, dVi, dVo, loss, self.mems = xl_full_grads(self.V, self.layers, x, y, self.dropout_seed, t, self.p,
                                                     self.mems, self.mem_valid, self.H, self.train, self.cutoffs)
        self.mem_valid = self.M
        return G, dVi, dVo, loss
