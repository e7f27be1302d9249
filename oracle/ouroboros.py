"""fp64 Ouroboros training step, stated from its definition (TEST INFRASTRUCTURE ONLY).

Restates the reference's model/engine/optim path:
  * parameter init order and scales      model.py:53-60, layers.py:107-112,149-166,283-284
  * contiguous partition + ring devices  model.py:85-141
  * full backprop oracle                 engine.py:409-440 (sequential_gradients)
  * the delayed-gradient schedule        engine.py:246-259
  * mixed tied gradient                  engine.py:54-69
  * SGD / Adam with a global clock       optim.py:52-126, LR schedules optim.py:16-44

Instead of replaying the executor (rings, slots, boundary hand-offs) the
schedule is written from the paper's definition, which the reference proves
its executor equals bit-for-bit (tests/test_engine.py:145-209): at step t
module k applies the full-backprop gradient of sample s = t-K+k evaluated at
the weights w^s (zero if s < 0), and the tied matrix applies
 (1/2) dV_out(sample t, w^t) + (1/2) dV_in(sample t-K+1, w^{t-K+1}).
"""

import math

import numpy as np

from . import layers as L
from .rng import Stream, hash64

# ---------------------------------------------------------------------------
# model construction


def init_params(vocab, d, f, n_blocks, seq_len, init_seed):
    """Returns (tied V, per-layer dicts) in the reference draw order."""
    rs = Stream(hash64(init_seed))
    sd, sf = 1.0 / math.sqrt(d), 1.0 / math.sqrt(f)
    V = rs.uniform_signed((vocab, d), sd)
    layers = [{"pos": rs.uniform_signed((seq_len, d), sd)}]
    for _ in range(n_blocks):
        P = {"ln1_g": np.ones(d), "ln1_b": np.zeros(d)}
        for w in ("wq", "wk", "wv", "wo"):
            P[w] = rs.uniform_signed((d, d), sd)
        P["ln2_g"], P["ln2_b"] = np.ones(d), np.zeros(d)
        P["w1"] = rs.uniform_signed((d, f), sd)
        P["b1"] = np.zeros(f)
        P["w2"] = rs.uniform_signed((f, d), sf)
        P["b2"] = np.zeros(d)
        layers.append(P)
    layers.append({})  # projection owns only the tied matrix
    return V, layers


def flat_keys(layers):
    """Gradient keys 'L{idx}.{name}' in layer order (model.py:288-292)."""
    return [f"L{i}.{n}" for i, P in enumerate(layers) for n in P]


def copy_layers(layers):
    return [{n: a.copy() for n, a in P.items()} for P in layers]


def partition_sizes(L_, K, balance="even", costs=None):
    """model.py:85-131."""
    if K < 1 or K > L_:
        raise ValueError(f"need 1 <= K <= L, got K={K}, L={L_}")
    if balance == "even":
        q, r = divmod(L_, K)
        return [q + (1 if i < r else 0) for i in range(K)]
    if balance != "by_cost" or costs is None or len(costs) != L_:
        raise ValueError("by_cost needs one cost per layer")
    pre = np.concatenate([[0.0], np.cumsum(np.asarray(costs, dtype=float))])
    INF = float("inf")
    best = np.full((K + 1, L_ + 1), INF)
    cut = np.zeros((K + 1, L_ + 1), dtype=int)
    best[0, 0] = 0.0
    for k in range(1, K + 1):
        for j in range(k, L_ - (K - k) + 1):
            for i in range(k - 1, j):
                if best[k - 1, i] == INF:
                    continue
                val = max(best[k - 1, i], pre[j] - pre[i])
                if val < best[k, j] or (val == best[k, j] and i < cut[k, j]):
                    best[k, j], cut[k, j] = val, i
    sizes, j = [], L_
    for k in range(K, 0, -1):
        i = cut[k, j]
        sizes.append(j - i)
        j = i
    return sizes[::-1]


def ring_devices(K):
    """model.py:137-140: modules 1 and K share device 0."""
    return [0] if K == 1 else [0] + list(range(1, K - 1)) + [0]


def groups_from_sizes(sizes):
    out, pos = [], 0
    for s in sizes:
        out.append((pos, pos + s))
        pos += s
    return out


# ---------------------------------------------------------------------------
# full backprop (engine.py:409-440)


def full_grads(V, layers, x, y, dropout_seed, step, p, train=True):
    """Returns (grads by key, dV_in, dV_out, loss)."""
    nl = len(layers)
    h, ce = L.embed_fwd(V, layers[0]["pos"], x, hash64(dropout_seed, step, 0), p, train)
    caches = []
    for i in range(1, nl - 1):
        h, c = L.block_fwd(layers[i], h, hash64(dropout_seed, step, i), p, train)
        caches.append(c)
    loss, g, dVo = L.head_loss_grad(h, V, y)
    G = {}
    for i in range(nl - 2, 0, -1):
        g, Gi = L.block_bwd(layers[i], caches[i - 1], g)
        for n, a in Gi.items():
            G[f"L{i}.{n}"] = a
    dVi, gpos = L.embed_bwd(g, ce, V.shape[0], layers[0]["pos"].shape)
    G["L0.pos"] = gpos
    return G, dVi, dVo, loss


def forward_loss(V, layers, x, y, dropout_seed, step, p, train=True):
    nl = len(layers)
    h, _ = L.embed_fwd(V, layers[0]["pos"], x, hash64(dropout_seed, step, 0), p, train)
    for i in range(1, nl - 1):
        h, _ = L.block_fwd(layers[i], h, hash64(dropout_seed, step, i), p, train)
    return L.head_loss(h, V, y)


# ---------------------------------------------------------------------------
# optimizers (optim.py:16-126)


def lr_at(base, mode, t, warmup=0, total=0):
    if mode == "fixed":
        return base
    if mode == "diminishing":
        return base / (1.0 + t)
    if t < warmup:
        return base * (t + 1) / warmup
    frac = (t - warmup) / (total - warmup)
    return base * 0.5 * (1.0 + math.cos(math.pi * frac))


class Sgd:
    def __init__(self, lr_fn):
        self.lr_fn = lr_fn

    def update(self, t, params, grads):
        lr = self.lr_fn(t)
        for key in params:
            params[key] -= lr * grads[key]
        return lr


class Adam:
    def __init__(self, lr_fn, b1=0.9, b2=0.999, eps=1e-8):
        self.lr_fn, self.b1, self.b2, self.eps = lr_fn, b1, b2, eps
        self.m, self.v = {}, {}

    def update(self, t, params, grads):
        lr = self.lr_fn(t)
        c1 = 1.0 - self.b1 ** (t + 1)
        c2 = 1.0 - self.b2 ** (t + 1)
        for key, w in params.items():
            g = grads[key]
            m = self.m.setdefault(key, np.zeros_like(w))
            v = self.v.setdefault(key, np.zeros_like(w))
            m *= self.b1
            m += (1.0 - self.b1) * g
            v *= self.b2
            v += (1.0 - self.b2) * (g * g)
            w -= lr * (m / c1) / (np.sqrt(v / c2) + self.eps)
        return lr


# ---------------------------------------------------------------------------
# the Ouroboros step


class OuroborosOracle:
    """Delayed-gradient training of the tied LM over K modules (fp64).

    step(t, x, y) -> (loss, packet) where packet = {"module_grads": [dict]*K,
    "emb_grad": array, "sample_ids": [int|None]*K}.  K=1 is plain backprop.
    """

    def __init__(self, V, layers, K, dropout_seed, p, optimizer=None, tied_grad="half_avg",
                 balance="even", costs=None, train=True):
        self.V, self.layers = V, layers
        self.K = K
        self.groups = groups_from_sizes(partition_sizes(len(layers), K, balance, costs))
        self.dropout_seed, self.p, self.train = dropout_seed, p, train
        self.opt = optimizer
        self.tied_grad = tied_grad
        self.pending = {}  # sample step -> (grads, dVi) at w^s

    def _owner(self, key):
        idx = int(key.split(".")[0][1:])
        for k, (a, b) in enumerate(self.groups):
            if a <= idx < b:
                return k
        raise KeyError(key)

    def step(self, t, x, y):
        K = self.K
        G, dVi, dVo, loss = self._full_grads(t, x, y)
        self.pending[t] = (G, dVi)
        module_grads, sample_ids = [], []
        for k in range(1, K + 1):
            s = t - K + k
            lo, hi = self.groups[k - 1]
            keys = [f"L{i}.{n}" for i in range(lo, hi) for n in self.layers[i]]
            if s < 0:
                module_grads.append({key: np.zeros_like(self._param(key)) for key in keys})
                sample_ids.append(None)
            else:
                Gs = self.pending[s][0]
                module_grads.append({key: Gs[key] for key in keys})
                sample_ids.append(s)
        s_in = t - K + 1
        if s_in < 0:
            emb = np.zeros_like(self.V)
        else:
            vi = self.pending[s_in][1]
            emb = 0.5 * dVo + 0.5 * vi if self.tied_grad == "half_avg" else dVo + vi
        for s in [s for s in self.pending if s <= t - K + 1]:
            del self.pending[s]
        packet = {"module_grads": module_grads, "emb_grad": emb, "sample_ids": sample_ids}
        if self.opt is not None:
            params = {"tied": self.V}
            grads = {"tied": emb}
            for mg in module_grads:
                for key, g in mg.items():
                    params[key] = self._param(key)
                    grads[key] = g
            self.opt.update(t, params, grads)
        return loss, packet

    def _full_grads(self, t, x, y):
        """K=1 backprop of sample t at the current weights w^t."""
        return full_grads(self.V, self.layers, x, y, self.dropout_seed, t, self.p, self.train)

    def _param(self, key):
        idx, name = key.split(".", 1)
        return self.layers[int(idx[1:])][name]
