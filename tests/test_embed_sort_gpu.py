"""Embedding backward scatter (csrc/embed_head.cu) at token counts that span
several 1024-key sort chunks (ragged last chunk, Zipf-duplicated tokens):
the tied-gradient rows must equal, bitwise, an fp32 restatement of the
kernel's fixed summation order -- positions sorted by (token, position),
runs summed inside 32-position chunks, chunk partials summed in chunk order
(layers.py:130-136 scatter-add, made deterministic)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _expected(g, tok, vocab, beta):
    n, d = g.shape
    order = np.lexsort((np.arange(n), tok))
    st, sg = tok[order], g[order]
    emb = np.zeros((vocab, d), np.float32)
    partial = {}
    for c0 in range(0, n, 32):
        start, acc = c0, np.zeros(d, np.float32)
        for q in range(c0, min(c0 + 32, n)):
            acc = (acc + sg[q]).astype(np.float32)
            if q + 1 == min(c0 + 32, n) or st[q + 1] != st[q]:
                partial[start] = acc
                start, acc = q + 1, np.zeros(d, np.float32)
    i = 0
    while i < n:
        e = i + 1
        while e < n and st[e] == st[i]:
            e += 1
        total = partial[i].copy()
        for c in range((i // 32 + 1) * 32, e, 32):
            total = (total + partial[c]).astype(np.float32)
        emb[st[i]] = (emb[st[i]] + np.float32(beta) * total).astype(np.float32)
        i = e
    return emb


@pytest.mark.parametrize("B,T", [(1, 1), (3, 7), (2, 1024), (9, 1000), (16, 512)])
def test_embed_bwd_multi_chunk_sort(B, T):
    from paper_1909_06695_b200 import layers as Ly

    vocab, d = 300, 40
    rng = np.random.default_rng(B * 1000 + T)
    tok = np.minimum(rng.zipf(1.3, size=(B, T)) - 1, vocab - 1).astype(np.int64)
    g = rng.standard_normal((B * T, d)).astype(np.float32)
    dev = "cuda"
    tokens = torch.from_numpy(tok).to(dev)
    gd = torch.from_numpy(g).to(dev)
    outs = []
    for _ in range(2):
        emb = torch.zeros(vocab, d, device=dev)
        gpos = torch.empty(T, d, device=dev)
        Ly.embed_backward(gd, tokens, T, gpos, emb, 1.0, _Ws(), None)
        torch.cuda.synchronize()
        outs.append(emb.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])  # run-to-run deterministic
    assert np.array_equal(outs[0], _expected(g, tok.reshape(-1), vocab, 1.0))


class _Ws:
    def __init__(self):
        self.bufs = {}

    def get(self, name, shape, dtype):
        if name not in self.bufs:
            self.bufs[name] = torch.empty(shape, dtype=dtype, device="cuda")
        return self.bufs[name]
