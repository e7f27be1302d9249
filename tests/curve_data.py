"""Learnable synthetic token stream for the C1 loss-curve parity test
(tests/golden/make_curve_golden.py, tests/test_curve_gpu.py).

A seeded first-order Markov chain over the C1 vocabulary: every token has 4
preferred successors (80% of the mass) over a Zipf background, so the loss
falls well below ln(V) as the model learns.  Batches are a pure function of
t (numpy PCG64 with a fixed seed, identical on every machine)."""

import numpy as np

C1 = dict(vocab=1000, d=128, f=512, blocks=4, seq=64, batch=16, p=0.1, init_seed=11, dseed=7, K=2, lr=1e-3)
STEPS = 500

_rng = np.random.Generator(np.random.PCG64(20251018))
_V = C1["vocab"]
_SUCC = _rng.integers(0, _V, size=(_V, 4))
_ZIPF = 1.0 / np.arange(1, _V + 1)
_ZIPF /= _ZIPF.sum()


def batch_at(t):
    g = np.random.Generator(np.random.PCG64([20251018, t]))
    B, T = C1["batch"], C1["seq"]
    seq = np.empty((B, T + 1), dtype=np.int64)
    seq[:, 0] = g.choice(_V, size=B, p=_ZIPF)
    for i in range(1, T + 1):
        follow = g.random(B) < 0.8
        pick = _SUCC[seq[:, i - 1], g.integers(0, 4, size=B)]
        seq[:, i] = np.where(follow, pick, g.choice(_V, size=B, p=_ZIPF))
    return seq[:, :-1].copy(), seq[:, 1:].copy()
