"""Pins the CPU oracle (oracle/) to the reference before it is trusted.

Golden values come from the reference's own tests (tests/test_tensor.py:148-156,
tests/test_model.py:19-61, tests/test_layers.py:278-293) and from fixtures
made by running the live reference (tests/golden/make_golden.py)."""

import math
import os

import numpy as np
import pytest

from oracle import layers as OL
from oracle import ouroboros as OO
from oracle.rng import Stream, hash64, uniform

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CONFIGS = {
    "tiny": (7, 8, 8, 3, 4, 2, 0.2, 11, 7, 1),
    "small": (64, 32, 64, 2, 16, 4, 0.1, 5, 9, 3),
}


def load(name):
    return np.load(os.path.join(GOLD, name))


def test_rng_known_values():
    # reference tests/test_tensor.py:148-156
    expected = np.array([0.5665615751722809, 0.7457817572627011, 0.9710027535867962])
    assert np.array_equal(uniform(1, 0, (3,)), expected)
    assert np.array_equal(uniform(1, 1, (2,)), expected[1:])
    g = load("reference_basics.npz")
    assert np.array_equal(g["rng_mid"], uniform(12345, 1000, (5,)))


def test_rng_stream_contiguous():
    s = Stream(5)
    a = np.concatenate([s.uniform((10,)), s.uniform((10,))])
    assert np.array_equal(a, Stream(5).uniform((20,)))


def test_partition_goldens():
    g = load("reference_basics.npz")
    for L_, K in [(12, 4), (5, 3), (8, 2), (8, 5), (14, 9), (6, 2), (12, 1)]:
        groups = OO.groups_from_sizes(OO.partition_sizes(L_, K))
        assert np.array_equal(np.array(groups), g[f"part.{L_}.{K}.groups"])
        assert OO.ring_devices(K) == list(g[f"part.{L_}.{K}.dev"])
    assert np.array_equal(
        np.array(OO.groups_from_sizes(OO.partition_sizes(4, 2, "by_cost", [10.0, 1, 1, 1]))),
        g["part.bycost.groups"],
    )
    costs = [3.0, 1.0, 4.0, 1.0, 5.0, 9.0, 2.0, 6.0]
    assert np.array_equal(
        np.array(OO.groups_from_sizes(OO.partition_sizes(8, 3, "by_cost", costs))), g["part.bycost2.groups"]
    )


@pytest.mark.parametrize("cfg", list(CONFIGS))
def test_init_matches_reference(cfg):
    vocab, d, f, nb, seq, _, _, seed, _, _ = CONFIGS[cfg]
    V, layers = OO.init_params(vocab, d, f, nb, seq, seed)
    g = load("reference_basics.npz")
    assert np.array_equal(V, g[f"init.{cfg}.tied"])
    for i, P in enumerate(layers):
        for n, a in P.items():
            assert np.array_equal(a, g[f"init.{cfg}.L{i}.{n}"]), (i, n)


def test_closed_form_losses():
    # uniform logits -> ln V (reference tests/test_layers.py:278-283)
    h = np.zeros((1, 3, 4))
    V = np.random.default_rng(0).normal(size=(4, 4))
    assert abs(OL.head_loss(h, V, np.array([[0, 1, 2]])) - math.log(4)) < 1e-12
    # +30 margin on the target -> ~0 (tests/test_layers.py:285-293)
    V = np.eye(4) * 30.0
    h = np.eye(4)[None, :3, :]
    assert OL.head_loss(h, V, np.array([[0, 1, 2]])) < 1e-10


def test_head_grad_finite_difference():
    rng = np.random.default_rng(1)
    h = rng.normal(size=(2, 3, 5))
    V = rng.normal(size=(7, 5))
    y = rng.integers(0, 7, size=(2, 3))
    _, gh, gV = OL.head_loss_grad(h, V, y)
    eps = 1e-6
    for idx in [(0, 1, 2), (1, 2, 4)]:
        hp, hm = h.copy(), h.copy()
        hp[idx] += eps
        hm[idx] -= eps
        fd = (OL.head_loss(hp, V, y) - OL.head_loss(hm, V, y)) / (2 * eps)
        assert abs(fd - gh[idx]) < 1e-8


def test_block_finite_difference():
    rng = np.random.default_rng(2)
    d, f = 6, 10
    V, layers = OO.init_params(5, d, f, 1, 4, 3)
    P = layers[1]
    x = rng.normal(size=(2, 4, d))
    go = rng.normal(size=(2, 4, d))
    seed, p = 99, 0.2

    def obj():
        out, _ = OL.block_fwd(P, x, seed, p, True)
        return float((out * go).sum())

    _, c = OL.block_fwd(P, x, seed, p, True)
    gx, G = OL.block_bwd(P, c, go)
    eps = 1e-6
    for name in ("wq", "wk", "w1", "w2", "ln1_g", "b1"):
        arr = P[name]
        flat = arr.reshape(-1)
        for i in (0, flat.size // 2, flat.size - 1):
            old = flat[i]
            flat[i] = old + eps
            fp = obj()
            flat[i] = old - eps
            fm = obj()
            flat[i] = old
            fd = (fp - fm) / (2 * eps)
            assert abs(fd - G[name].reshape(-1)[i]) < 1e-6 * max(1.0, abs(fd)), name
    for i in (0, 17, x.size - 1):
        xf = x.reshape(-1)
        old = xf[i]
        xf[i] = old + eps
        fp = obj()
        xf[i] = old - eps
        fm = obj()
        xf[i] = old
        assert abs((fp - fm) / (2 * eps) - gx.reshape(-1)[i]) < 1e-6


def oracle_batches(cfg, n):
    vocab, _, _, _, seq, batch, _, _, _, data_seed = CONFIGS[cfg]
    s = Stream(data_seed)
    out = []
    for _ in range(n):
        x = (s.uniform((batch, seq)) * vocab).astype(np.int64)
        y = (s.uniform((batch, seq)) * vocab).astype(np.int64)
        out.append((x, y))
    return out


TRAJ = [
    ("tiny", 1, "adam", 0.005, 8, "sequential"),
    ("tiny", 1, "sgd", 0.005, 8, "pipeline"),
    ("tiny", 2, "adam", 0.005, 8, "pipeline"),
    ("tiny", 3, "sgd", 0.005, 8, "pipeline"),
    ("tiny", 4, "adam", 0.005, 8, "pipeline"),
    ("small", 1, "adam", 0.002, 6, "sequential"),
    ("small", 2, "adam", 0.002, 6, "pipeline"),
    ("small", 4, "sgd", 0.05, 6, "pipeline"),
]


@pytest.mark.parametrize("cfg,K,opt,lr,steps,kind", TRAJ)
def test_trajectory_matches_reference(cfg, K, opt, lr, steps, kind):
    vocab, d, f, nb, seq, batch, p, seed, dseed, _ = CONFIGS[cfg]
    g = load(f"traj_{cfg}_K{K}_{opt}_{kind}.npz")
    V, layers = OO.init_params(vocab, d, f, nb, seq, seed)
    lr_fn = lambda t: OO.lr_at(lr, "fixed", t)  # noqa: E731
    optimizer = OO.Adam(lr_fn) if opt == "adam" else OO.Sgd(lr_fn)
    eng = OO.OuroborosOracle(V, layers, K, dseed, p, optimizer)
    keys = list(g["pk_keys"])
    for t, (x, y) in enumerate(oracle_batches(cfg, steps)):
        loss, pk = eng.step(t, x, y)
        assert abs(loss - g["losses"][t]) <= 1e-12 * abs(g["losses"][t]) + 1e-13
        flat = {k: v for mg in pk["module_grads"] for k, v in mg.items()}
        flat["emb"] = pk["emb_grad"]
        assert sorted(flat) == keys
        sums = np.array([flat[k].sum() for k in keys])
        sqs = np.array([(flat[k] ** 2).sum() for k in keys])
        np.testing.assert_allclose(sqs, g["pk_sq"][t], rtol=1e-9, atol=1e-20)
        np.testing.assert_allclose(sums, g["pk_sum"][t], rtol=1e-7, atol=1e-12)
        sid = [-1 if s is None else s for s in pk["sample_ids"]]
        if kind == "pipeline":
            assert sid == list(g["pk_sid"][t])
    np.testing.assert_allclose(eng.V, g["final.tied"], rtol=1e-9, atol=1e-12)
    for i, P in enumerate(layers):
        for n, a in P.items():
            np.testing.assert_allclose(a, g[f"final.L{i}.{n}"], rtol=1e-9, atol=1e-12)
