"""The fp64 Transformer-XL restatement (oracle/xl.py).  The reference has no
XL path, so parity is pinned by (1) reduction to the reference block, which
oracle/layers.py matches against the live reference's goldens, and (2)
central finite differences for every parameter with memory present."""

import numpy as np
import pytest

from oracle import layers as L
from oracle import xl as X
from oracle.rng import Stream

B, T, M, D, H, F = 2, 5, 3, 8, 2, 12


def rand_params(rs, d=D, f=F, h=H, zero_rel=False):
    P = {"ln1_g": 1.0 + 0.1 * rs.uniform_signed((d,), 1.0), "ln1_b": 0.1 * rs.uniform_signed((d,), 1.0)}
    for w in ("wq", "wk", "wv", "wo", "wr"):
        P[w] = rs.uniform_signed((d, d), 0.5)
    P["r_w_bias"] = rs.uniform_signed((h, d // h), 0.5)
    P["r_r_bias"] = rs.uniform_signed((h, d // h), 0.5)
    P["ln2_g"] = 1.0 + 0.1 * rs.uniform_signed((d,), 1.0)
    P["ln2_b"] = 0.1 * rs.uniform_signed((d,), 1.0)
    P["w1"] = rs.uniform_signed((d, f), 0.5)
    P["b1"] = 0.1 * rs.uniform_signed((f,), 1.0)
    P["w2"] = rs.uniform_signed((f, d), 0.5)
    P["b2"] = 0.1 * rs.uniform_signed((d,), 1.0)
    if zero_rel:
        for k in ("wr", "r_w_bias", "r_r_bias"):
            P[k] = np.zeros_like(P[k])
    return P


def test_rel_shift_adjoint_and_index():
    rs = Stream(3)
    a = rs.uniform((2, T, M + T))
    b = rs.uniform((2, T, M + T))
    assert np.isclose((X.rel_shift(a, T) * b).sum(), (a * X.rel_shift_back(b, T)).sum())
    s = X.rel_shift(a, T)
    for i in range(T):
        for j in range(M + i + 1):  # every visible key reads row T-1-i+j = Kl-1-distance
            assert s[0, i, j] == a[0, i, T - 1 - i + j]
    R = X.sinusoid(M + T, D)
    assert np.allclose(R[-1], np.r_[np.zeros(D // 2), np.ones(D // 2)])  # distance 0


def test_reduces_to_reference_block():
    rs = Stream(11)
    P = rand_params(rs, h=1, zero_rel=True)
    x = rs.uniform_signed((B, T, D), 1.0)
    mem = rs.uniform_signed((B, M, D), 1.0)  # masked: mem_len = 0
    ref_P = {k: P[k] for k in L.BLOCK_KEYS}
    for train in (False, True):
        y_ref, c_ref = L.block_fwd(ref_P, x, 99, 0.2, train)
        y_xl, c_xl = X.xl_block_fwd(P, x, mem, 0, 1, 99, 0.2, train)
        np.testing.assert_allclose(y_xl, y_ref, rtol=1e-12, atol=1e-12)
        g = rs.uniform_signed((B, T, D), 1.0)
        gx_ref, G_ref = L.block_bwd(ref_P, c_ref, g)
        gx_xl, G_xl = X.xl_block_bwd(P, c_xl, g)
        np.testing.assert_allclose(gx_xl, gx_ref, rtol=1e-10, atol=1e-12)
        for k in L.BLOCK_KEYS:
            np.testing.assert_allclose(G_xl[k], G_ref[k], rtol=1e-10, atol=1e-12, err_msg=k)


@pytest.mark.parametrize("mem_len", [M, 1])
def test_block_finite_differences(mem_len):
    rs = Stream(5 + mem_len)
    P = rand_params(rs)
    x = rs.uniform_signed((B, T, D), 1.0)
    mem = rs.uniform_signed((B, M, D), 1.0)
    wout = rs.uniform_signed((B, T, D), 1.0)

    def loss():
        y, _ = X.xl_block_fwd(P, x, mem, mem_len, H, 7, 0.25, True)
        return float((y * wout).sum())

    _, c = X.xl_block_fwd(P, x, mem, mem_len, H, 7, 0.25, True)
    gx, G = X.xl_block_bwd(P, c, wout)
    G["x"] = gx
    P_all = dict(P, x=x)
    h = 1e-6
    for name, arr in P_all.items():
        flat = arr.reshape(-1)
        for idx in range(0, flat.size, max(1, flat.size // 7)):
            old = flat[idx]
            flat[idx] = old + h
            lp = loss()
            flat[idx] = old - h
            lm = loss()
            flat[idx] = old
            fd = (lp - lm) / (2 * h)
            an = G[name].reshape(-1)[idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, an)


def test_memory_receives_no_gradient_and_masking():
    rs = Stream(21)
    P = rand_params(rs)
    x = rs.uniform_signed((B, T, D), 1.0)
    mem = rs.uniform_signed((B, M, D), 1.0)
    y0, _ = X.xl_block_fwd(P, x, mem, 0, H, 7, 0.0, False)
    y1, _ = X.xl_block_fwd(P, x, mem * 5.0, 0, H, 7, 0.0, False)
    np.testing.assert_array_equal(y0, y1)  # invalid memory rows are invisible
    y2, _ = X.xl_block_fwd(P, x, mem * 5.0, M, H, 7, 0.0, False)
    assert np.abs(y2 - y0).max() > 1e-3  # valid ones are not


def test_xl_model_finite_differences():
    V, layers = X.init_xl_params(11, D, F, 2, T, H, 3)
    rs = Stream(8)
    x = (rs.uniform((B, T)) * 11).astype(np.int64)
    y = (rs.uniform((B, T)) * 11).astype(np.int64)
    mems = [rs.uniform_signed((B, M, D), 1.0) for _ in range(2)]
    G, dVi, dVo, loss, new_mems = X.xl_full_grads(V, layers, x, y, 4, 2, 0.1, mems, M, H)
    assert len(new_mems) == 2 and new_mems[0].shape == (B, M, D)
    h = 1e-6
    checks = [("tied", V, dVi + dVo)] + [(k, layers[int(k.split(".")[0][1:])][k.split(".", 1)[1]], g)
                                          for k, g in G.items()]
    for name, arr, an in checks:
        flat = arr.reshape(-1)
        for idx in range(0, flat.size, max(1, flat.size // 3)):
            old = flat[idx]
            flat[idx] = old + h
            lp = X.xl_forward_loss(V, layers, x, y, 4, 2, 0.1, mems, M, H)
            flat[idx] = old - h
            lm = X.xl_forward_loss(V, layers, x, y, 4, 2, 0.1, mems, M, H)
            flat[idx] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - an.reshape(-1)[idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx)
