"""Teacher-forced per-step parity (SURVEY 8(c) protocol item 1).

BASELINE configs[0] (C1: 4 blocks, d 128, d_ff 512, V 1000, T 64, B 16,
dropout 0.1), K = 1, 2 and 4 modules, Adam and SGD, 30 steps.  Every step
the complete fp64 state of the oracle (the restatement pinned to the live
reference's trajectories, tests/test_oracle.py) is rounded to fp32 and loaded
into the device engine -- weights, Adam moments, snapshot rings, the pending
stale slots (their tapes re-derived on the device from the slot inputs at the
snapshot weights) and the boundary gradients -- through the same
`runner.restore_state` the checkpoint loader uses.  The device runs ONE
Ouroboros step in the fp32 check mode; then

  * the loss                                     rel <= 1e-6
  * every tensor of the packet (the K delayed module gradients, the mixed
    tied gradient, zero padding)                 rel-L2 <= 2e-4 (+ kink bound),
                                                 median <= 5e-5
  * every parameter's update w^{t+1} - w^t (all 4 blocks, positions, the
    tied matrix) against the fp64 optimizer (optim.py:60-126) applied to the
    same state and to the packet's gradient: rel-L2 <= 1e-5 plus the fp32
    rounding of w^{t+1} (2^-23 ||w^{t+1}||)

against the oracle's own step from the same state (the pattern of reference
tests/test_engine.py:145-209 and engine.py:409-440).  The update is checked
on the device's gradient because Adam's first steps are sign-like
(m / sqrt(v) = g / |g|): an element whose gradient is within tolerance of 0
takes a full +-lr step either way, so the update of the oracle's gradient
is not a meaningful target -- the packet check covers the gradient, this one
the optimizer arithmetic.  Then the oracle -- not the device -- advances.

ReLU kinks: a pre-activation within rounding of zero can
take the other side of the kink in fp32 than in fp64, which moves that
element's whole gradient contribution -- one such element shifts a position
gradient by ~1e-3.  The oracle therefore also back-propagates with every
"ambiguous" pre-activation (|z1| < 1e-5 rms(z1)) flipped; the difference of
the two fp64 gradients bounds what a flip can do, and each tensor may deviate
by at most 2e-4 of its norm plus that bound (and the update check is skipped
for a tensor whose bound exceeds 5e-5 of its gradient).  The test reports
how many (step, tensor) pairs needed the allowance.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import layers as OL  # noqa: E402
from oracle import ouroboros as OO  # noqa: E402
from oracle.rng import Stream, hash64  # noqa: E402

C1 = dict(vocab=1000, d=128, f=512, blocks=4, seq=64, batch=16, p=0.1, init_seed=11, dseed=7)
STEPS = 30
TAU = 1e-5  # ambiguous pre-activation band, relative to rms(z1)
# per-tensor rel-L2 of the packet: the tf32x3 GEMMs are ~1e-6 relative, and the
# softmax backward dS = P (dP - D) cancels (dP ~ D), which amplifies it to the
# 1e-5 .. 1e-4 measured on the attention weights (also at the C2 shape with the
# ReLU pattern forced, tests/test_production_gpu.py)
TOL = 2e-4
LR = {"adam": 1e-3, "sgd": 0.05}


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b.ravel())
    if nb == 0.0:
        return float(np.linalg.norm(a.ravel()))
    return float(np.linalg.norm((a - b).ravel()) / nb)


def batches():
    s = Stream(1)
    out = []
    for _ in range(STEPS):
        x = (s.uniform((C1["batch"], C1["seq"])) * C1["vocab"]).astype(np.int64)
        y = (s.uniform((C1["batch"], C1["seq"])) * C1["vocab"]).astype(np.int64)
        out.append((x, y))
    return out


def trace(V, layers, x, y, step):
    """fp64 full backprop of one sample that also keeps every layer
    boundary: hs[i] = input of layer i, gs[i] = dL/d(input of layer i)."""
    nl = len(layers)
    hs = [x]
    h, ce = OL.embed_fwd(V, layers[0]["pos"], x, hash64(C1["dseed"], step, 0), C1["p"], True)
    caches = []
    for i in range(1, nl - 1):
        hs.append(h)
        h, c = OL.block_fwd(layers[i], h, hash64(C1["dseed"], step, i), C1["p"], True)
        caches.append(c)
    hs.append(h)
    _, g, _ = OL.head_loss_grad(h, V, y)
    gs = {nl - 1: g}
    for i in range(nl - 2, 0, -1):
        g, _ = OL.block_bwd(layers[i], caches[i - 1], g)
        gs[i] = g
    return hs, gs


def kink_grads(V, layers, x, y, step):
    """fp64 full backprop twice: with the fp64 ReLU pattern and with every
    ambiguous pre-activation flipped.  Returns (G, dVi, dVo, loss, bound)
    where bound[key] = ||G_flipped - G|| (and "Vi", "Vo")."""
    nl = len(layers)
    h, ce = OL.embed_fwd(V, layers[0]["pos"], x, hash64(C1["dseed"], step, 0), C1["p"], True)
    caches = []
    for i in range(1, nl - 1):
        h, c = OL.block_fwd(layers[i], h, hash64(C1["dseed"], step, i), C1["p"], True)
        caches.append(c)
    loss, g_head, dVo = OL.head_loss_grad(h, V, y)

    def backward(cs):
        G = {}
        g = g_head
        for i in range(nl - 2, 0, -1):
            g, Gi = OL.block_bwd(layers[i], cs[i - 1], g)
            for n, a in Gi.items():
                G[f"L{i}.{n}"] = a
        dVi, gpos = OL.embed_bwd(g, ce, V.shape[0], layers[0]["pos"].shape)
        G["L0.pos"] = gpos
        return G, dVi

    G, dVi = backward(caches)
    flipped = []
    for c in caches:
        z = c["z1"]
        amb = np.abs(z) < TAU * np.sqrt(np.mean(z * z))
        flipped.append(dict(c, z1=np.where(amb, -z, z)))
    G2, dVi2 = backward(flipped)
    bound = {k: float(np.linalg.norm(G2[k] - G[k])) for k in G}
    bound["Vi"] = float(np.linalg.norm(dVi2 - dVi))
    bound["Vo"] = 0.0  # the head has no ReLU
    return G, dVi, dVo, loss, bound


class KinkOracle(OO.OuroborosOracle):
    """The oracle, plus the kink bound of every sample it differentiates."""

    bounds = None

    def _full_grads(self, t, x, y):
        G, dVi, dVo, loss, bound = kink_grads(self.V, self.layers, x, y, t)
        if self.bounds is None:
            self.bounds = {}
        self.bounds[t] = bound
        return G, dVi, dVo, loss


class Teacher:
    """The oracle plus the history the device state needs (snapshots w^s and
    batches of the pending samples)."""

    def __init__(self, K, kind):
        V, layers = OO.init_params(C1["vocab"], C1["d"], C1["f"], C1["blocks"], C1["seq"], C1["init_seed"])
        self.K = K
        self.kind = kind
        opt = OO.Adam(lambda t: LR["adam"]) if kind == "adam" else OO.Sgd(lambda t: LR["sgd"])
        self.ora = KinkOracle(V, layers, K, C1["dseed"], C1["p"], opt)
        self.groups = self.ora.groups
        self.snaps = {}
        self.data = batches()
        self._traces = {}

    def weights(self):
        return self.ora.V, self.ora.layers

    def record(self, t):
        self.snaps[t] = (self.ora.V.copy(), OO.copy_layers(self.ora.layers))
        for s in [s for s in self.snaps if s < t - self.K]:
            del self.snaps[s]

    def _trace(self, s):
        if s not in self._traces:
            V, layers = self.snaps[s]
            self._traces[s] = trace(V, layers, *self.data[s], s)
        return self._traces[s]

    def state_arrays(self, t):
        """The device state at the start of step t, named like a checkpoint."""
        K, nl = self.K, len(self.ora.layers)
        A = {"stack.tied": self.ora.V}
        for i, P in enumerate(self.ora.layers):
            for n, a in P.items():
                A[f"stack.L{i}.{n}"] = a
        if self.kind == "adam":
            for key in ["tied"] + OO.flat_keys(self.ora.layers):
                if key in self.ora.opt.m:
                    A[f"optim.adam.m.{key}"] = self.ora.opt.m[key]
                    A[f"optim.adam.v.{key}"] = self.ora.opt.v[key]
        for k, (lo, hi) in enumerate(self.groups, start=1):
            pre = f"m{k}."
            for s in range(max(0, t - K + k), t):  # ring: the pending samples' weights
                V, layers = self.snaps[s]
                for i in range(lo, hi):
                    for n, a in layers[i].items():
                        A[f"{pre}ring.{s}.L{i}.{n}"] = a
                if lo == 0:
                    A[f"{pre}ring.{s}.L0.tied"] = V  # module 1 re-derives its embedding from V^s
            if k == K:
                continue  # module K's slot is consumed in its own step
            for j, s in enumerate(range(max(0, t - K + k), t)):
                x, _ = self.data[s]
                hs, _ = self._trace(s)
                A[f"{pre}slot{j}.meta"] = np.array([s, s], dtype=np.int64)
                A[f"{pre}slot{j}.seeds"] = np.array([hash64(C1["dseed"], s, i) for i in range(lo, hi)],
                                                    dtype=np.uint64)
                A[f"{pre}slot{j}.inputs"] = x if lo == 0 else hs[lo]
        for k in range(1, K):  # boundary[k] = dL/d(output of module k), sample t-K+k
            s = t - K + k
            if s < 0:
                continue
            _, gs = self._trace(s)
            A[f"boundary.{k}"] = gs[self.groups[k][0]]
        for s in [s for s in self._traces if s < t - K + 1]:
            del self._traces[s]
        return A


def device_engine(K, kind):
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O

    c = C1
    stack = M.build_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], c["init_seed"], dtype="fp32")
    eng = E.PipelineEngine(stack, M.partition(stack.num_layers, K), c["dseed"])
    opt = O.make_optimizer(kind, O.LrSchedule(LR[kind], "fixed"))
    if hasattr(opt, "bind"):
        opt.bind(eng.modules)
    return stack, eng, opt


def host_params(stack):
    out = {"tied": stack.tied.detach().double().cpu().numpy()}
    for i, P in enumerate(stack.params):
        for n, v in P.items():
            if n != "tied":
                out[f"L{i}.{n}"] = v.detach().double().cpu().numpy()
    return out


@pytest.mark.parametrize("K,kind", [(1, "adam"), (2, "adam"), (4, "adam"), (2, "sgd"), (4, "sgd")])
def test_teacher_forced_steps_match_oracle(K, kind):
    from paper_1909_06695_b200.engine import BatchSample
    from paper_1909_06695_b200.runner import restore_state

    teacher = Teacher(K, kind)
    stack, eng, opt = device_engine(K, kind)
    worst = {"loss": 0.0, "packet": 0.0, "update": 0.0}
    allowed = checked = 0
    errs = []
    for t in range(STEPS):
        teacher.record(t)
        state = teacher.state_arrays(t)
        # the moments as loaded (fp32), for the optimizer check below
        m_pre = {k[len("optim.adam.m."):]: np.float32(v).astype(np.float64) for k, v in state.items()
                 if k.startswith("optim.adam.m.")}
        v_pre = {k[len("optim.adam.v."):]: np.float32(v).astype(np.float64) for k, v in state.items()
                 if k.startswith("optim.adam.v.")}
        restore_state(stack, eng, opt, state, t)
        before = host_params(stack)
        x, y = teacher.data[t]
        packet, loss = eng.step(t, BatchSample(x, y, t), opt)
        got = packet.cpu()
        after = host_params(stack)
        w0 = {"tied": teacher.ora.V.copy(), **{f"L{i}.{n}": a.copy() for i, P in enumerate(teacher.ora.layers)
                                              for n, a in P.items()}}
        oloss, opk = teacher.ora.step(t, x, y)
        w1 = {"tied": teacher.ora.V, **{f"L{i}.{n}": a for i, P in enumerate(teacher.ora.layers)
                                       for n, a in P.items()}}
        e = abs(loss - oloss) / abs(oloss)
        worst["loss"] = max(worst["loss"], e)
        assert e <= 1e-6, (t, loss, oloss)
        kinked = set()
        for k in range(K):
            s_ = opk["sample_ids"][k]
            assert got.sample_ids[k] == s_
            for key, want in opk["module_grads"][k].items():
                g = got.module_grads[k][key]
                if not np.any(want):
                    assert not np.any(g), (t, k, key)
                    continue
                nrm = np.linalg.norm(want)
                b = teacher.ora.bounds[s_][key] / nrm
                e = rel(g, want)
                errs.append(e)
                checked += 1
                if e > TOL:
                    allowed += 1
                    kinked.add(key)
                else:
                    worst["packet"] = max(worst["packet"], e)
                assert e <= TOL + 1.01 * b, (t, k, key, e, b)
        if np.any(opk["emb_grad"]):
            s_in, s_out = t - K + 1, t
            b = (0.5 * teacher.ora.bounds[s_in]["Vi"] + 0.5 * teacher.ora.bounds[s_out]["Vo"]) \
                / np.linalg.norm(opk["emb_grad"])
            e = rel(got.emb_grad, opk["emb_grad"])
            errs.append(e)
            checked += 1
            if e > TOL:
                allowed += 1
                kinked.add("tied")
            else:
                worst["packet"] = max(worst["packet"], e)
            assert e <= TOL + 1.01 * b, (t, "emb", e, b)
        else:
            assert not np.any(got.emb_grad)
        # the optimizer on the device's own gradient, in fp64 (optim.py:60-126)
        gdev = {"tied": got.emb_grad}
        for mg in got.module_grads:
            gdev.update(mg)
        for key in w1:
            g = gdev[key]
            if kind == "sgd":
                want = -LR["sgd"] * g
            else:
                b1, b2, eps = 0.9, 0.999, 1e-8
                m = b1 * m_pre.get(key, 0.0) + (1 - b1) * g
                v = b2 * v_pre.get(key, 0.0) + (1 - b2) * g * g
                want = -LR["adam"] * (m / (1 - b1 ** (t + 1))) / (np.sqrt(v / (1 - b2 ** (t + 1))) + eps)
            if not np.any(want):
                continue
            err = np.linalg.norm((after[key] - before[key]) - want)
            allow = 1e-5 * np.linalg.norm(want) + 2.0 ** -23 * np.linalg.norm(after[key])
            worst["update"] = max(worst["update"], err / np.linalg.norm(want))
            assert err <= allow, (t, key, err / np.linalg.norm(want), allow / np.linalg.norm(want))
    q50, q95 = np.quantile(errs, [0.5, 0.95])
    print(f"teacher-forced C1 K={K} {kind}: worst loss rel {worst['loss']:.1e}; packet rel-L2 median {q50:.1e}, "
          f"p95 {q95:.1e}, max within tolerance {worst['packet']:.1e} (kink allowance used on {allowed} of "
          f"{checked} tensors); update vs fp64 optimizer {worst['update']:.1e}")
    assert q50 <= 5e-5
