"""End-to-end parity of the B200 Ouroboros step against the fp64 CPU oracle.

fp32 check mode (3-pass tf32 GEMMs, fp32 activations): per-step loss and
every packet tensor (module gradients at their stale snapshots, the mixed
tied gradient) and the post-update weights, over a short free run at
K = 1, 2, 4 with SGD and Adam.  Free runs stay comparable for a few steps
before ReLU sign flips make fp32 and fp64 trajectories diverge
(SURVEY.md section 0, fact 3).

Tolerances (stated): loss rel <= 2e-5; packet tensor rel-L2 <= 2e-4;
weights rel-L2 of the update (w_t - w_0) <= 2e-3.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ouroboros as OO  # noqa: E402
from oracle.rng import Stream  # noqa: E402

SMALL = dict(vocab=64, d=32, f=64, blocks=2, seq=16, batch=4, p=0.1, init_seed=5, dseed=9, data_seed=3)


def batches(cfg, n):
    s = Stream(cfg["data_seed"])
    out = []
    for _ in range(n):
        x = (s.uniform((cfg["batch"], cfg["seq"])) * cfg["vocab"]).astype(np.int64)
        y = (s.uniform((cfg["batch"], cfg["seq"])) * cfg["vocab"]).astype(np.int64)
        out.append((x, y))
    return out


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def make_pair(cfg, K, opt, lr, dtype="fp32", concurrent=False):
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O

    stack = M.build_stack(cfg["vocab"], cfg["d"], cfg["f"], cfg["blocks"], cfg["seq"], cfg["p"], cfg["init_seed"],
                          dtype=dtype)
    part = M.partition(stack.num_layers, K)
    cls = E.ConcurrentPipelineEngine if concurrent else E.PipelineEngine
    eng = cls(stack, part, cfg["dseed"])
    sched = O.LrSchedule(lr, "fixed")
    gopt = O.make_optimizer(opt, sched)
    V, layers = OO.init_params(cfg["vocab"], cfg["d"], cfg["f"], cfg["blocks"], cfg["seq"], cfg["init_seed"])
    lr_fn = lambda t: lr  # noqa: E731
    oopt = OO.Adam(lr_fn) if opt == "adam" else OO.Sgd(lr_fn)
    ora = OO.OuroborosOracle(V, layers, K, cfg["dseed"], cfg["p"], oopt)
    return stack, eng, gopt, ora


@pytest.mark.parametrize("K,opt,lr", [(1, "sgd", 0.05), (2, "adam", 2e-3), (4, "sgd", 0.05), (4, "adam", 2e-3)])
def test_fp32_free_run_matches_oracle(K, opt, lr):
    from paper_1909_06695_b200.engine import BatchSample

    cfg = SMALL
    stack, eng, gopt, ora = make_pair(cfg, K, opt, lr)
    init = {"tied": ora.V.copy()}
    steps = 5
    for t, (x, y) in enumerate(batches(cfg, steps)):
        packet, loss = eng.step(t, BatchSample(x, y, t), gopt)
        got = packet.cpu()
        oloss, opk = ora.step(t, x, y)
        assert abs(loss - oloss) <= 2e-5 * abs(oloss), (t, loss, oloss)
        assert got.sample_ids == opk["sample_ids"]
        for k in range(K):
            for key, ref in opk["module_grads"][k].items():
                g = got.module_grads[k][key]
                if not np.any(ref):
                    assert not np.any(g), (t, k, key)
                else:
                    assert rel(g, ref) <= 2e-4, (t, k, key, rel(g, ref))
        if np.any(opk["emb_grad"]):
            assert rel(got.emb_grad, opk["emb_grad"]) <= 2e-4, (t, rel(got.emb_grad, opk["emb_grad"]))
        else:
            assert not np.any(got.emb_grad)
    V_gpu = stack.tied.double().cpu().numpy()
    assert rel(V_gpu - init["tied"], ora.V - init["tied"]) <= 2e-3


def test_concurrent_streams_bitwise_equal_reference_executor():
    from paper_1909_06695_b200.engine import BatchSample

    cfg = SMALL
    _, e1, o1, _ = make_pair(cfg, 3, "adam", 2e-3)
    _, e2, o2, _ = make_pair(cfg, 3, "adam", 2e-3, concurrent=True)
    for t, (x, y) in enumerate(batches(cfg, 6)):
        p1, l1 = e1.step(t, BatchSample(x, y, t), o1)
        c1 = p1.cpu()
        p2, l2 = e2.step(t, BatchSample(x, y, t), o2)
        c2 = p2.cpu()
        assert l1 == l2
        assert np.array_equal(c1.emb_grad, c2.emb_grad)
        for g1, g2 in zip(c1.module_grads, c2.module_grads):
            for key in g1:
                assert np.array_equal(g1[key], g2[key]), key


def test_bf16_loss_tracks_oracle():
    from paper_1909_06695_b200.engine import BatchSample

    cfg = SMALL
    _, eng, gopt, ora = make_pair(cfg, 2, "adam", 2e-3, dtype="bf16")
    for t, (x, y) in enumerate(batches(cfg, 8)):
        _, loss = eng.step(t, BatchSample(x, y, t), gopt)
        oloss, _ = ora.step(t, x, y)
        assert abs(loss - oloss) <= 2e-2 * abs(oloss), (t, loss, oloss)


def test_distributed_engine_single_rank_equals_pipeline_engine():
    """The multi-GPU engine driving real device modules (1 rank, K=2: both
    modules on GPU 0, no communication) is bitwise equal to PipelineEngine."""
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200.distributed import DistributedPipelineEngine, build_local_modules

    cfg = SMALL
    _, e1, o1, _ = make_pair(cfg, 2, "adam", 2e-3, dtype="bf16")
    stack = M.build_stack(cfg["vocab"], cfg["d"], cfg["f"], cfg["blocks"], cfg["seq"], cfg["p"], cfg["init_seed"],
                          dtype="bf16")
    part = M.partition(stack.num_layers, 2)
    mods = build_local_modules(stack, part, cfg["dseed"], 0)
    e2 = DistributedPipelineEngine(mods, part, 0, tied=stack.tied_store, device=stack.runtime.device)
    o2 = O.make_optimizer("adam", O.LrSchedule(2e-3, "fixed"))
    for t, (x, y) in enumerate(batches(cfg, 5)):
        p1, l1 = e1.step(t, E.BatchSample(x, y, t), o1)
        c1 = p1.cpu()
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        p2, l2 = e2.step(t, E.BatchSample(xd, yd, t), o2)
        assert l1 == float(l2)
        assert np.array_equal(c1.emb_grad, p2.emb_grad.double().cpu().numpy())
        for g1, g2 in zip(c1.module_grads, p2.module_grads):
            for key in g1:
                assert np.array_equal(g1[key], g2[key].double().cpu().numpy()), key


@pytest.mark.parametrize("micro", [2, 4])
def test_micro_batched_relay_matches_oracle(micro):
    """The micro-batched relay (distributed.py) on real device
    modules: the batch streams through the modules as `micro` row blocks at
    the same weights; dropout positions and the 1/(B*T) normaliser stay the
    whole batch's, so in the fp32 check mode every step matches the fp64
    oracle like the whole-batch engine does (loss rel <= 2e-5, packets rel-L2
    <= 2e-4), and the weight gradients sum over the row blocks in a fixed
    order (a re-run is bitwise identical)."""
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200.distributed import DistributedPipelineEngine, build_local_modules

    cfg = dict(SMALL, batch=8)
    runs = []
    for _ in range(2):
        _, _, _, ora = make_pair(cfg, 2, "adam", 2e-3)
        stack = M.build_stack(cfg["vocab"], cfg["d"], cfg["f"], cfg["blocks"], cfg["seq"], cfg["p"],
                              cfg["init_seed"], dtype="fp32")
        part = M.partition(stack.num_layers, 2)
        mods = build_local_modules(stack, part, cfg["dseed"], 0)
        eng = DistributedPipelineEngine(mods, part, 0, tied=stack.tied_store, device=stack.runtime.device,
                                        micro_batches=micro)
        opt = O.make_optimizer("adam", O.LrSchedule(2e-3, "fixed"))
        rec = []
        for t, (x, y) in enumerate(batches(cfg, 5)):
            packet, loss = eng.step(t, E.BatchSample(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), t),
                                    opt)
            got = packet.cpu()
            oloss, opk = ora.step(t, x, y)
            assert abs(loss - oloss) <= 2e-5 * abs(oloss), (t, loss, oloss)
            for k in range(2):
                for key, want in opk["module_grads"][k].items():
                    g = got.module_grads[k][key]
                    if not np.any(want):
                        assert not np.any(g), (t, k, key)
                    else:
                        assert rel(g, want) <= 2e-4, (t, k, key, rel(g, want))
            if np.any(opk["emb_grad"]):
                assert rel(got.emb_grad, opk["emb_grad"]) <= 2e-4
            rec.append((loss, got.emb_grad.copy()))
        runs.append(rec)
    for (l1, e1), (l2, e2) in zip(*runs):
        assert l1 == l2 and np.array_equal(e1, e2)


def test_micro_batched_xl_relay_matches_restatement():
    """The same with Transformer-XL blocks: each row block carries its rows of
    the segment memory."""
    from oracle import xl as X
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200.data import SegmentStream
    from paper_1909_06695_b200.distributed import DistributedPipelineEngine, build_local_modules

    c = dict(vocab=64, d=32, f=64, blocks=2, seq=8, mem=8, heads=4, batch=4, p=0.1, init_seed=5, dseed=9)
    stack = M.build_xl_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], c["init_seed"], c["heads"],
                             c["mem"], dtype="fp32")
    part = M.partition(stack.num_layers, 2)
    mods = build_local_modules(stack, part, c["dseed"], 0)
    eng = DistributedPipelineEngine(mods, part, 0, tied=stack.tied_store, device=stack.runtime.device,
                                    micro_batches=2)
    opt = O.make_optimizer("adam", O.LrSchedule(2e-3, "fixed"))
    V, layers = X.init_xl_params(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["heads"], c["init_seed"])
    ora = X.XLOuroborosOracle(V, layers, 2, c["dseed"], c["p"], c["heads"], c["mem"], c["batch"],
                              OO.Adam(lambda t: 2e-3))
    toks = (Stream(2).uniform((c["batch"] * 7 * c["seq"] + 4,)) * c["vocab"]).astype(np.int64)
    src = SegmentStream(toks, c["seq"], c["batch"])
    for t in range(6):
        b = src.batch_at(t)
        packet, loss = eng.step(t, E.BatchSample(torch.as_tensor(b.x).cuda(), torch.as_tensor(b.y).cuda(), t), opt)
        got = packet.cpu()
        oloss, opk = ora.step(t, b.x, b.y)
        assert abs(loss - oloss) <= 2e-5 * abs(oloss), (t, loss, oloss)
        for k in range(2):
            for key, want in opk["module_grads"][k].items():
                g = got.module_grads[k][key]
                if np.any(want):
                    assert rel(g, want) <= 2e-4, (t, k, key, rel(g, want))
