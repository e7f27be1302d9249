"""Schedule semantics of the B200 engines, mirroring the reference's own
tests (tests/test_engine.py:47-310, tests/test_model.py:131-220) on the
reference's tiny stack (vocab 7, dim 8, ffn 8, seq 4, batch 2 -- odd vocab
and T exercise the padded layouts), fp32 check mode."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ouroboros as OO  # noqa: E402
from oracle.rng import Stream  # noqa: E402

VOCAB, DIM, SEQ = 7, 8, 4


def make_batches(n, batch=2, seed=1):
    # reference tests/test_engine.py:26-33
    from paper_1909_06695_b200.engine import BatchSample

    rng = Stream(seed)
    out = []
    for t in range(n):
        x = (rng.uniform((batch, SEQ)) * VOCAB).astype(np.int64)
        y = (rng.uniform((batch, SEQ)) * VOCAB).astype(np.int64)
        out.append(BatchSample(x, y, t))
    return out


def make_engine(K, blocks=3, dropout=0.1, seed=11, concurrent=False, **kw):
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M

    stack = M.build_stack(VOCAB, DIM, DIM, blocks, SEQ, dropout, seed, dtype="fp32")
    part = M.partition(stack.num_layers, K)
    cls = E.ConcurrentPipelineEngine if concurrent else E.PipelineEngine
    return stack, cls(stack, part, dropout_seed=7, **kw)


def all_zero(grads):
    return all(not torch.any(g) for g in grads.values())


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_exhaustive_zero_padding(K):
    stack, engine = make_engine(K, blocks=8)
    for t, batch in enumerate(make_batches(K + 2)):
        packet, _ = engine.step(t, batch)
        for k in range(1, K + 1):
            if t - K + k < 0:
                assert all_zero(packet.module_grads[k - 1])
                assert packet.sample_ids[k - 1] is None
            else:
                assert not all_zero(packet.module_grads[k - 1])
                assert packet.sample_ids[k - 1] == t - K + k
        assert bool(torch.any(packet.emb_grad)) == (t - K + 1 >= 0)


def test_oracle_equivalence_tiny_k3():
    """Every delayed gradient equals full backprop at its snapshot (the
    reference's test_delayed_grads_match_sequential_at_snapshots config)."""
    from paper_1909_06695_b200.optim import LrSchedule, make_optimizer

    stack, engine = make_engine(3, blocks=3, dropout=0.2)
    opt = make_optimizer("sgd", LrSchedule(0.005, "fixed"))
    V, layers = OO.init_params(VOCAB, DIM, DIM, 3, SEQ, 11)
    ora = OO.OuroborosOracle(V, layers, 3, 7, 0.2, OO.Sgd(lambda t: 0.005))
    for t, b in enumerate(make_batches(10)):
        packet, loss = engine.step(t, b, opt)
        got = packet.cpu()
        oloss, opk = ora.step(t, b.x, b.y)
        assert abs(loss - oloss) <= 2e-5 * abs(oloss)
        for k in range(3):
            for key, ref in opk["module_grads"][k].items():
                g = got.module_grads[k][key]
                den = np.linalg.norm(ref)
                if den == 0:
                    assert not np.any(g)
                else:
                    assert np.linalg.norm(g - ref) / den <= 5e-4, (t, key)
        den = np.linalg.norm(opk["emb_grad"])
        if den:
            assert np.linalg.norm(got.emb_grad - opk["emb_grad"]) / den <= 5e-4


def test_tie_identity_and_shared_views():
    from paper_1909_06695_b200.optim import LrSchedule, make_optimizer

    stack, engine = make_engine(3)
    opt = make_optimizer("adam", LrSchedule(0.01, "fixed"))
    emb = engine.modules[0].params[0]
    proj = engine.modules[-1].params[-1]
    for t, b in enumerate(make_batches(4)):
        engine.step(t, b, opt)
        assert emb["tied"] is proj["tied"] is stack.tied
    assert engine.modules[0].params[0] is stack.params[0]


def test_staleness_and_one_step_behind():
    from paper_1909_06695_b200.engine import check_one_step_behind

    K = 4
    stack, engine = make_engine(K, blocks=4)
    for t, b in enumerate(make_batches(9)):
        packet, _ = engine.step(t, b)
        for sid in packet.sample_ids:
            if sid is not None:
                assert 0 <= t - sid <= K - 1
        assert packet.sample_ids[-1] == t
    assert check_one_step_behind(engine.trace, K)
    for k in range(1, K + 1):
        assert engine.trace.idle_backward_steps(k, from_step=K) == []
        assert engine.trace.idle_backward_steps(k) == list(range(K - k))


def test_k1_pipeline_equals_sequential_runner_bitwise():
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200.optim import LrSchedule, make_optimizer

    sa = M.build_stack(VOCAB, DIM, DIM, 2, SEQ, 0.1, 11, dtype="fp32")
    sb = M.build_stack(VOCAB, DIM, DIM, 2, SEQ, 0.1, 11, dtype="fp32")
    ea = E.PipelineEngine(sa, M.partition(sa.num_layers, 1), dropout_seed=7)
    eb = E.SequentialRunner(sb, M.partition(sb.num_layers, 2), dropout_seed=7)
    oa = make_optimizer("adam", LrSchedule(0.01))
    ob = make_optimizer("adam", LrSchedule(0.01))
    for t, b in enumerate(make_batches(6)):
        pa, la = ea.step(t, b, oa)
        ca = pa.cpu()
        pb, lb = eb.step(t, b, ob)
        assert la == lb
        assert np.array_equal(ca.emb_grad, pb.emb_grad.double().cpu().numpy())
        assert pb.sample_ids == [t, t]
    assert torch.equal(sa.tied, sb.tied)


def test_sum_convention_is_twice_half_avg():
    _, e1 = make_engine(2, blocks=2, dropout=0.0)
    _, e2 = make_engine(2, blocks=2, dropout=0.0, tied_grad="sum")
    for t, b in enumerate(make_batches(3)):
        p1, _ = e1.step(t, b)
        g1 = p1.emb_grad.clone()
        p2, _ = e2.step(t, b)
        assert torch.allclose(p2.emb_grad, 2.0 * g1, rtol=0, atol=0)


def test_current_mode_equals_snapshot_before_drift_then_differs():
    from paper_1909_06695_b200.optim import LrSchedule, make_optimizer

    _, es = make_engine(3, blocks=3, dropout=0.1)
    _, ec = make_engine(3, blocks=3, dropout=0.1, stale_weights="current")
    os_, oc = make_optimizer("sgd", LrSchedule(0.05)), make_optimizer("sgd", LrSchedule(0.05))
    diffs = []
    for t, b in enumerate(make_batches(5)):
        ps, _ = es.step(t, b, os_)
        cs = ps.cpu()
        pc, _ = ec.step(t, b, oc)
        cc = pc.cpu()
        same = all(np.array_equal(cs.module_grads[0][k], cc.module_grads[0][k]) for k in cs.module_grads[0])
        diffs.append(same)
    # module 1 first backs up sample 0 at step 2, when live weights already moved
    assert not all(diffs[2:])


def test_slot_overflow_and_missing_snapshot_raise():
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200.errors import ScheduleViolation

    stack = M.build_stack(VOCAB, DIM, DIM, 1, SEQ, 0.1, 11, dtype="fp32")
    part = M.partition(stack.num_layers, 2)
    m1, m2 = M.build_modules(stack, part, 3)
    toks = torch.zeros(2, SEQ, dtype=torch.int64, device="cuda")
    for s in range(2):
        m1.snapshot(s)
        m1.forward(toks, s, s)
    with pytest.raises(ScheduleViolation):
        m1.snapshot(2)
        m1.forward(toks, 2, 2)
    slot = m1.pop_slot()
    m1.snapshot(5)
    m1.snapshot(6)  # evicts step 0's entry (capacity 2)
    with pytest.raises(ScheduleViolation):
        m1.recompute_backward(slot, None)


def test_out_of_range_token_raises_dimension_error():
    from paper_1909_06695_b200.engine import BatchSample
    from paper_1909_06695_b200.errors import DimensionError

    _, engine = make_engine(2, blocks=2)
    x = np.full((2, SEQ), VOCAB, dtype=np.int64)  # one past the vocabulary
    with pytest.raises(DimensionError):
        engine.step(0, BatchSample(x, np.zeros_like(x), 0))


def test_nan_weights_abort_with_worker_failure_naming_module():
    # reference tests/test_engine.py:251-261
    from paper_1909_06695_b200.errors import WorkerFailure

    stack, conc = make_engine(3, blocks=3, concurrent=True)
    conc.modules[1].params[0]["wq"][:] = float("nan")
    stack.refresh()
    with pytest.raises(WorkerFailure) as excinfo:
        for t, b in enumerate(make_batches(4)):
            conc.step(t, b)
    assert "module 2" in str(excinfo.value)
    conc.close()


def test_packet_norm_deterministic_and_matches_host():
    from paper_1909_06695_b200.engine import packet_grad_sq_norm

    _, engine = make_engine(2, blocks=2)
    bs = make_batches(2)
    engine.step(0, bs[0])
    packet, _ = engine.step(1, bs[1])
    a = packet_grad_sq_norm(packet)
    assert a == packet_grad_sq_norm(packet) and a > 0
    host = packet.cpu()
    ref = sum(float((g * g).sum()) for mg in host.module_grads for g in mg.values()) + float((host.emb_grad ** 2).sum())
    assert abs(a - ref) <= 1e-9 * ref


@pytest.mark.parametrize("K", [1, 2])
def test_out_of_range_host_ids_raise_before_any_update(K):
    """Host batches are range-checked before a launch (reference layers.py:116-117):
    no weight moves, at K=1 too (where the embedding scatter runs in the same step)."""
    from paper_1909_06695_b200.engine import BatchSample
    from paper_1909_06695_b200.errors import DimensionError

    stack, engine = make_engine(K, blocks=2)
    before = stack.tied.detach().clone()
    for bad in (VOCAB, -1):
        x = np.zeros((2, SEQ), dtype=np.int64)
        x[1, 2] = bad
        with pytest.raises(DimensionError):
            engine.step(0, BatchSample(x, np.zeros_like(x), 0))
        with pytest.raises(DimensionError):
            engine.step(0, BatchSample(np.zeros_like(x), x, 0))
    torch.cuda.synchronize()
    assert torch.equal(stack.tied, before)


@pytest.mark.parametrize("K", [1, 2])
def test_out_of_range_device_ids_are_contained(K):
    """Device-resident ids are checked by the kernels: the forward raises the
    dimension flag and the tied-gradient scatter skips ids outside [0, V), so
    a bad id (V, or negative) never addresses memory and the context stays
    usable (the K=1 scatter runs in the same step)."""
    from paper_1909_06695_b200.engine import BatchSample
    from paper_1909_06695_b200.errors import DimensionError

    batches = make_batches(K + 2)
    for bad in (VOCAB, -5, 2 ** 33):
        stack, engine = make_engine(K, blocks=2)
        x = torch.zeros((2, SEQ), dtype=torch.int64, device="cuda")
        x[0, 1] = bad
        y = torch.zeros_like(x)
        with pytest.raises(DimensionError):
            # K=2: step 0's slot (bad ids) is scattered at step 1, before the poll
            for t in range(K):
                engine.step(t, BatchSample(x, y, t), sync=(t == K - 1))
        torch.cuda.synchronize()  # no illegal address
    # a fresh engine on the same device still runs and matches the oracle's loss
    stack2, engine2 = make_engine(K, blocks=2)
    _, loss = engine2.step(0, batches[0])
    assert np.isfinite(loss)


def _snapshot_params(params):
    return [{n: v.detach().clone() for n, v in P.items()} for P in params]


@pytest.mark.parametrize("opt_kind", ["sgd", "adam"])
def test_delayed_grads_match_sequential_gradients_at_snapshots(opt_kind):
    """Reference tests/test_engine.py:145-190 through the drop-in
    `sequential_gradients(layers, params_list, batch, dropout_seed, step)`
    (engine.py:409-440): every delayed module gradient equals full backprop
    at the snapshot it was taken at -- exactly (same kernels, same inputs,
    deterministic reductions); the mixed tied gradient 0.5 Vo(t) + 0.5 Vi(t-K+1)
    to fp32 rounding of the two-term sum (the reference sums in fp64)."""
    from paper_1909_06695_b200.engine import sequential_gradients
    from paper_1909_06695_b200.optim import LrSchedule, make_optimizer

    K, steps = 3, 10
    batches = make_batches(steps)
    stack, engine = make_engine(K, blocks=3, dropout=0.2)
    opt = make_optimizer(opt_kind, LrSchedule(0.005, "fixed"))
    packets, snapshots = [], []
    for t, batch in enumerate(batches):
        snapshots.append(_snapshot_params(stack.params))
        packet, _ = engine.step(t, batch, opt)
        packets.append(packet.cpu())
    live = [{n: v.detach().clone() for n, v in P.items()} for P in stack.params]
    part = engine.part
    seq = {}
    for s in range(steps):
        seq[s] = sequential_gradients(stack.layers, snapshots[s], batches[s], dropout_seed=7, step=s)
        grads, vi, vo, loss, logits = seq[s]
        assert logits.shape == (2, SEQ, VOCAB)
        for k in range(1, K + 1):
            t = s + K - k
            if t >= steps:
                continue
            got = packets[t].module_grads[k - 1]
            start, end = part.groups[k - 1]
            for key, ref in grads.items():
                if start <= int(key.split(".")[0][1:]) < end:
                    diff = np.abs(got[key] - ref).max()
                    assert diff == 0.0, f"t={t} k={k} {key}: {diff}"
    for t in range(K - 1, steps):
        expect = 0.5 * seq[t][2] + 0.5 * seq[t - K + 1][1]
        assert np.abs(packets[t].emb_grad - expect).max() <= 1e-6 * np.abs(expect).max()
    # the live weights were not touched by the oracle calls
    for P, Q in zip(stack.params, live):
        for n in P:
            assert torch.equal(P[n], Q[n])
