"""bf16 production loss curve against the live reference's fp64 curve
(SURVEY 8(c) parity protocol item 3): BASELINE configs[0] (C1), Ouroboros
K=2, Adam, 500 steps of a learnable synthetic stream
(tests/curve_data.py; fixture by tests/golden/make_curve_golden.py).

Stated tolerance: the running-mean loss stays within 2% (relative) of the
reference's at every step, and the mean over the last 100 steps within 1%."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from curve_data import C1, STEPS, batch_at  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "c1_curve.npz")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_c1_loss_curve_tracks_reference(dtype):
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O

    ref = np.load(GOLD)["losses"]
    assert ref.shape == (STEPS,)
    c = C1
    stack = M.build_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], c["init_seed"], dtype=dtype)
    eng = E.ConcurrentPipelineEngine(stack, M.partition(stack.num_layers, c["K"]), c["dseed"])
    opt = O.make_optimizer("adam", O.LrSchedule(c["lr"], "fixed"))
    losses = []
    for t in range(STEPS):
        x, y = batch_at(t)
        _, loss = eng.step(t, E.BatchSample(x, y, t), opt, sync=False)
        losses.append(loss.clone())  # the device loss buffer is reused next step
    ours = torch.stack(losses).double().cpu().numpy()
    eng.runtime.check("curve", eng.modules)
    run_ours = np.cumsum(ours) / np.arange(1, STEPS + 1)
    run_ref = np.cumsum(ref) / np.arange(1, STEPS + 1)
    worst = float(np.max(np.abs(run_ours - run_ref) / run_ref))
    print(f"\n{dtype}: running-mean worst rel {worst:.2e}", end="")
    assert worst <= 0.02, worst
    tail = abs(ours[-100:].mean() - ref[-100:].mean()) / ref[-100:].mean()
    print(f", last-100 mean rel {tail:.2e}")
    assert tail <= 0.01, tail
    assert ref[-100:].mean() < 0.8 * ref[:10].mean()  # the stream is learnable: the curve really falls
