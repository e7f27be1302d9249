"""engine.step(sync="lagged"): the host reads each step's loss one step later
from pinned memory; the losses equal the synchronous run's, bad ids raise at
the next step's read (reference exception classes)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.rng import Stream  # noqa: E402


def _run(concurrent, sync, steps=5, bad_at=None):
    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as MD
    from paper_1909_06695_b200 import optim as O

    stack = MD.build_stack(64, 32, 64, 2, 8, 0.1, 3, dtype="bf16")
    cls = E.ConcurrentPipelineEngine if concurrent else E.PipelineEngine
    eng = cls(stack, MD.partition(stack.num_layers, 2), 7)
    opt = O.make_optimizer("adam", O.LrSchedule(1e-3, "fixed"))
    rs = Stream(4)
    out = []
    for t in range(steps):
        x = (rs.uniform((2, 8)) * 64).astype(np.int64)
        y = (rs.uniform((2, 8)) * 64).astype(np.int64)
        if bad_at == t:
            x = torch.from_numpy(x).cuda()
            x[0, 0] = 64  # a device batch: checked by the kernels, reported through the status word
        _, loss = eng.step(t, E.BatchSample(x, y, t), opt, sync=sync)
        out.append(loss)
    if sync == "lagged":
        out = out[1:] + [eng.flush_lagged()]
    return out


@pytest.mark.parametrize("concurrent", [False, True])
def test_lagged_losses_equal_synchronous(concurrent):
    a = _run(concurrent, True)
    b = _run(concurrent, "lagged")
    assert a == b


def test_lagged_reports_bad_ids_at_the_next_read():
    from paper_1909_06695_b200.errors import DimensionError

    with pytest.raises(DimensionError, match="step 2"):
        _run(False, "lagged", bad_at=2)
