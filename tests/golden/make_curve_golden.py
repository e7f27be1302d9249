"""Generates tests/golden/c1_curve.npz: the live reference's 500-step loss
curve at BASELINE configs[0] (C1: vocab 1000, d 128, f 512, 4 blocks, T 64,
B 16, dropout 0.1), Ouroboros K=2 (`PipelineEngine`), Adam lr 1e-3, on a
learnable synthetic stream (SURVEY 8(c) parity protocol item 3: the bf16
production loss curve against the reference's fp64 curve).

Run in the build container only (takes ~10 min on one core):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_curve_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from curve_data import C1, STEPS, batch_at  # noqa: E402
from ringpipe.engine import BatchSample, PipelineEngine  # noqa: E402
from ringpipe.model import build_stack, partition  # noqa: E402
from ringpipe.optim import LrSchedule, make_optimizer  # noqa: E402


def main():
    c = C1
    stack = build_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], c["init_seed"])
    eng = PipelineEngine(stack, partition(stack.num_layers, c["K"]), c["dseed"])
    opt = make_optimizer("adam", LrSchedule(c["lr"], "fixed"))
    losses = []
    for t in range(STEPS):
        x, y = batch_at(t)
        _, loss = eng.step(t, BatchSample(x, y, t), opt)
        losses.append(loss)
        if t % 50 == 0:
            print(t, loss, file=sys.stderr, flush=True)
    np.savez_compressed(os.path.join(HERE, "c1_curve.npz"), losses=np.array(losses))


if __name__ == "__main__":
    main()
