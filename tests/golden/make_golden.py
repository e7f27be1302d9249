"""Generates tests/golden/*.npz by running the live reference `ringpipe`.

Run in the build container only (the reference tree is not shipped to the GPU
box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/) to the reference: RNG prefix,
partitions, parameter init, and full training trajectories (losses, per-key
packet checksums, final weights) of `PipelineEngine` / `SequentialRunner`
at K = 1..4 with SGD and Adam, dropout on.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from ringpipe.engine import BatchSample, PipelineEngine, SequentialRunner  # noqa: E402
from ringpipe.model import build_stack, partition  # noqa: E402
from ringpipe.optim import LrSchedule, make_optimizer  # noqa: E402
from ringpipe.tensor import SeededRng  # noqa: E402

# name -> (vocab, dim, ffn, blocks, seq, batch, dropout, init_seed, dropout_seed, data_seed)
CONFIGS = {
    # the reference test-suite's tiny stack (tests/test_engine.py:20-39)
    "tiny": (7, 8, 8, 3, 4, 2, 0.2, 11, 7, 1),
    # GPU-friendly shapes (dims multiple of 8 for TMA): the parity config
    "small": (64, 32, 64, 2, 16, 4, 0.1, 5, 9, 3),
}
RUNS = [
    # (config, K, optimizer, lr, steps, engine)
    ("tiny", 1, "adam", 0.005, 8, "sequential"),
    ("tiny", 1, "sgd", 0.005, 8, "pipeline"),
    ("tiny", 2, "adam", 0.005, 8, "pipeline"),
    ("tiny", 3, "sgd", 0.005, 8, "pipeline"),
    ("tiny", 4, "adam", 0.005, 8, "pipeline"),
    ("small", 1, "adam", 0.002, 6, "sequential"),
    ("small", 2, "adam", 0.002, 6, "pipeline"),
    ("small", 4, "sgd", 0.05, 6, "pipeline"),
]


def batches(cfg, n):
    vocab, _, _, _, seq, batch, _, _, _, data_seed = CONFIGS[cfg]
    rng = SeededRng(data_seed)
    out = []
    for t in range(n):
        x = (rng.uniform((batch, seq)) * vocab).astype(np.int64)
        y = (rng.uniform((batch, seq)) * vocab).astype(np.int64)
        out.append(BatchSample(x, y, t))
    return out


def stack_for(cfg):
    vocab, dim, ffn, blocks, seq, _, p, init_seed, _, _ = CONFIGS[cfg]
    return build_stack(vocab, dim, ffn, blocks, seq, p, init_seed)


def run(cfg, K, opt_kind, lr, steps, engine_kind):
    stack = stack_for(cfg)
    dropout_seed = CONFIGS[cfg][8]
    part = partition(stack.num_layers, K)
    if engine_kind == "sequential":
        eng = SequentialRunner(stack, part, dropout_seed)
    else:
        eng = PipelineEngine(stack, part, dropout_seed)
    opt = make_optimizer(opt_kind, LrSchedule(lr, "fixed"))
    out = {}
    losses, sums, sqs, sids = [], [], [], []
    keys = None
    for t, b in enumerate(batches(cfg, steps)):
        packet, loss = eng.step(t, b, opt)
        losses.append(loss)
        flat = {key: g for grads in packet.module_grads for key, g in grads.items()}
        flat["emb"] = packet.emb_grad
        keys = sorted(flat)
        sums.append([flat[k].sum() for k in keys])
        sqs.append([(flat[k] ** 2).sum() for k in keys])
        sids.append([-1 if s is None else s for s in packet.sample_ids])
    out["losses"] = np.array(losses)
    out["pk_keys"] = np.array(keys)
    out["pk_sum"] = np.array(sums)
    out["pk_sq"] = np.array(sqs)
    out["pk_sid"] = np.array(sids)
    out["final.tied"] = stack.tied.copy()
    for i, P in enumerate(stack.params):
        for n, a in P.items():
            if n != "tied":
                out[f"final.L{i}.{n}"] = a.copy()
    return out


def main():
    data = {"rng_prefix": SeededRng(1).uniform((3,)), "rng_mid": SeededRng(12345, 1000).uniform((5,))}
    for L_, K in [(12, 4), (5, 3), (8, 2), (8, 5), (14, 9), (6, 2), (12, 1)]:
        p = partition(L_, K)
        data[f"part.{L_}.{K}.groups"] = np.array(p.groups)
        data[f"part.{L_}.{K}.dev"] = np.array(p.device_of)
    p = partition(4, 2, balance="by_cost", costs=[10.0, 1.0, 1.0, 1.0])
    data["part.bycost.groups"] = np.array(p.groups)
    costs = [3.0, 1.0, 4.0, 1.0, 5.0, 9.0, 2.0, 6.0]
    p = partition(8, 3, balance="by_cost", costs=costs)
    data["part.bycost2.groups"] = np.array(p.groups)
    for cfg in CONFIGS:
        st = stack_for(cfg)
        data[f"init.{cfg}.tied"] = st.tied
        for i, P in enumerate(st.params):
            for n, a in P.items():
                if n != "tied":
                    data[f"init.{cfg}.L{i}.{n}"] = a
    np.savez_compressed(os.path.join(HERE, "reference_basics.npz"), **data)
    for cfg, K, opt, lr, steps, kind in RUNS:
        res = run(cfg, K, opt, lr, steps, kind)
        name = f"traj_{cfg}_K{K}_{opt}_{kind}.npz"
        np.savez_compressed(os.path.join(HERE, name), **res)
        print(name, "losses", res["losses"], file=sys.stderr)


if __name__ == "__main__":
    main()
