"""gloo runs of DistributedPipelineEngine (the multi-GPU schedule: ring
placement, P2P relay of activations on one process group, boundary-gradient
exchange one step later on another, tied gradient on rank 0) against the
single-process oracle.

world size 2 -> K = 3 modules (1 and 3 on rank 0, 2 on rank 1); world size 3
-> K = 4 (1 and 4 on rank 0); reference model.py:137-140.  Each with the
whole-batch relay and the micro-batched relay (the batch streams through the
ring as m row blocks; dropout positions and the loss normaliser stay those of
the whole batch, weight gradients sum over the blocks in a fixed order).
Module compute is the fp64 oracle layer math (tests/cpu_modules.py), so
packets must match the oracle to ~1e-12."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ouroboros as OO
from oracle.rng import Stream

CFG = dict(vocab=11, d=8, f=12, blocks=4, seq=5, batch=4, p=0.15, init_seed=4, dseed=6, data_seed=2)
STEPS = 6
LR = 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _batches():
    s = Stream(CFG["data_seed"])
    out = []
    for _ in range(STEPS):
        x = (s.uniform((CFG["batch"], CFG["seq"])) * CFG["vocab"]).astype(np.int64)
        y = (s.uniform((CFG["batch"], CFG["seq"])) * CFG["vocab"]).astype(np.int64)
        out.append((x, y))
    return out


class _Batch:
    def __init__(self, x, y, sid, shape):
        self.x, self.y, self.sample_id, self.shape = x, y, sid, shape


def _worker(rank, world, port, K, outdir, micro=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_modules import CpuModule, CpuSgd, TiedStore
        from paper_1909_06695_b200.distributed import DistributedPipelineEngine
        from paper_1909_06695_b200.model import partition

        V, layers = OO.init_params(CFG["vocab"], CFG["d"], CFG["f"], CFG["blocks"], CFG["seq"], CFG["init_seed"])
        part = partition(len(layers), K)
        tied = TiedStore(V) if rank == 0 else None
        mods = {}
        for k, (lo, hi) in enumerate(part.groups, start=1):
            if part.device_of[k - 1] == rank:
                mods[k] = CpuModule(k, K, lo, hi, layers[lo:hi], CFG["dseed"], CFG["p"],
                                    tied if (lo == 0 or hi == len(layers)) else None, CFG["d"])
        eng = DistributedPipelineEngine(mods, part, rank, tied=tied, d_model=CFG["d"], grad_dtype=torch.float64,
                                        micro_batches=micro)
        opt = CpuSgd(LR)
        rec = {}
        for t, (x, y) in enumerate(_batches()):
            b = _Batch(x if rank == 0 else None, y if rank == 0 else None, t, (CFG["batch"], CFG["seq"]))
            packet, loss = eng.step(t, b, opt)
            if loss is not None:
                rec[f"loss.{t}"] = np.array(float(loss))
            for g in packet.module_grads:
                for key, v in g.items():
                    rec[f"g.{t}.{key}"] = v.numpy().copy()
            if packet.emb_grad is not None:
                rec[f"emb.{t}"] = packet.emb_grad.numpy().copy()
            rec[f"sid.{t}"] = np.array([-1 if s is None else s for s in packet.sample_ids])
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **rec)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,micro", [(2, 1), (2, 2), (3, 1), (3, 4)])
def test_ring_matches_oracle(world, micro):
    K = world + 1
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), K, d, micro), nprocs=world, join=True)
        recs = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    r0 = recs[0]
    V, layers = OO.init_params(CFG["vocab"], CFG["d"], CFG["f"], CFG["blocks"], CFG["seq"], CFG["init_seed"])
    ora = OO.OuroborosOracle(V, layers, K, CFG["dseed"], CFG["p"], OO.Sgd(lambda t: LR))
    for t, (x, y) in enumerate(_batches()):
        loss, pk = ora.step(t, x, y)
        assert abs(r0[f"loss.{t}"] - loss) <= 1e-12 * abs(loss)
        for k, mg in enumerate(pk["module_grads"], start=1):
            rec = r0 if k in (1, K) else recs[k - 1]
            for key, ref in mg.items():
                np.testing.assert_allclose(rec[f"g.{t}.{key}"], ref, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(r0[f"emb.{t}"], pk["emb_grad"], rtol=1e-10, atol=1e-13)
        # rank 0 reports modules (1, K), rank r module r + 1
        sids = pk["sample_ids"]
        assert list(r0[f"sid.{t}"]) == [-1 if s is None else s for s in (sids[0], sids[-1])]
        for r in range(1, world):
            assert list(recs[r][f"sid.{t}"]) == [-1 if sids[r] is None else sids[r]]


def test_hop_order_is_global():
    """Relay hops k->k+1 and boundary hops k->k-1 follow the ring owners."""
    from paper_1909_06695_b200.model import partition

    for K in range(2, 10):
        part = partition(K + 3, K)
        owners = part.device_of
        relay = [(owners[k - 1], owners[k]) for k in range(1, K)]
        back = [(owners[k - 1], owners[k - 2]) for k in range(K, 1, -1)]
        assert relay[0][0] == 0 and back[-1][1] == 0
        assert all(a != b for a, b in relay) or K == 2
