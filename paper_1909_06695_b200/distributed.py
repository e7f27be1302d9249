"""Multi-GPU Ouroboros: one process per GPU, modules placed on a ring.

`partition(L, K)` puts module k on device `device_of[k-1]` = [0, 1, .., K-2, 0]
(reference model.py:137-140): G GPUs run K = G + 1 modules and GPU 0 hosts
both the first module (embedding) and the last (projection + loss), so both
halves of the tied gradient are produced on GPU 0 and there is no all-reduce.
The only collectives are point-to-point:

  relay    module k -> k+1   activations [B*T, d]  (compute dtype), in order k = 1..K-1
  boundary module k -> k-1   dL/dx       [B*T, d]  (fp32), produced at step t,
                                                     consumed at step t+1, in order k = K..2

Every rank walks the same global hop order and only takes part in the hops
that touch it, so blocking send/recv cannot deadlock.  With NCCL the sends
and receives are stream-ordered after the producing kernels; a rank's stale
backward overlaps the other ranks' relay work.

The engine is written against a small module interface (input_buffer,
forward, pop_slot, recompute_backward, zero_grads, snapshot, grad_views) so
the exchange logic is exercised on CPU with gloo by tests that plug in
host-side module doubles (tests/test_distributed_cpu.py).
"""

import os

import torch
import torch.distributed as dist

from .engine import GradientPacket, tied_coefficients
from .errors import ScheduleViolation


class P2P:
    """torch.distributed point-to-point transport (nccl on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group

    def send(self, t, dst):
        dist.send(t.contiguous(), dst, group=self.group)

    def recv(self, t, src):
        if t.is_contiguous():
            dist.recv(t, src, group=self.group)
        else:
            tmp = torch.empty_like(t, memory_format=torch.contiguous_format)
            dist.recv(tmp, src, group=self.group)
            t.copy_(tmp)


def rank_env():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class DistributedPipelineEngine:
    """Ouroboros step over several processes (reference engine.py:246-259).

    modules: {k: module} for the modules this rank owns (device_of[k-1] == rank).
    tied:    the TiedMatrix-like store on the Ouroboros rank (0), else None.
    Returns (packet of the local modules, loss) -- the loss on rank 0 (which
    owns module K), None elsewhere.
    """

    def __init__(self, modules, part, rank, tied=None, tied_grad="half_avg", stale_weights="snapshot", train=True,
                 transport=None, d_model=None, grad_dtype=torch.float32, device=None):
        self.part = part
        self.K = part.k
        self.rank = rank
        self.owner = list(part.device_of)
        self.mods = dict(modules)
        for k, m in self.mods.items():
            if self.owner[k - 1] != rank:
                raise ValueError(f"module {k} lives on rank {self.owner[k - 1]}, not {rank}")
        self.tied = tied
        self.tied_grad = tied_grad
        self.stale_weights = stale_weights
        self.train = train
        self.p2p = transport or P2P()
        self.d = d_model if d_model is not None else next(iter(self.mods.values())).d
        self.grad_dtype = grad_dtype  # boundary gradients (fp32 on the GPU path)
        self.device = device
        self.boundary = {}  # k -> dL/d(input of module k+1) consumed by module k this step
        self._next_boundary = {}
        self._bufs = {}

    def _buf(self, key, shape, dtype, device):
        b = self._bufs.get(key)
        if b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype:
            b = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = b
        return b

    def owns(self, k):
        return self.owner[k - 1] == self.rank

    # -- phases -------------------------------------------------------------
    def _relay(self, t, x, y, sid, B, T):
        out_loss = None
        cur = x
        for k in range(1, self.K + 1):
            if not self.owns(k):
                continue
            m = self.mods[k]
            if k > 1 and not self.owns(k - 1):
                buf = m.input_buffer(t, B, T)
                self.p2p.recv(buf, self.owner[k - 2])
                cur = buf.view(B, T, -1)
            nxt_local = k < self.K and self.owns(k + 1)
            out = self.mods[k + 1].input_buffer(t, B, T) if nxt_local else None
            res = m.forward(cur, t, sid, y if m.has_projection else None, self.train, out=out)
            if k == self.K:
                out_loss = res
            else:
                if not nxt_local:
                    self.p2p.send(res.reshape(B * T, -1), self.owner[k])
                cur = res.view(B, T, -1)
        return out_loss

    def _backward(self, t, B, T):
        coef = tied_coefficients(t, self.K, self.tied_grad)
        if self.tied is not None:
            self.tied.grad.zero_()
        sids = {}
        produced = {}
        for k in sorted(self.mods):  # any order: inputs are local by now
            m = self.mods[k]
            s = t - self.K + k
            if s < 0:
                m.zero_grads()
                sids[k] = None
                continue
            slot = m.pop_slot()
            if slot.step != s:
                raise ScheduleViolation(f"module {k} popped slot for step {slot.step}, expected {s}")
            grad_out = None
            if not m.has_projection:
                if k not in self.boundary:
                    raise ScheduleViolation(f"module {k} missing boundary gradient")
                grad_out = self.boundary[k]
            g_in = None
            if k > 1:
                g_in = self._buf(("g", k, t & 1), (B * T, self.d), self.grad_dtype, self.device or grad_out_device(m))
            emb = None
            if self.tied is not None and (m.has_embedding or m.has_projection):
                emb = (coef[0] if m.has_projection else 0.0, coef[1] if m.has_embedding else 0.0, self.tied.grad)
            m.recompute_backward(slot, grad_out, self.stale_weights, self.train, g_in=g_in, emb=emb, live_step=t)
            sids[k] = slot.sample_id
            if k > 1:
                produced[k] = g_in
        return sids, produced

    def _exchange(self, t, produced, B, T):
        nb = {}
        for k in range(self.K, 1, -1):
            if t - self.K + k < 0:
                continue  # module k was still zero-padded: no boundary for k-1
            src, dst = self.owner[k - 1], self.owner[k - 2]
            if src == self.rank and dst == self.rank:
                nb[k - 1] = produced[k]
            elif src == self.rank:
                self.p2p.send(produced[k], dst)
            elif dst == self.rank:
                buf = self._buf(("b", k - 1, t & 1), (B * T, self.d), self.grad_dtype,
                                self.device or grad_out_device(self.mods[k - 1]))
                self.p2p.recv(buf, src)
                nb[k - 1] = buf
        self.boundary = nb

    def step(self, t, batch, optimizer=None):
        if t < 0:
            raise ValueError("step index must be >= 0")
        x = batch.x
        y = batch.y
        if self.owns(1):
            B, T = x.shape
        else:
            B, T = x.shape if x is not None else batch.shape
        for m in self.mods.values():
            m.snapshot(t)
        loss = self._relay(t, x, y, batch.sample_id, B, T)
        sids, produced = self._backward(t, B, T)
        self._exchange(t, produced, B, T)
        mods = [self.mods[k] for k in sorted(self.mods)]
        packet = GradientPacket(t, [m.grad_views for m in mods],
                                self.tied.grad if self.tied is not None else None,
                                [sids[k] for k in sorted(self.mods)], loss)
        if optimizer is not None:
            optimizer.apply(t, packet, mods, self.tied.master if self.tied is not None else None)
        return packet, loss


def grad_out_device(m):
    return getattr(m, "device", torch.device("cpu"))


def build_local_modules(stack, part, dropout_seed, rank):
    """This rank's ModuleStates (GPU path)."""
    from .model import build_modules

    return {m.index: m for m in build_modules(stack, part, dropout_seed) if part.device_of[m.index - 1] == rank}
