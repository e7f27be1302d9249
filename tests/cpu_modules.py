"""Host-side (fp64, CPU) module doubles for exercising the distributed
schedule with gloo -- TEST INFRASTRUCTURE ONLY.

They implement the module interface DistributedPipelineEngine drives
(input_buffer / forward / pop_slot / recompute_backward / zero_grads /
snapshot / grad_views) with the oracle's layer math, following the
reference ModuleState (model.py:199-304): slots hold the module input and
seeds, the delayed backward recomputes the forward at the ring snapshot.
"""

from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from oracle import layers as OL
from oracle.rng import hash64


@dataclass
class Slot:
    step: int
    sample_id: int
    inputs: object
    targets: object
    seeds: list


class TiedStore:
    def __init__(self, V):
        self.master = torch.from_numpy(V.copy())
        self.grad = torch.zeros_like(self.master)


class CpuModule:
    supports_micro = True

    def __init__(self, index, K, lo, hi, layers, dropout_seed, p, tied, d):
        self.index, self.K, self.lo, self.hi = index, K, lo, hi
        self.params = layers  # list of dicts of numpy arrays (live, shared with the optimizer)
        self.kinds = ["embedding" if i == 0 else ("projection" if not P and i > 0 else "block")
                      for i, P in zip(range(lo, hi), layers)]
        self.has_embedding = self.kinds[0] == "embedding"
        self.has_projection = self.kinds[-1] == "projection"
        self.dropout_seed, self.p, self.tied, self.d = dropout_seed, p, tied, d
        self.cap = K - index + 1
        self.ring = {}
        self.slots = deque()
        self.device = torch.device("cpu")
        self.grads = {}
        for off, P in enumerate(layers):
            for name, a in P.items():
                self.grads[f"L{lo + off}.{name}"] = torch.zeros(a.shape, dtype=torch.float64)
        self.grad_views = self.grads
        self._inputs = {}

    def snapshot(self, t):
        self.ring[t] = ([{n: a.copy() for n, a in P.items()} for P in self.params],
                        self.tied.master.numpy().copy() if self.tied is not None else None)
        for s in sorted(self.ring):
            if len(self.ring) > self.cap:
                del self.ring[s]

    def input_buffer(self, t, B, T, micro=None):
        rows = B * T if micro is None else B // micro[1] * T
        buf = torch.empty(rows, self.d, dtype=torch.float64)
        self._inputs[t] = buf
        return buf

    def _run(self, params, V, x, seeds, train, pos0=0, n_total=None):
        caches = []
        h = x
        for off, kind in enumerate(self.kinds):
            P = params[off]
            if kind == "embedding":
                h, c = OL.embed_fwd(V, P["pos"], h, seeds[off], self.p, train, pos0=pos0)
            elif kind == "block":
                h, c = OL.block_fwd(P, h, seeds[off], self.p, train, pos0=pos0, n_total=n_total)
            else:
                c = None
            caches.append(c)
        return h, caches

    def _forward_block(self, x, step, sample_id, targets, train, out, micro, batch_shape):
        """Row block j of m (the micro-batched relay): the block's rows of the
        whole-batch forward -- dropout positions offset by its first row."""
        j, m = micro
        B, T = batch_shape
        mb = B // m
        seeds = [hash64(self.dropout_seed, step, self.lo + off) for off in range(len(self.kinds))]
        xin = np.asarray(x) if self.has_embedding else x.numpy().reshape(mb, T, -1).copy()
        tg = None if targets is None else np.asarray(targets)
        if j == 0:
            self.slots.append(Slot(step, sample_id, [xin], [tg], seeds))
            if len(self.slots) > self.cap:
                raise RuntimeError("slot overflow")
        else:
            self.slots[-1].inputs.append(xin)
            self.slots[-1].targets.append(tg)
        V = self.tied.master.numpy() if self.tied is not None else None
        h, _ = self._run(self.params, V, xin, seeds, train, pos0=j * mb * T * self.d, n_total=B * T * self.d)
        if self.has_projection:
            self._block_losses = ([] if j == 0 else self._block_losses) + [OL.head_loss(h, V, tg)]
            return torch.tensor(float(np.mean(self._block_losses)), dtype=torch.float64)
        res = torch.from_numpy(np.ascontiguousarray(h.reshape(-1, h.shape[-1])))
        if out is not None:
            out.copy_(res)
            return out
        return res

    def forward(self, x, step, sample_id, targets=None, train=True, out=None, micro=None, batch_shape=None):
        if micro is not None and micro[1] > 1:
            return self._forward_block(x, step, sample_id, targets, train, out, micro, batch_shape)
        seeds = [hash64(self.dropout_seed, step, self.lo + off) for off in range(len(self.kinds))]
        if self.has_embedding:
            xin = np.asarray(x)
        else:
            xin = x.reshape(-1, x.shape[-1]).numpy().reshape(x.shape[0], x.shape[1], -1).copy() if x.dim() == 3 \
                else x.numpy().copy()
        self.slots.append(Slot(step, sample_id, xin, None if targets is None else np.asarray(targets), seeds))
        if len(self.slots) > self.cap:
            raise RuntimeError("slot overflow")
        V = self.tied.master.numpy() if self.tied is not None else None
        h, _ = self._run(self.params, V, xin, seeds, train)
        if self.has_projection:
            return torch.tensor(OL.head_loss(h, V, targets), dtype=torch.float64)
        res = torch.from_numpy(np.ascontiguousarray(h.reshape(-1, h.shape[-1])))
        if out is not None:
            out.copy_(res)
            return out
        return res

    def pop_slot(self):
        return self.slots.popleft()

    def zero_grads(self):
        for g in self.grads.values():
            g.zero_()
        return self.grads

    def _backward_blocks(self, slot, grad_out, train, g_in, emb):
        """Row blocks in order; block 0 writes the weight gradients, later
        blocks add theirs (the device's fixed order)."""
        params, V = self.ring[slot.step]
        m = len(slot.inputs)
        mb, T = slot.inputs[0].shape[0], slot.inputs[0].shape[1]
        B = mb * m
        loss = []
        for j in range(m):
            r0 = j * mb * T
            h, caches = self._run(params, V, slot.inputs[j], slot.seeds, train, pos0=r0 * self.d,
                                  n_total=B * T * self.d)
            if self.has_projection:
                lj, g, dvo = OL.head_loss_grad(h, V, slot.targets[j])
                g, dvo = g / m, dvo / m  # the whole batch's 1/(B*T) normaliser
                loss.append(lj)
                if emb is not None and emb[0]:
                    emb[2].add_(torch.from_numpy(emb[0] * dvo))
            else:
                g = grad_out.numpy().reshape(B, T, self.d)[j * mb:(j + 1) * mb]
            for off in range(len(self.kinds) - 1, -1, -1):
                kind = self.kinds[off]
                if kind == "block":
                    g, G = OL.block_bwd(params[off], caches[off], g)
                    for n, a in G.items():
                        dst = self.grads[f"L{self.lo + off}.{n}"]
                        dst.copy_(torch.from_numpy(a)) if j == 0 else dst.add_(torch.from_numpy(a))
                elif kind == "embedding":
                    dvi, gpos = OL.embed_bwd(g, caches[off], V.shape[0], params[off]["pos"].shape)
                    dst = self.grads[f"L{self.lo + off}.pos"]
                    dst.copy_(torch.from_numpy(gpos)) if j == 0 else dst.add_(torch.from_numpy(gpos))
                    if emb is not None and emb[1]:
                        emb[2].add_(torch.from_numpy(emb[1] * dvi))
                    g = None
            if g is not None and g_in is not None:
                g_in[j * mb * T:(j + 1) * mb * T].copy_(torch.from_numpy(np.ascontiguousarray(g.reshape(-1, self.d))))
        return g_in, self.grads, {}, (float(np.mean(loss)) if loss else None)

    def recompute_backward(self, slot, grad_out, stale_mode="snapshot", train=True, *, g_in=None, emb=None,
                           live_step=None):
        if isinstance(slot.inputs, list):
            return self._backward_blocks(slot, grad_out, train, g_in, emb)
        params, V = self.ring[slot.step]
        h, caches = self._run(params, V, slot.inputs, slot.seeds, train)
        B, T = (slot.inputs.shape[0], slot.inputs.shape[1])
        loss = None
        if self.has_projection:
            loss, g, dvo = OL.head_loss_grad(h, V, slot.targets)
            if emb is not None and emb[0]:
                emb[2].add_(torch.from_numpy(emb[0] * dvo))
        else:
            g = grad_out.numpy().reshape(B, T, self.d)
        for off in range(len(self.kinds) - 1, -1, -1):
            kind = self.kinds[off]
            if kind == "block":
                g, G = OL.block_bwd(params[off], caches[off], g)
                for n, a in G.items():
                    self.grads[f"L{self.lo + off}.{n}"].copy_(torch.from_numpy(a))
            elif kind == "embedding":
                dvi, gpos = OL.embed_bwd(g, caches[off], V.shape[0], params[off]["pos"].shape)
                self.grads[f"L{self.lo + off}.pos"].copy_(torch.from_numpy(gpos))
                if emb is not None and emb[1]:
                    emb[2].add_(torch.from_numpy(emb[1] * dvi))
                g = None
        if g is not None and g_in is not None:
            g_in.copy_(torch.from_numpy(np.ascontiguousarray(g.reshape(B * T, self.d))))
        return g_in, self.grads, {}, loss


class CpuSgd:
    """w -= lr * g on the live numpy params and the tied master (optim.py:60-75)."""

    def __init__(self, lr):
        self.lr = lr

    def apply(self, t, packet, modules, tied):
        for m in modules:
            for off, P in enumerate(m.params):
                for n, a in P.items():
                    a -= self.lr * m.grads[f"L{m.lo + off}.{n}"].numpy()
        if tied is not None:
            tied -= self.lr * packet.emb_grad
        return self.lr
