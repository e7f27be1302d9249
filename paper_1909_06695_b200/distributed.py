"""Multi-GPU Ouroboros: one process per GPU, modules placed on a ring.

`partition(L, K)` puts module k on device `device_of[k-1]` = [0, 1, .., K-2, 0]
(reference model.py:137-140): G GPUs run K = G + 1 modules and GPU 0 hosts
both the first module (embedding) and the last (projection + loss), so both
halves of the tied gradient are produced on GPU 0 and there is no all-reduce.
The only collectives are point-to-point:

  relay    module k -> k+1   activations [B*T, d]  (compute dtype), hops k = 1..K-1
  boundary module k -> k-1   dL/dx       [B*T, d]  (fp32), produced at step t,
                                                     consumed at step t+1, hops k = K..2

Schedule per rank and step t (the dependencies of reference engine.py:246-259,
SURVEY 7.3):

  * the stale backward of every local module k < K depends only on last
    step's boundary gradient, so it is issued FIRST, on the module's own
    backward stream -- it runs while this rank waits for the relay;
  * the relay runs on the modules' forward streams; activations leave and
    arrive on a dedicated relay communication stream (its own process group,
    so its NCCL communicator and stream are independent of the boundary's);
  * module K's backward (rank 0) follows its fresh forward;
  * boundary gradients leave on a second communication stream/group as soon
    as their producing backward is done and land in a ping-pong buffer read
    by the next step's stale backward;
  * each module's optimizer update follows its own backward on its stream,
    the tied update follows both tied halves (rank 0).

Deadlock freedom: NCCL point-to-point operations on one communicator execute
in issue order on both peers, so every rank issues its relay hops in the
global order k = 1..K-1 and its boundary hops in the global order k = K..2;
relay and boundary use separate groups (separate communicators/streams), so
neither direction waits behind the other.  On CPU (gloo, host-blocking
send/recv) the same global orders make the run deadlock-free too.

Micro-batched relay (`micro_batches=m`): the batch is split into
m row blocks that stream through the ring at the same weights w^t, so rank
r+1 starts module k+1's forward of block j while rank r computes block j+1;
the delayed backward of a slot runs its m row blocks in a fixed order and
sums their weight gradients in that order (deterministic; the loss
normaliser stays N = B*T and dropout positions stay the flat [B, T, d]
indices, so only the fp32 summation order differs from m = 1).

The engine is written against a small module interface (input_buffer,
forward, pop_slot, recompute_backward, zero_grads, snapshot, grad_views) so
the exchange logic is exercised on CPU with gloo by tests that plug in
host-side module doubles (tests/test_distributed_cpu.py).
"""

import contextlib
import os

import torch
import torch.distributed as dist

from .engine import GradientPacket, tied_coefficients
from .errors import DimensionError, NonFiniteError, ScheduleViolation, WorkerFailure


class P2P:
    """torch.distributed point-to-point transport (nccl on GPUs, gloo on CPU).

    Relay and boundary traffic use separate process groups: each gets its own
    NCCL communicator (and internal stream), so the two directions never
    serialise behind each other."""

    def __init__(self, relay_group=None, boundary_group=None):
        self.groups = {"relay": relay_group, "boundary": boundary_group}

    @classmethod
    def create(cls):
        if not dist.is_initialized() or dist.get_world_size() == 1:
            return cls()
        ranks = list(range(dist.get_world_size()))
        return cls(dist.new_group(ranks), dist.new_group(ranks))

    def send(self, t, dst, kind="relay"):
        dist.send(t.contiguous(), dst, group=self.groups[kind])

    def recv(self, t, src, kind="relay"):
        if t.is_contiguous():
            dist.recv(t, src, group=self.groups[kind])
        else:
            tmp = torch.empty_like(t, memory_format=torch.contiguous_format)
            dist.recv(tmp, src, group=self.groups[kind])
            t.copy_(tmp)


def rank_env():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class _Streams:
    """CUDA streams/events on a GPU rank; no-ops on a CPU (gloo) rank."""

    def __init__(self, device):
        self.gpu = device is not None and torch.device(device).type == "cuda"
        self.device = device

    def new(self, priority=0):
        return torch.cuda.Stream(device=self.device, priority=priority) if self.gpu else None

    def ctx(self, s):
        return torch.cuda.stream(s) if s is not None else contextlib.nullcontext()

    def record(self, s=None):
        if not self.gpu:
            return None
        ev = torch.cuda.Event()
        ev.record(s if s is not None else torch.cuda.current_stream(self.device))
        return ev

    @staticmethod
    def wait(s, ev):
        if s is not None and ev is not None:
            s.wait_event(ev)


class DistributedPipelineEngine:
    """Ouroboros step over several processes (reference engine.py:246-259).

    modules: {k: module} for the modules this rank owns (device_of[k-1] == rank).
    tied:    the TiedMatrix-like store on the Ouroboros rank (0), else None.
    Returns (packet of the local modules, loss) -- the loss on rank 0 (which
    owns module K), None elsewhere.
    """

    def __init__(self, modules, part, rank, tied=None, tied_grad="half_avg", stale_weights="snapshot", train=True,
                 transport=None, d_model=None, grad_dtype=torch.float32, device=None, micro_batches=1):
        self.part = part
        self.K = part.k
        self.rank = rank
        self.owner = list(part.device_of)
        self.mods = dict(modules)
        for k, m in self.mods.items():
            if self.owner[k - 1] != rank:
                raise ValueError(f"module {k} lives on rank {self.owner[k - 1]}, not {rank}")
        if micro_batches < 1:
            raise ValueError("micro_batches must be >= 1")
        self.tied = tied
        self.tied_grad = tied_grad
        self.stale_weights = stale_weights
        self.train = train
        self.p2p = transport or P2P.create()
        self.d = d_model if d_model is not None else next(iter(self.mods.values())).d
        self.grad_dtype = grad_dtype  # boundary gradients (fp32 on the GPU path)
        self.device = device
        self.micro = micro_batches
        self.boundary = {}  # k -> dL/d(input of module k+1) consumed by module k this step
        self._boundary_ev = {}  # k -> event: boundary[k] has landed
        self._bufs = {}
        self.streams = _Streams(device)
        S = self.streams
        # the relay and module K's backward are the critical path: high priority
        self._fs = {k: S.new(-1) for k in self.mods}
        self._bs = {k: S.new(-1 if k == self.K else 0) for k in self.mods}
        self._comm = {"relay": S.new(-1), "boundary": S.new(0)}
        self._ts = S.new(0)
        self.last_loss_device = None

    def _buf(self, key, shape, dtype, device):
        b = self._bufs.get(key)
        if b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype:
            b = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = b
        return b

    def owns(self, k):
        return self.owner[k - 1] == self.rank

    def _dev(self, m):
        return self.device or getattr(m, "device", torch.device("cpu"))

    def _micro_ok(self, m, B):
        if self.micro > 1 and (B % self.micro != 0 or not getattr(m, "supports_micro", False)):
            raise DimensionError(f"micro-batching needs B % m == 0 and row-block capable modules (B={B}, m={self.micro})")

    # -- phases -------------------------------------------------------------
    def _stale_backward(self, t, k, coef, B, T, hooks):
        """Delayed backward of local module k (sample t-K+k), issued on its
        backward stream; returns the gradient w.r.t. its input (k > 1)."""
        m = self.mods[k]
        S = self.streams
        s_ = t - self.K + k
        if s_ < 0:
            with S.ctx(self._bs[k]):
                m.zero_grads()
            return None, None
        slot = m.pop_slot()
        if slot.step != s_:
            raise ScheduleViolation(f"module {k} popped slot for step {slot.step}, expected {s_}")
        grad_out = None
        if not m.has_projection:
            if k not in self.boundary:
                raise ScheduleViolation(f"module {k} missing boundary gradient")
            grad_out = self.boundary[k]
            S.wait(self._bs[k], self._boundary_ev.get(k))
        g_in = None
        if k > 1:
            g_in = self._buf(("g", k, t & 1), (B * T, self.d), self.grad_dtype, self._dev(m))
        emb = None
        if self.tied is not None and (m.has_embedding or m.has_projection):
            emb = (coef[0] if m.has_projection else 0.0, coef[1] if m.has_embedding else 0.0, self.tied.grad)
        with S.ctx(self._bs[k]):
            kw = dict(g_in=g_in, emb=emb, live_step=t)
            if hooks is not None:
                kw.update(hooks)
            m.recompute_backward(slot, grad_out, self.stale_weights, self.train, **kw)
        return g_in, slot.sample_id

    def _relay(self, t, x, y, sid, B, T, start_ev):
        """Forward relay of batch t (or its m row blocks) through the local modules."""
        S = self.streams
        comm = self._comm["relay"]
        out_loss = None
        fwd_done = {}
        m_ = self.micro
        mb = B // m_
        for j in range(m_):
            micro = (j, m_) if m_ > 1 else None
            kw_mb = {"micro": micro, "batch_shape": (B, T)} if micro else {}
            prev_ev = start_ev
            for k in range(1, self.K + 1):
                if not self.owns(k):
                    continue
                m = self.mods[k]
                self._micro_ok(m, B)
                fs = self._fs[k]
                S.wait(fs, start_ev)
                cur = x[j * mb:(j + 1) * mb] if (k == 1 and micro) else x
                if k > 1:
                    buf = m.input_buffer(t, B, T, micro=micro) if micro else m.input_buffer(t, B, T)
                    if not self.owns(k - 1):
                        S.wait(comm, start_ev)
                        with S.ctx(comm):
                            self.p2p.recv(buf, self.owner[k - 2], "relay")
                        S.wait(fs, S.record(comm))
                    else:
                        S.wait(fs, prev_ev)
                    cur = buf.view(-1, T, self.d)
                nxt_local = k < self.K and self.owns(k + 1)
                out = None
                if nxt_local:
                    nm = self.mods[k + 1]
                    out = nm.input_buffer(t, B, T, micro=micro) if micro else nm.input_buffer(t, B, T)
                yin = y if m.has_projection else None
                if yin is not None and micro:
                    yin = yin[j * mb:(j + 1) * mb]
                with S.ctx(fs):
                    res = m.forward(cur, t, sid, yin, self.train, out=out, **kw_mb)
                ev = S.record(fs)
                prev_ev = ev
                fwd_done[k] = ev
                if k == self.K:
                    out_loss = res
                elif not nxt_local:
                    S.wait(comm, ev)
                    with S.ctx(comm):
                        self.p2p.send(res.reshape(-1, self.d), self.owner[k], "relay")
        return out_loss, fwd_done

    def _exchange(self, t, produced, bwd_ev, B, T, start_ev):
        """Boundary gradients for step t+1, in the global hop order k = K..2."""
        S = self.streams
        comm = self._comm["boundary"]
        # receive buffers of parity t&1 were last read by step t-1's stale
        # backwards, which precede this step's start
        S.wait(comm, start_ev)
        nb, nev = {}, {}
        for k in range(self.K, 1, -1):
            if t - self.K + k < 0:
                continue  # module k was still zero-padded: no boundary for k-1
            src, dst = self.owner[k - 1], self.owner[k - 2]
            if src == self.rank and dst == self.rank:
                nb[k - 1] = produced[k]
                nev[k - 1] = bwd_ev[k]
            elif src == self.rank:
                S.wait(comm, bwd_ev[k])
                with S.ctx(comm):
                    self.p2p.send(produced[k], dst, "boundary")
            elif dst == self.rank:
                m = self.mods[k - 1]
                buf = self._buf(("b", k - 1, t & 1), (B * T, self.d), self.grad_dtype, self._dev(m))
                with S.ctx(comm):
                    self.p2p.recv(buf, src, "boundary")
                nb[k - 1] = buf
                nev[k - 1] = S.record(comm)
        self.boundary = nb
        self._boundary_ev = nev

    def step(self, t, batch, optimizer=None, sync=True, shape=None):
        """One schedule step.  Ranks other than 0 pass batch.x = batch.y =
        None and give the (B, T) shape via `shape` (or `batch.shape`)."""
        if t < 0:
            raise ValueError("step index must be >= 0")
        S = self.streams
        x, y = batch.x, batch.y
        if self.owns(1):
            if not torch.is_tensor(x):
                import numpy as np

                x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64))
                y = torch.from_numpy(np.ascontiguousarray(y, dtype=np.int64))
            if S.gpu:
                if not x.is_cuda:  # host batches: range-checked, staged through pinned memory
                    V = getattr(self.tied, "vocab", None)
                    for a, what in ((x, "token"), (y, "target")):
                        if V is not None and a.numel() and (int(a.min()) < 0 or int(a.max()) >= V):
                            raise DimensionError(f"{what} id out of range [0, {V})")
                    x, y = x.pin_memory(), y.pin_memory()
                x = x.to(self.device, non_blocking=True)
                y = y.to(self.device, non_blocking=True)
            B, T = x.shape
        else:
            B, T = shape if shape is not None else batch.shape
        main = torch.cuda.current_stream(self.device) if S.gpu else None
        start_ev = S.record(main)
        for m in self.mods.values():
            m.snapshot(t)
        coef = tied_coefficients(t, self.K, self.tied_grad)
        overwrite = self.tied is not None and coef[0] != 0.0 and self.owns(self.K) and S.gpu
        if self.tied is not None and not overwrite:
            self.tied.grad.zero_()
        zero_ev = S.record(main)
        split = S.gpu and optimizer is not None and hasattr(optimizer, "apply_module")
        if split:
            optimizer.prepare([self.mods[k] for k in sorted(self.mods)])
        head_ev = [None]

        def gpu_hooks(k, s):
            if not S.gpu or not getattr(self.mods[k], "supports_hooks", True) or self.tied is None:
                return None
            if k == self.K:
                def after_head():
                    head_ev[0] = S.record(s)
                return {"after_head": after_head, "vo_overwrite": overwrite}
            if k == 1:
                def before_embedding():
                    if overwrite and head_ev[0] is not None:
                        s.wait_event(head_ev[0])
                return {"before_embedding": before_embedding, "vo_overwrite": overwrite}
            return None

        sids, produced, bwd_ev, opt_ev = {}, {}, {}, []
        # 1. stale backwards first (they need only last step's boundary)
        stale = [k for k in sorted(self.mods) if k < self.K]
        for k in stale:
            S.wait(self._bs[k], zero_ev)
        # module 1's tied scatter must follow module K's head backward when K
        # overwrites the tied gradient: issue module 1 after module K below
        early = [k for k in stale if not (k == 1 and self.owns(self.K) and overwrite)]
        for k in early:
            g_in, sids[k] = self._stale_backward(t, k, coef, B, T, gpu_hooks(k, self._bs[k]))
            produced[k] = g_in
            bwd_ev[k] = S.record(self._bs[k])
        # 2. relay
        loss, fwd_done = self._relay(t, x, y, batch.sample_id, B, T, start_ev)
        # 3. module K's fresh backward, then a deferred module 1
        late = ([self.K] if self.owns(self.K) else []) + [k for k in stale if k not in early]
        for k in late:
            if k == self.K:
                S.wait(self._bs[k], zero_ev)
                S.wait(self._bs[k], fwd_done[k])
            g_in, sids[k] = self._stale_backward(t, k, coef, B, T, gpu_hooks(k, self._bs[k]))
            produced[k] = g_in
            bwd_ev[k] = S.record(self._bs[k])
        # 4. optimizer updates on the modules' own streams, tied after both halves
        if split:
            for k in sorted(self.mods):
                with S.ctx(self._bs[k]):
                    optimizer.apply_module(t, self.mods[k])
                opt_ev.append(S.record(self._bs[k]))
            if self.tied is not None:
                for k in (1, self.K):
                    S.wait(self._ts, bwd_ev.get(k))
                with S.ctx(self._ts):
                    optimizer.apply_tied(t, self.tied, self._flag())
                opt_ev.append(S.record(self._ts))
        # 5. boundary exchange for step t+1
        self._exchange(t, produced, bwd_ev, B, T, start_ev)
        if S.gpu:
            for ev in list(fwd_done.values()) + list(bwd_ev.values()) + opt_ev:
                main.wait_event(ev)
            if self._boundary_ev:
                for ev in self._boundary_ev.values():
                    main.wait_event(ev)
        mods = [self.mods[k] for k in sorted(self.mods)]
        packet = GradientPacket(t, [m.grad_views for m in mods],
                                self.tied.grad if self.tied is not None else None,
                                [sids.get(k) for k in sorted(self.mods)], loss)
        if optimizer is not None and not split:
            optimizer.apply(t, packet, mods, self.tied.master if self.tied is not None else None)
        self.last_loss_device = loss
        if sync == "lagged" and S.gpu:
            # the host stays one step ahead: step t-1's loss / status words
            # are read (pinned D2H) after step t was issued
            from .engine import LaggedReader

            if getattr(self, "_lag", None) is None:
                self._lag = LaggedReader(self.device)
            rt = getattr(mods[0], "runtime", None)
            try:
                prev = self._lag.submit(t, loss, mods, rt.flag)
            except (NonFiniteError, DimensionError) as exc:
                raise WorkerFailure(f"distributed schedule aborted on rank {self.rank}: "
                                    f"{type(exc).__name__}: {exc}") from exc
            return packet, prev
        if sync and S.gpu:
            rt = getattr(mods[0], "runtime", None)
            if rt is not None:
                try:
                    rt.check(f"step {t}", mods)
                except (NonFiniteError, DimensionError) as exc:
                    raise WorkerFailure(f"distributed schedule aborted at step {t} on rank {self.rank}: "
                                        f"{type(exc).__name__}: {exc}") from exc
            if loss is not None:
                loss = float(loss.item())
                packet.loss = loss
        return packet, loss

    def flush_lagged(self):
        """sync="lagged": the last step's host loss on rank 0 (waits for it)."""
        lag = getattr(self, "_lag", None)
        if lag is None:
            return None
        try:
            return lag.flush()
        except (NonFiniteError, DimensionError) as exc:
            raise WorkerFailure(f"distributed schedule aborted on rank {self.rank}: "
                                f"{type(exc).__name__}: {exc}") from exc

    def _flag(self):
        m = next(iter(self.mods.values()))
        return m.runtime.flag

    def export_boundary(self):
        return dict(self.boundary)

    def import_boundary(self, grads):
        self.boundary = {k: torch.as_tensor(v).to(self._dev(self.mods[k]), self.grad_dtype).reshape(-1, self.d)
                         for k, v in grads.items()}
        self._boundary_ev = {}


def grad_out_device(m):
    return getattr(m, "device", torch.device("cpu"))


def build_local_modules(stack, part, dropout_seed, rank):
    """This rank's ModuleStates (GPU path)."""
    from .model import build_modules

    return {m.index: m for m in build_modules(stack, part, dropout_seed) if part.device_of[m.index - 1] == rank}
