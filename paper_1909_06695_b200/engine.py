"""The Ouroboros delayed-gradient schedule on B200s.

Drop-in for reference engine.py: `BatchSample`, `GradientPacket`,
`embedding_gradient`, `packet_grad_sq_norm`, `LogicalCostModel`,
`ScheduleTrace`, `PipelineEngine`, `ConcurrentPipelineEngine`,
`SequentialRunner`, `sequential_gradients`, `check_one_step_behind`,
`WorkerFailure`.

Step t (reference engine.py:246-259):
  1. every module's snapshot ring holds w^t (written by the previous step's
     fused optimizer, so this is free),
  2. batch t relays forward through modules 1..K at w^t; module K ends in the
     fused tied-vocab cross-entropy (no [N, V] logits in HBM),
  3. module k back-propagates sample t-K+k at w^{t-K+k} from its stored slot
     and the boundary gradient module k+1 produced at t-1 (zero while
     t-K+k < 0); the two tied halves are added onto a zeroed buffer (in
     either order: with two terms on zero, fp32 addition is order-free),
  4. the packet's tied gradient is 1/2 Vo(t) + 1/2 Vi(t-K+1) (engine.py:54-69),
  5. the optimizer applies the packet.

`PipelineEngine` issues everything on the current CUDA stream;
`ConcurrentPipelineEngine` gives every module its own forward and backward
streams ordered only by the true dependencies (events), so a module's stale
backward overlaps the relay (the GPU analogue of the reference's worker
threads, engine.py:271-406), and its packets are bitwise identical because
every kernel is deterministic.
"""

import json
from dataclasses import dataclass

import numpy as np
import torch

from .errors import DimensionError, NonFiniteError, ScheduleViolation, WorkerFailure  # noqa: F401
from .model import build_modules

# ---------------------------------------------------------------------------
# records


@dataclass
class BatchSample:
    x: object  # token ids [B, T] (numpy or torch)
    y: object  # next-token targets [B, T]
    sample_id: int


@dataclass
class GradientPacket:
    """module_grads: per module {"L{idx}.{name}": fp32 device view};
    emb_grad: the mixed tied gradient [V, d] (fp32, device).  Views are
    overwritten by the next step; use `.cpu()` to keep a copy."""

    step: int
    module_grads: list
    emb_grad: object
    sample_ids: list
    loss: float

    def cpu(self):
        return GradientPacket(
            self.step,
            [{k: v.detach().double().cpu().numpy() for k, v in g.items()} for g in self.module_grads],
            self.emb_grad.detach().double().cpu().numpy(),
            list(self.sample_ids),
            self.loss,
        )


def embedding_gradient(t, K, grad_vo_fresh, grad_vi_stale, convention="half_avg"):
    """Reference engine.py:54-69.  fp32 CUDA tensors go through
    `rp_embedding_gradient`; host arrays (the reference's own argument type)
    are combined on the host -- the engines never call this, they fuse the
    two halves into the head / embedding backward."""
    if convention not in ("half_avg", "sum"):
        raise ValueError(f"unknown tied_grad convention {convention!r}")
    if (torch.is_tensor(grad_vo_fresh) and grad_vo_fresh.is_cuda and grad_vo_fresh.dtype == torch.float32
            and (grad_vi_stale is None or (torch.is_tensor(grad_vi_stale) and grad_vi_stale.dtype == torch.float32))):
        from . import _native as N
        from . import ops

        if grad_vi_stale is not None and tuple(grad_vo_fresh.shape) != tuple(grad_vi_stale.shape):
            raise DimensionError("embedding gradient shape mismatch")
        vo = grad_vo_fresh.contiguous()
        vi = None if grad_vi_stale is None else grad_vi_stale.contiguous()
        out = torch.empty_like(vo)
        N.check(N.lib().rp_embedding_gradient(t, K, vo.data_ptr(), None if vi is None else vi.data_ptr(),
                                              out.data_ptr(), vo.numel(), 0 if convention == "half_avg" else 1,
                                              ops._stream()), "embedding_gradient")
        return out
    if t - K + 1 < 0:
        if grad_vi_stale is not None:
            raise ScheduleViolation("stale embedding gradient before step K-1")
        return grad_vo_fresh * 0
    if grad_vi_stale is None:
        raise ScheduleViolation("missing stale embedding gradient")
    if tuple(grad_vo_fresh.shape) != tuple(grad_vi_stale.shape):
        raise DimensionError("embedding gradient shape mismatch")
    if convention == "half_avg":
        return 0.5 * grad_vo_fresh + 0.5 * grad_vi_stale
    if convention == "sum":
        return grad_vo_fresh + grad_vi_stale
    raise ValueError(f"unknown tied_grad convention {convention!r}")


def tied_coefficients(t, K, convention):
    """(alpha_out, beta_in) of the fused tied gradient; (0, 0) = zero packet."""
    if convention not in ("half_avg", "sum"):
        raise ValueError(f"unknown tied_grad convention {convention!r}")
    if t - K + 1 < 0:
        return 0.0, 0.0
    return (0.5, 0.5) if convention == "half_avg" else (1.0, 1.0)


def packet_grad_sq_norm(packet):
    """Squared norm of the packet, accumulated in fp64 on the device in a
    fixed key order (engine.py:72-80)."""
    from . import ops

    dev = packet.emb_grad.device
    part = torch.empty(296, dtype=torch.float64, device=dev)
    out = torch.zeros((), dtype=torch.float64, device=dev)
    for grads in packet.module_grads:
        for key in sorted(grads):
            g = grads[key]
            ops.sq_norm(g.contiguous(), part, out, accumulate=True)
    ops.sq_norm(packet.emb_grad.contiguous(), part, out, accumulate=True)
    return float(out.item())


# ---------------------------------------------------------------------------
# logical clock + trace (engine.py:83-135), kept for API compatibility


@dataclass
class LogicalCostModel:
    fwd: list
    bwd: list
    relay: float = 0.05

    @classmethod
    def derived(cls, part, relay=0.05, recompute=True):
        sizes = [hi - lo for lo, hi in part.groups]
        factor = 3.0 if recompute else 2.0
        return cls([float(s) for s in sizes], [factor * s for s in sizes], relay)

    @classmethod
    def synthetic(cls, K, module_cost=1.0, relay=0.05):
        return cls([module_cost] * K, [module_cost] * K, relay)


class ScheduleTrace:
    """Occupancy rows {step, module, phase, sample, start, end}.  `engine.trace`
    carries the reference's logical clock (engine.py:104-135); with
    `timed=True` the engines also fill `engine.device_trace` from CUDA events
    recorded on each module's stream around its forward and delayed backward
    (milliseconds since the first timed step's start)."""

    def __init__(self):
        self.rows = []

    def record(self, step, module, phase, sample_id, start, end):
        self.rows.append({"step": step, "module": module, "phase": phase, "sample": sample_id,
                          "start": start, "end": end})

    def to_jsonl(self, path):
        with open(path, "w") as fh:
            for row in self.rows:
                fh.write(json.dumps(row) + "\n")

    def backward_rows(self):
        return [r for r in self.rows if r["phase"] == "backward"]

    def idle_backward_steps(self, module, from_step=0):
        return [r["step"] for r in self.rows if r["phase"] == "idle" and r["module"] == module
                and r["step"] >= from_step]


def check_one_step_behind(trace, K):
    for row in trace.backward_rows():
        if row["step"] != row["sample"] + K - row["module"]:
            raise ScheduleViolation(
                f"backward of module {row['module']} for sample {row['sample']} at step {row['step']}")
    return True


# ---------------------------------------------------------------------------
# executors


def _to_device_tokens(a, device, vocab=None, what="token"):
    """Host batches are range-checked before anything launches, so a bad id
    raises DimensionError before any update, like the reference's forward
    (layers.py:116-117, 299-305); device batches are checked by the kernels
    (RP_FLAG_DIMENSION, polled at step granularity)."""
    if torch.is_tensor(a) and a.is_cuda:
        return a.to(device=device, dtype=torch.int64, non_blocking=True)
    arr = np.ascontiguousarray(a.numpy() if torch.is_tensor(a) else np.asarray(a), dtype=np.int64)
    if vocab is not None and arr.size and (arr.min() < 0 or arr.max() >= vocab):
        raise DimensionError(f"{what} id out of range [0, {vocab})")
    return torch.from_numpy(arr).pin_memory().to(device, non_blocking=True)


class LaggedReader:
    """sync="lagged": queue the D2H copy of step t's loss and status words
    into pinned host memory (no host wait) and hand back the previous step's
    host loss after checking its status words -- the host stays one step
    ahead of the device and still reads every step's result."""

    def __init__(self, device):
        self.device = device
        self.bufs = None
        self.pending = None

    def submit(self, t, loss_dev, modules, runtime_flag):
        words = [m.flag for m in modules] + [runtime_flag]
        if self.bufs is None or self.bufs[0][1].numel() != len(words):
            pin = lambda n, dt: torch.zeros(n, dtype=dt).pin_memory()  # noqa: E731
            self.bufs = [(pin(1, torch.float32), pin(len(words), torch.int32)) for _ in range(2)]
        hl, hw = self.bufs[t % 2]
        main = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(main):
            if loss_dev is not None:
                hl.copy_(loss_dev.detach().reshape(1).float(), non_blocking=True)
            for i, w in enumerate(words):
                hw[i: i + 1].copy_(w.view(1), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(main)
        prev, self.pending = self.pending, (t, ev, hl if loss_dev is not None else None, hw, words, modules)
        return self._read(prev)

    def flush(self):
        entry, self.pending = self.pending, None
        return self._read(entry)

    @staticmethod
    def _read(entry):
        from . import _native as N

        if entry is None:
            return None
        t, ev, hl, hw, words, modules = entry
        ev.synchronize()
        bad = [(i, int(b)) for i, b in enumerate(hw.tolist()) if b]
        if bad:
            for w in words:
                w.zero_()
            i, bits = bad[0]
            where = f"module {modules[i].index}" if i < len(modules) else "optimizer update"
            if bits & N.FLAG_DIMENSION:
                raise DimensionError(f"token or target id out of range in {where} (step {t})")
            raise NonFiniteError(f"non-finite values in {where} (step {t})")
        return None if hl is None else float(hl.item())


class _DeviceClock:
    """CUDA-event timing of (step, module, phase) spans for ScheduleTrace:
    events are recorded on the stream the work runs on and resolved to
    milliseconds (relative to the first span's origin event) once they have
    completed, so timing never adds a host synchronisation to the step."""

    def __init__(self, device):
        self.device = device
        self.origin = None
        self.pending = []  # (step, module, phase, sample, start_ev, end_ev)

    def begin(self):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        if self.origin is None:
            self.origin = ev
        return ev

    def end(self, step, module, phase, sample, start_ev):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.pending.append((step, module, phase, sample, start_ev, ev))

    def flush(self, trace, wait=False):
        keep = []
        for row in self.pending:
            if not wait and not row[5].query():
                keep.append(row)
                continue
            row[5].synchronize()
            trace.record(row[0], row[1], row[2], row[3], self.origin.elapsed_time(row[4]),
                         self.origin.elapsed_time(row[5]))
        self.pending = keep


class PipelineEngine:
    """Deterministic single-stream executor of the delayed-gradient schedule."""

    def __init__(self, stack, part, dropout_seed, tied_grad="half_avg", stale_weights="snapshot", train=True,
                 cost_model=None, timed=False):
        if tied_grad not in ("half_avg", "sum"):
            raise ValueError(f"unknown tied_grad convention {tied_grad!r}")
        if stale_weights not in ("snapshot", "current"):
            raise ValueError(f"unknown stale_weights mode {stale_weights!r}")
        self.stack = stack
        self.part = part
        self.K = part.k
        self.modules = build_modules(stack, part, dropout_seed)
        self.tied_grad = tied_grad
        self.stale_weights = stale_weights
        self.train = train
        self.costs = cost_model or LogicalCostModel.derived(part)
        self.trace = ScheduleTrace()
        self.device_trace = ScheduleTrace()
        self._dclock = _DeviceClock(stack.runtime.device) if timed else None
        self.clock = 0.0
        self.last_step_logical = 0.0
        self.last_backward_logical = 0.0
        self.runtime = stack.runtime
        self.device = stack.runtime.device
        self.boundary = {}  # k -> fp32 [B*T, d] produced by module k+1 at the previous step
        self._bpool = {}
        self.last_loss_device = None

    # -- boundary buffers (ping-pong by step parity) --------------------------
    def _bbuf(self, k, parity, Nt, d):
        key = (k, parity)
        b = self._bpool.get(key)
        if b is None or b.shape != (Nt, d):
            b = torch.empty(Nt, d, dtype=torch.float32, device=self.device)
            self._bpool[key] = b
        return b

    # -- phases ---------------------------------------------------------------
    def _relay(self, t, x, y, sample_id):
        B, T = x.shape
        cur = x
        start = self.clock
        for m in self.modules:
            nxt = self.modules[m.index] if m.index < self.K else None
            out = nxt.input_buffer(t, B, T) if nxt is not None else None
            end = start + self.costs.fwd[m.index - 1]
            self.trace.record(t, m.index, "forward", sample_id, start, end)
            ev = self._dclock.begin() if self._dclock else None
            cur = m.forward(cur, t, sample_id, y if m.has_projection else None, self.train, out=out)
            if ev is not None:
                self._dclock.end(t, m.index, "forward", sample_id, ev)
            if m.index < self.K:
                cur = cur.view(B, T, -1)
            start = end + (self.costs.relay if m.index < self.K else 0.0)
        return cur, start

    def _backward_one(self, t, k, coef, B, T, after_head=None, before_embedding=None, vo_overwrite=False):
        m = self.modules[k - 1]
        s = t - self.K + k
        if s < 0:
            m.zero_grads()
            return None
        slot = m.pop_slot()
        if slot.step != s:
            raise ScheduleViolation(f"module {k} popped slot for step {slot.step}, expected {s}")
        grad_out = None
        if not m.has_projection:
            if k not in self.boundary:
                raise ScheduleViolation(f"module {k} missing boundary gradient")
            grad_out = self.boundary[k]
        g_in = self._bbuf(k - 1, t & 1, B * T, m.d) if k > 1 else None
        alpha, beta = coef
        emb = (alpha if m.has_projection else 0.0, beta if m.has_embedding else 0.0, self.stack.tied_store.grad)
        ev = self._dclock.begin() if self._dclock else None
        m.recompute_backward(slot, grad_out, self.stale_weights, self.train, g_in=g_in, emb=emb, live_step=t,
                             after_head=after_head, before_embedding=before_embedding, vo_overwrite=vo_overwrite)
        if ev is not None:
            self._dclock.end(t, k, "backward", slot.sample_id, ev)
        return g_in, slot.sample_id

    def _backward_all(self, t, B, T):
        coef = tied_coefficients(t, self.K, self.tied_grad)
        self.stack.tied_store.grad.zero_()  # both tied halves accumulate onto zero
        results = {}
        for k in range(self.K, 0, -1):
            results[k] = self._backward_one(t, k, coef, B, T)
        return results

    def _assemble(self, t, results, loss):
        nb = {}
        sids = []
        grads = []
        for k in range(1, self.K + 1):
            m = self.modules[k - 1]
            res = results[k]
            grads.append(m.grad_views)
            if res is None:
                sids.append(None)
                continue
            g_in, sid = res
            sids.append(sid)
            if k > 1:
                nb[k - 1] = g_in
        self.boundary = nb
        return GradientPacket(t, grads, self.stack.tied_store.grad, sids, loss)

    def _advance_clock(self, t, results, relay_end):
        longest = 0.0
        for k in range(1, self.K + 1):
            res = results[k]
            if res is None:
                self.trace.record(t, k, "idle", None, relay_end, relay_end)
                continue
            dur = self.costs.bwd[k - 1]
            self.trace.record(t, k, "backward", res[1], relay_end, relay_end + dur)
            longest = max(longest, dur)
        handoff = self.costs.relay if self.K > 1 else 0.0
        end = relay_end + longest + handoff
        self.last_step_logical = end - self.clock
        self.last_backward_logical = longest + handoff
        self.clock = end

    # -- lagged result read (sync="lagged") --------------------------------------
    def _lag_submit(self, t, loss_dev):
        if getattr(self, "_lag", None) is None:
            self._lag = LaggedReader(self.device)
        return self._lag.submit(t, loss_dev, self.modules, self.runtime.flag)

    def flush_lagged(self):
        """sync="lagged": the last step's host loss (waits for it)."""
        lag = getattr(self, "_lag", None)
        return None if lag is None else lag.flush()

    # -- public -----------------------------------------------------------------
    def step(self, t, batch, optimizer=None, sync=True):
        """One schedule step.  Returns (packet, loss); with sync=False the loss
        stays a 0-d device tensor and the status word is not polled; with
        sync="lagged" the step is issued without waiting and `loss` is the
        host loss of step t-1 (None for the first), read from pinned memory
        after its status words were checked -- the host stays one step ahead
        of the device (flush_lagged() returns the last step's loss)."""
        if t < 0:
            raise ValueError("step index must be >= 0")
        V = self.stack.tied_store.vocab
        x = _to_device_tokens(batch.x, self.device, V, "token")
        y = _to_device_tokens(batch.y, self.device, V, "target")
        B, T = x.shape
        for m in self.modules:
            m.snapshot(t)
        loss_dev, relay_end = self._relay(t, x, y, batch.sample_id)
        results = self._backward_all(t, B, T)
        packet = self._assemble(t, results, loss_dev)
        self._advance_clock(t, results, relay_end)
        if optimizer is not None:
            optimizer.apply(t, packet, self.modules, self.stack.tied)
        self.last_loss_device = loss_dev
        if self._dclock:
            self._dclock.flush(self.device_trace)
        if sync == "lagged":
            return packet, self._lag_submit(t, loss_dev)
        if sync:
            self.runtime.check(f"step {t}", self.modules)
            loss = float(loss_dev.item())
            packet.loss = loss
            return packet, loss
        return packet, loss_dev

    def flush_device_trace(self):
        """Resolve every recorded span (waits for the device)."""
        if self._dclock:
            self._dclock.flush(self.device_trace, wait=True)
        return self.device_trace

    def export_boundary(self):
        return dict(self.boundary)

    def import_boundary(self, grads):
        self.boundary = {k: torch.as_tensor(v).to(self.device, torch.float32).reshape(-1, self.modules[0].d)
                         for k, v in grads.items()}

    def close(self):
        pass


class ConcurrentPipelineEngine(PipelineEngine):
    """Same schedule with per-module CUDA streams.

    fwd(k,t) waits fwd(k-1,t); bwd(k,t) waits bwd(k+1,t-1) (its boundary) and,
    for k=K, fwd(K,t); module k's optimizer update follows its own backward;
    fwd(k,t+1) waits every update of step t.  Module K writes the tied
    gradient's output half and module 1's embedding scatter adds the input
    half after it (bitwise the reference executor's sum), so module K's
    backward -- the critical path -- never waits for module 1.
    """

    def __init__(self, *args, timeout=120.0, **kwargs):
        super().__init__(*args, **kwargs)
        if self.K < 2:
            raise ValueError("concurrent execution needs K >= 2")
        self._timeout = timeout
        # the relay and module K's backward form the step's critical path:
        # high-priority streams; stale backwards of modules k < K run beside
        # them on low-priority streams with a capped SM budget
        hi, lo = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, 0)
        self._fs = [torch.cuda.Stream(device=self.device, priority=-1) for _ in range(self.K)]
        self._bs = [torch.cuda.Stream(device=self.device, priority=(-1 if k == self.K else 0))
                    for k in range(1, self.K + 1)]
        import os

        self.side_ctas = int(os.environ.get("RP_SIDE_CTAS", "0"))
        self._bwd_done = {}
        # the tied matrix's optimizer update runs on its own stream as soon as
        # both gradient halves are in, beside module K's block backwards
        self._ts = torch.cuda.Stream(device=self.device, priority=0)
        self.split_optimizer = os.environ.get("RP_SPLIT_OPT", "1") != "0"

    def step(self, t, batch, optimizer=None, sync=True):
        if t < 0:
            raise ValueError("step index must be >= 0")
        main = torch.cuda.current_stream(self.device)
        V = self.stack.tied_store.vocab
        x = _to_device_tokens(batch.x, self.device, V, "token")
        y = _to_device_tokens(batch.y, self.device, V, "target")
        B, T = x.shape
        start_ev = torch.cuda.Event()
        start_ev.record(main)
        for m in self.modules:
            m.snapshot(t)
        # forward relay on per-module forward streams
        fwd_done = []
        cur = x
        prev = start_ev
        for m in self.modules:
            s = self._fs[m.index - 1]
            s.wait_event(prev)
            nxt = self.modules[m.index] if m.index < self.K else None
            with torch.cuda.stream(s):
                out = nxt.input_buffer(t, B, T) if nxt is not None else None
                tev = self._dclock.begin() if self._dclock else None
                cur = m.forward(cur, t, batch.sample_id, y if m.has_projection else None, self.train, out=out)
                if tev is not None:
                    self._dclock.end(t, m.index, "forward", batch.sample_id, tev)
                if m.index < self.K:
                    cur = cur.view(B, T, -1)
                ev = torch.cuda.Event()
                ev.record(s)
            fwd_done.append(ev)
            prev = ev
        loss_dev = cur
        # Stale backwards.  Modules k < K depend only on last step's boundary,
        # so they start with the step and overlap the relay; module K needs its
        # fresh forward.  Tied gradient: module K *writes* its output half
        # alpha*dV_out (dense, every row) and module 1 then *adds* beta*dV_in
        # (a scatter into the touched rows) -- fp32 a + b == b + a, so this is
        # bitwise the reference executor's 0 + a + b, needs no zero fill, and
        # module K never waits for module 1: only module 1's final embedding
        # scatter waits for module K's head backward.
        coef = tied_coefficients(t, self.K, self.tied_grad)
        tied_grad = self.stack.tied_store.grad
        overwrite = coef[0] != 0.0  # module K's head writes every row
        if not overwrite:
            tied_grad.zero_()  # warm-up: a zero packet
        zero_ev = torch.cuda.Event()
        zero_ev.record(main)
        results = {}
        bwd_done = {}
        split = self.split_optimizer and optimizer is not None and hasattr(optimizer, "apply_module")
        if split:
            optimizer.prepare(self.modules)
        opt_done = []
        head_ev = [None]
        tied_ready = [None]
        from . import layers as _LY

        def after_head(s):
            ev = torch.cuda.Event()
            ev.record(s)
            head_ev[0] = ev

        def before_embedding(s):
            if overwrite and head_ev[0] is not None:
                s.wait_event(head_ev[0])

        # issue module K first (its head event gates module 1's scatter)
        for k in [self.K] + list(range(self.K - 1, 0, -1)):
            m = self.modules[k - 1]
            s = self._bs[k - 1]
            s.wait_event(zero_ev)
            if k == self.K:
                s.wait_event(fwd_done[k - 1])
            if (k + 1) in self._bwd_done:
                s.wait_event(self._bwd_done[k + 1])
            _LY.CTA_BUDGET["value"] = self.side_ctas if k < self.K else 0
            try:
                with torch.cuda.stream(s):
                    results[k] = self._backward_one(
                        t, k, coef, B, T,
                        after_head=(lambda s=s: after_head(s)) if k == self.K else None,
                        before_embedding=(lambda s=s: before_embedding(s)) if k == 1 else None,
                        vo_overwrite=overwrite)
                    ev = torch.cuda.Event()  # gradients (and the boundary) of module k are in
                    ev.record(s)
                    if k == 1:
                        tied_ready[0] = ev  # both tied halves are in
                    if split:
                        optimizer.apply_module(t, self.modules[k - 1])
                        done = torch.cuda.Event()
                        done.record(s)
                        opt_done.append(done)
            finally:
                _LY.CTA_BUDGET["value"] = 0
            bwd_done[k] = ev
        tied_done = None
        if split:
            # the tied update runs beside whatever backward work is left
            self._ts.wait_event(tied_ready[0])
            if head_ev[0] is not None:
                self._ts.wait_event(head_ev[0])
            with torch.cuda.stream(self._ts):
                optimizer.apply_tied(t, self.stack.tied_store, self.runtime.flag)
                tied_done = torch.cuda.Event()
                tied_done.record(self._ts)
        self._bwd_done = bwd_done
        for ev in fwd_done + list(bwd_done.values()) + opt_done + ([tied_done] if tied_done is not None else []):
            main.wait_event(ev)
        packet = self._assemble(t, results, loss_dev)
        relay_end = self.clock + sum(self.costs.fwd) + self.costs.relay * (self.K - 1)
        self._advance_clock(t, results, relay_end)
        if optimizer is not None and not split:
            optimizer.apply(t, packet, self.modules, self.stack.tied)
        if self._dclock:
            self._dclock.flush(self.device_trace)
        # the next step's side streams order themselves after this step's
        # optimizer through start_ev / zero_ev (recorded on the main stream),
        # so no trailing fork is left open (CUDA-graph capture needs joins)
        self.last_loss_device = loss_dev
        if sync == "lagged":
            return packet, self._lag_submit(t, loss_dev)
        if sync:
            try:
                self.runtime.check(f"step {t}", self.modules)
            except (NonFiniteError, DimensionError) as exc:
                # the reference's threaded executor reports worker errors as
                # WorkerFailure with a per-module diagnostic (engine.py:300-311, 390-396)
                raise WorkerFailure(self._diagnostic(t, exc)) from exc
            loss = float(loss_dev.item())
            packet.loss = loss
            return packet, loss
        return packet, loss_dev

    def _diagnostic(self, t, exc):
        lines = [f"concurrent schedule aborted at step {t}", f"{type(exc).__name__}: {exc}"]
        for row in self.trace.rows[-3 * self.K:]:
            lines.append(str(row))
        return "\n".join(lines)

    def close(self):
        torch.cuda.synchronize(self.device)


class SequentialRunner(PipelineEngine):
    """Plain backprop over the whole stack (engine.py:443-491): the K=1
    baseline, keeping the caller's partition only for packet slicing."""

    def __init__(self, stack, part, dropout_seed, tied_grad="half_avg", train=True, cost_model=None, timed=False):
        from .model import partition

        super().__init__(stack, partition(stack.num_layers, 1), dropout_seed, tied_grad, "snapshot", train,
                         cost_model or LogicalCostModel.derived(part, recompute=False), timed=timed)
        self.user_part = part

    def step(self, t, batch, optimizer=None, sync=True):
        packet, loss = super().step(t, batch, optimizer, sync)
        grads = []
        allg = packet.module_grads[0]
        for lo, hi in self.user_part.groups:
            grads.append({k: v for k, v in allg.items() if lo <= int(k.split(".")[0][1:]) < hi})
        packet.module_grads = grads
        packet.sample_ids = [batch.sample_id] * self.user_part.k
        return packet, loss


def sequential_gradients(layers, params_list, batch, dropout_seed, step, train=True):
    """Reference engine.py:409-440: full-network backprop at explicit weights,
    the verification oracle.  `layers` is a stack's `.layers` list (or the
    stack), `params_list` one dict of arrays per layer -- the live
    `stack.params`, or a snapshot of them (numpy or torch, any dtype; the
    embedding and projection dicts carry "tied").  The weights are loaded
    into the stack's twin (`LayerStack.twin`), so the live weights are not
    touched.  Returns (grads keyed "L{idx}.{name}" as host fp64 arrays,
    grad_vi, grad_vo, loss, logits); `logits` [B, T, V] is an fp32 device
    tensor (the training path never materialises it; at V = 267,735 it is
    N * V * 4 bytes)."""
    from .model import stack_of

    stack = stack_of(layers)
    if len(params_list) != stack.num_layers:
        raise DimensionError(f"params_list has {len(params_list)} entries for {stack.num_layers} layers")
    if stack.layers[-1].kind != "projection":
        raise ValueError("stack must end with the output projection")
    twin = stack.twin()
    with torch.no_grad():
        for idx, params in enumerate(params_list):
            for name, arr in params.items():
                dst = twin.tied if name == "tied" else twin.params[idx][name]
                src = torch.as_tensor(np.asarray(arr) if not torch.is_tensor(arr) else arr)
                if tuple(src.shape) != tuple(dst.shape):
                    raise DimensionError(f"L{idx}.{name}: shape {tuple(src.shape)} != {tuple(dst.shape)}")
                dst.copy_(src)
    twin.refresh()
    mod = getattr(twin, "_seq_module", None)
    if mod is None:
        from .model import build_modules, partition

        (mod,) = build_modules(twin, partition(twin.num_layers, 1), dropout_seed)
        twin._seq_module = mod
    mod.dropout_seed = dropout_seed
    grads, gvi, gvo, loss = stack_gradients(twin, batch, dropout_seed, step, train, module=mod)
    # logits of the final hidden state (layers.py:268-273), on demand
    from . import ops

    h = mod._last_hidden
    B, T = h[1]
    logits = ops.gemm(h[0], twin.tied_store.compute, out_dtype=torch.float32).view(B, T, -1)
    return grads, gvi, gvo, loss, logits


def stack_gradients(stack, batch, dropout_seed, step, train=True, module=None):
    """Full backprop at the stack's current weights without touching them:
    returns (grads by key as host fp64 arrays, grad_vi, grad_vo, loss).
    `module`: a K=1 module of `stack` to reuse across calls -- it carries the
    Transformer-XL segment memory from one segment to the next."""
    from .model import build_modules, partition

    if module is None:
        (module,) = build_modules(stack, partition(stack.num_layers, 1), dropout_seed)
    m = module
    m.snapshot(step)
    V = stack.tied_store.vocab
    x = _to_device_tokens(batch.x, stack.runtime.device, V, "token")
    y = _to_device_tokens(batch.y, stack.runtime.device, V, "target")
    loss = m.forward(x, step, batch.sample_id, y, train)
    slot = m.pop_slot()
    m._last_hidden = (slot.arena.acts[-1], (slot.arena.B, slot.arena.T))
    _, grads, tied, _ = m.recompute_backward(slot, None, "snapshot", train)
    stack.runtime.check("sequential_gradients", [m])
    host = {k: v.double().cpu().numpy() for k, v in grads.items()}
    return host, tied["Vi"].double().cpu().numpy(), tied["Vo"].double().cpu().numpy(), float(loss.item())
