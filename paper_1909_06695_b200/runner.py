"""Training, verification and benchmark runs over a RunConfig (reference
runner.py), on the B200 engines.

* `train` steps the configured engine, streams the metrics CSV, writes the
  schedule trace and RPCK checkpoints (runner.py:233-305); `resume` restores
  the complete device state, so a halted run continues bit-exactly.
* `verify` replays a short run and re-derives every delayed gradient with
  this package's own K=1 backprop (`sequential_gradients`) at the recorded
  weight snapshots (runner.py:424-534).  Both sides run the same
  deterministic kernels on the same inputs, so the expected deviation is
  exactly zero, as in the reference.  The CPU fp64 oracle in `oracle/` is
  the test suite's checker, not this function's.
* `bench` reports the logical-clock speed-up table across K
  (runner.py:564-620) and, beside it, the measured device time per step.

Checkpoint names follow the reference (runner.py:111-226): `stack.*`
masters, `optim.adam.{m,v}.*` moments, `m{k}.ring.{s}.L{i}.{name}` snapshot
entries, `m{k}.slot{j}.{inputs,targets,meta,seeds}` pending slots and
`boundary.{k}` gradients; the sidecar holds next_step, the logical clock
and the config.  Ring entries hold this package's compute copies (bf16 in
production) -- the weights the stale backward actually reads.  The tied
matrix is not snapshotted (no stale pass reads V: the embedding backward is
a scatter, the head runs at the live weights), so ring entries for `tied`
are neither written nor required.  A reference checkpoint loads too: its
fp64 arrays are rounded to fp32 masters / compute copies, and pending slots
are rebuilt by re-running their forward from the saved inputs at the
snapshot weights and seeds.
"""

import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import checkpoint as ckpt
from .config import RunConfig
from .data import BatchSource, SegmentStream, load_corpus
from .engine import (
    ConcurrentPipelineEngine,
    LogicalCostModel,
    PipelineEngine,
    SequentialRunner,
    WorkerFailure,
    packet_grad_sq_norm,
    sequential_gradients,
    stack_gradients,
)
from .errors import DimensionError, NonFiniteError
from .metrics import MetricsRow, MetricsWriter
from .model import StaleSlot, build_modules, build_stack, build_xl_stack, measure_layer_costs, partition
from .optim import make_optimizer
from .rng import SeededRng, mix64

# verify: pipeline gradients vs this package's K=1 backprop at the same
# snapshots, same kernels -> exact (reference ORACLE_TOLERANCE, runner.py:42)
ORACLE_TOLERANCE = 0.0
# verify's finite-difference spot check runs in the fp32 check mode
FD_H_REL = 1e-3
FD_TOLERANCE = 2e-3

# config fields a resumed run must share with its checkpoint (runner.py:45-51)
STRUCTURAL_FIELDS = (
    "data", "vocab_mode", "seq_len", "batch_size", "n_blocks", "model_dim",
    "ffn_dim", "dropout_p", "k", "mode", "tied_grad", "stale_weights",
    "balance", "optimizer", "lr", "lr_mode", "warmup_steps", "steps",
    "adam_beta1", "adam_beta2", "adam_eps", "seed_init", "seed_data",
    "seed_dropout", "n_heads", "mem_len", "adaptive_cutoffs", "activation",
)


@dataclass
class Runtime:
    cfg: RunConfig
    source: BatchSource
    stack: object
    part: object
    engine: object
    optimizer: object
    vocab_size: int


def _make_engine(cfg, stack, part, cost_model):
    common = dict(dropout_seed=cfg.seed_dropout, tied_grad=cfg.tied_grad, cost_model=cost_model,
                  timed=bool(getattr(cfg, "timed_trace", False)))
    if cfg.mode == "sequential":
        return SequentialRunner(stack, part, **common)
    if cfg.mode == "ouroboros-ref":
        return PipelineEngine(stack, part, stale_weights=cfg.stale_weights, **common)
    if cfg.mode == "ouroboros-concurrent":
        return ConcurrentPipelineEngine(stack, part, stale_weights=cfg.stale_weights, **common)
    raise ValueError(f"unknown mode {cfg.mode!r}")


def build_runtime(cfg, synthetic_cost=None, device=None):
    tokens, vocab = load_corpus(cfg.data, cfg.vocab_mode)
    if cfg.n_heads:
        # XL: contiguous segment streams so each row's memory precedes it
        source = SegmentStream(tokens, cfg.seq_len, cfg.batch_size)
        stack = build_xl_stack(vocab, cfg.model_dim, cfg.ffn_dim, cfg.n_blocks, cfg.seq_len, cfg.dropout_p,
                               cfg.seed_init, cfg.n_heads, cfg.mem_len, dtype=cfg.dtype, device=device,
                               cutoffs=cfg.cutoffs, activation=cfg.activation)
    else:
        source = BatchSource(tokens, cfg.seq_len, cfg.batch_size, cfg.seed_data)
        stack = build_stack(vocab, cfg.model_dim, cfg.ffn_dim, cfg.n_blocks, cfg.seq_len, cfg.dropout_p,
                            cfg.seed_init, dtype=cfg.dtype, device=device, activation=cfg.activation)
    costs = None
    if cfg.balance == "by_cost":
        costs = measure_layer_costs(stack, source.batch_at(0).x, cfg.seed_dropout)
    k = 1 if cfg.mode == "sequential" else cfg.k
    part = partition(stack.num_layers, k, cfg.balance, costs)
    if synthetic_cost is not None:
        cost_model = LogicalCostModel.synthetic(k, synthetic_cost, cfg.relay_cost)
    else:
        cost_model = LogicalCostModel.derived(part, cfg.relay_cost, recompute=cfg.mode != "sequential")
    engine = _make_engine(cfg, stack, part, cost_model)
    optimizer = make_optimizer(cfg.optimizer, cfg.lr_schedule(), cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps)
    if hasattr(optimizer, "bind"):
        optimizer.bind(engine.modules)
    return Runtime(cfg, source, stack, part, engine, optimizer, vocab)


# ---------------------------------------------------------------------------
# checkpoint state


def _layer_entries(stack):
    """(checkpoint name, live fp32 view) of every master parameter."""
    yield "stack.tied", stack.tied
    for idx, params in enumerate(stack.params):
        for name, view in params.items():
            if name != "tied":
                yield f"stack.L{idx}.{name}", view


def _ring_entries(module, step):
    """(name, compute-copy view) of module's snapshot of `step`."""
    start = module.layer_range[0]
    for off, st in enumerate(module.storage):
        i = st.ring_slot(step)
        if st.ring_step[i] != step:
            continue
        for name, view in st._public(st.ring[i][2]).items():
            yield f"m{module.index}.ring.{step}.L{start + off}.{name}", view


def _ring_steps(module):
    steps = set()
    for st in module.storage:
        steps.update(s for s in st.ring_step if s is not None)
    return sorted(steps)


def collect_state(runtime, next_step):
    """Named arrays + sidecar of the complete training state."""
    torch.cuda.synchronize(runtime.stack.runtime.device)
    arrays = dict(_layer_entries(runtime.stack))
    for key, arr in runtime.optimizer.state_arrays().items():
        arrays[f"optim.{key}"] = arr
    engine = runtime.engine
    d = runtime.stack.tied_store.d
    for m in engine.modules:
        for s in _ring_steps(m):
            arrays.update(_ring_entries(m, s))
        for j, slot in enumerate(m.slots):
            a = slot.arena
            pre = f"m{m.index}.slot{j}."
            arrays[pre + "inputs"] = a.tokens if m.has_embedding else a.acts[0].view(a.B, a.T, d)
            if m.has_embedding and a.acts:
                # the embedding output depends on V at the slot's step, which
                # the ring does not keep (an extra entry; the reference
                # loader ignores it)
                arrays[pre + "embedded"] = a.acts[0].view(a.B, a.T, d)
            if m.has_projection:
                arrays[pre + "targets"] = a.targets.view(a.B, a.T)
            for j2, off in enumerate(m.block_idx):
                tp = a.tapes[j2]
                if m.layers[off].kind == "xl_block" and tp.M:
                    arrays[pre + f"mem.L{m.layer_range[0] + off}"] = tp.mem.view(a.B, tp.M, d)
                    arrays[pre + "mem_len"] = np.array([tp.mem_len], dtype=np.int64)
            arrays[pre + "meta"] = np.array([slot.step, slot.sample_id], dtype=np.int64)
            arrays[pre + "seeds"] = np.array(slot.layer_seeds, dtype=np.uint64)
    for m in engine.modules:
        for off, buf in m.mem.items():
            arrays[f"m{m.index}.mem.L{m.layer_range[0] + off}"] = buf
        if m.mem:
            arrays[f"m{m.index}.mem_len"] = np.array([m.mem_len], dtype=np.int64)
    B, T = runtime.cfg.batch_size, runtime.cfg.seq_len
    for k, g in engine.export_boundary().items():
        arrays[f"boundary.{k}"] = g.view(B, T, d) if g.numel() == B * T * d else g
    sidecar = {"format": ckpt.VERSION, "next_step": int(next_step), "clock": float(engine.clock),
               "config": runtime.cfg.to_dict(), "dtype": runtime.cfg.dtype}
    return arrays, sidecar


def save_training_state(path, runtime, next_step):
    arrays, sidecar = collect_state(runtime, next_step)
    ckpt.save_arrays(path, arrays)
    ckpt.save_sidecar(path, sidecar)


def _put(dst, src, name):
    src = torch.as_tensor(np.asarray(src))
    if src.numel() != dst.numel():
        raise ckpt.CheckpointError(f"checkpoint entry {name!r} has {src.numel()} elements, expected {dst.numel()}")
    dst.copy_(src.reshape(dst.shape))


def load_training_state(path, runtime):
    """Restore weights, moments, rings, pending slots (their tapes are
    re-derived on the device) and boundary gradients in place; returns the
    next step index (reference runner.py:156-226)."""
    arrays = ckpt.load_arrays(path)
    sidecar = ckpt.load_sidecar(path)
    saved = sidecar.get("config", {})
    for name in STRUCTURAL_FIELDS:
        # fields the reference lacks (n_heads, mem_len) default like ours
        ours, theirs = getattr(runtime.cfg, name), saved.get(name, getattr(RunConfig(), name))
        if ours != theirs:
            raise ckpt.CheckpointError(f"checkpoint config mismatch on {name!r}: {theirs!r} != {ours!r}")
    return restore_state(runtime.stack, runtime.engine, runtime.optimizer, arrays, int(sidecar["next_step"]),
                         float(sidecar["clock"]))


def restore_state(stack, engine, optimizer, arrays, next_step, clock=0.0):
    """The in-memory half of `load_training_state`: named arrays (our or the
    reference's checkpoint entry names) -> weights, moments, rings, pending
    slots (re-derived on the device) and boundary gradients.  Also the entry
    point of the teacher-forced parity test, which feeds it the fp64 oracle's
    state every step.  `arrays` is consumed."""
    arrays = dict(arrays)
    with torch.no_grad():
        for name, view in _layer_entries(stack):
            if name not in arrays:
                raise ckpt.CheckpointError(f"checkpoint lacks {name!r}")
            _put(view, arrays.pop(name), name)
        stack.refresh()  # compute copies of V; ring entries are reloaded below
        optim = {n[len("optim."):]: arrays.pop(n) for n in list(arrays) if n.startswith("optim.")}
        optimizer.load_state_arrays(optim)
        d = stack.tied_store.d
        # the rings hold exactly the snapshots the state names: forget every
        # other entry (a later step's entry would shadow the restored masters)
        for m in engine.modules:
            for st in m.storage:
                st.ring_step = [None] * len(st.ring_step)
        ref_tied = {}
        for m in engine.modules:
            pre = f"m{m.index}."
            ring_steps = sorted({int(n.split(".")[2]) for n in arrays if n.startswith(pre + "ring.")})
            start = m.layer_range[0]
            for s in ring_steps:
                for off, st in enumerate(m.storage):
                    _, _, carved = st.ring[st.ring_slot(s)]
                    views = st._public(carved)
                    for name, view in views.items():
                        key = f"{pre}ring.{s}.L{start + off}.{name}"
                        if key in arrays:
                            _put(view, arrays.pop(key), key)
                        elif name != "tied":
                            raise ckpt.CheckpointError(f"checkpoint lacks {key!r}")
                    st.ring_step[st.ring_slot(s)] = s
                for n in [n for n in arrays if n.startswith(f"{pre}ring.{s}.")]:
                    if n.endswith(".tied"):  # the reference snapshots V too
                        ref_tied.setdefault(m.index, {})[s] = arrays.pop(n)
            m.slots.clear()
            j = 0
            while f"{pre}slot{j}.meta" in arrays:
                step, sample_id = (int(v) for v in arrays.pop(f"{pre}slot{j}.meta"))
                seeds = [int(v) for v in arrays.pop(f"{pre}slot{j}.seeds")]
                inputs = arrays.pop(f"{pre}slot{j}.inputs")
                targets = arrays.pop(f"{pre}slot{j}.targets", None)
                embedded = arrays.pop(f"{pre}slot{j}.embedded", None)
                B, T = inputs.shape[:2]
                arena = m._arena(step, B, T)
                if m.has_embedding:
                    _put(arena.tokens, inputs, "inputs")
                else:
                    _put(arena.acts[0], inputs.reshape(B * T, d), "inputs")
                if m.has_projection:
                    _put(arena.targets, targets, "targets")
                slot_mem_len = arrays.pop(f"{pre}slot{j}.mem_len", None)
                for j2, off in enumerate(m.block_idx):
                    tp = arena.tapes[j2]
                    key = f"{pre}slot{j}.mem.L{m.layer_range[0] + off}"
                    if m.layers[off].kind == "xl_block" and tp.M:
                        if key not in arrays:
                            raise ckpt.CheckpointError(f"checkpoint lacks {key!r}")
                        _put(tp.mem, arrays.pop(key), key)
                        tp.mem_len = int(slot_mem_len[0])
                slot = StaleSlot(step, sample_id, arena.tokens if m.has_embedding else arena.acts[0], targets,
                                 seeds, arena)
                m.slots.append(slot)
                # the stored intermediates are a pure function of (input,
                # snapshot weights, seeds): re-derive them.  The embedding
                # needs V at the slot's step: our checkpoints carry the
                # embedding output, the reference's carry V in its ring.
                kw = {}
                if m.has_embedding and arena.acts:
                    if embedded is not None:
                        _put(arena.acts[0], embedded.reshape(B * T, d), "embedded")
                        kw["from_act0"] = True
                    elif step in ref_tied.get(m.index, {}):
                        kw["tied_c"] = torch.as_tensor(ref_tied[m.index][step]).to(stack.runtime.device,
                                                                                    stack.cdtype)
                    else:
                        raise ckpt.CheckpointError(f"slot {j} of module {m.index} lacks V for step {step}")
                m._run_forward(step, arena, seeds, engine.train, None, m.ws_fwd, live=False, **kw)
                j += 1
            m.last_forward_step = next_step - 1
            for off in m.block_idx:
                key = f"{pre}mem.L{m.layer_range[0] + off}"
                if key in arrays:
                    src = arrays.pop(key)
                    m.mem[off] = torch.empty(src.size // d, d, dtype=stack.cdtype,
                                             device=stack.runtime.device)
                    _put(m.mem[off], src, key)
            if f"{pre}mem_len" in arrays:
                m.mem_len = int(arrays.pop(f"{pre}mem_len")[0])
        engine.import_boundary({int(n.split(".")[1]): arrays.pop(n) for n in list(arrays)
                                if n.startswith("boundary.")})
        engine.clock = clock
    torch.cuda.synchronize(stack.runtime.device)
    stack.runtime.check("load_training_state", engine.modules)
    return next_step


# ---------------------------------------------------------------------------
# train


def train(cfg, progress=None):
    """Run the configured training; returns a summary dict.  Stops with
    `diverged` set at the first non-finite loss or gradient; writes
    metrics.csv, trace.jsonl and checkpoint.bin under cfg.out_dir."""
    cfg.validate()
    runtime = build_runtime(cfg)
    os.makedirs(cfg.out_dir, exist_ok=True)
    paths = {n: os.path.join(cfg.out_dir, f) for n, f in
             (("metrics", "metrics.csv"), ("trace", "trace.jsonl"), ("checkpoint", "checkpoint.bin"))}
    start_step = load_training_state(cfg.resume, runtime) if cfg.resume else 0
    engine, optimizer = runtime.engine, runtime.optimizer
    end_step = min(cfg.steps, cfg.halt_at) if cfg.halt_at else cfg.steps
    diverged_at, last_loss, steps_run = None, math.nan, 0
    writer = MetricsWriter(paths["metrics"])
    try:
        for t in range(start_step, end_step):
            t0 = time.perf_counter()
            if getattr(runtime.source, "wraps_at", None) and runtime.source.wraps_at(t):
                for m in engine.modules:
                    m.reset_memory()  # the segment streams restart
            try:
                packet, loss = engine.step(t, runtime.source.batch_at(t), optimizer)
            except (NonFiniteError, WorkerFailure, DimensionError):
                diverged_at = t
                break
            if not math.isfinite(loss):
                diverged_at = t
                break
            wall_ms = (time.perf_counter() - t0) * 1e3
            writer.write(MetricsRow(t, wall_ms, engine.last_step_logical, loss, packet_grad_sq_norm(packet),
                                    optimizer.schedule.at(t)))
            last_loss, steps_run = loss, steps_run + 1
            if progress is not None:
                progress(t, loss)
            if cfg.checkpoint_every and (t + 1) % cfg.checkpoint_every == 0:
                save_training_state(paths["checkpoint"], runtime, t + 1)
        if diverged_at is None:
            save_training_state(paths["checkpoint"], runtime, end_step)
    finally:
        writer.close()
        engine.trace.to_jsonl(paths["trace"])
        if getattr(cfg, "timed_trace", False):
            engine.flush_device_trace().to_jsonl(os.path.join(cfg.out_dir, "trace_device.jsonl"))
        engine.close()
    return {
        "mode": cfg.mode, "k": runtime.part.k, "steps_run": steps_run, "start_step": start_step,
        "final_loss": last_loss, "diverged": diverged_at is not None, "diverged_at": diverged_at,
        "metrics_path": paths["metrics"], "trace_path": paths["trace"], "checkpoint_path": paths["checkpoint"],
    }


# ---------------------------------------------------------------------------
# verify


def _masters(stack):
    return [st.master.clone() for st in stack.storage], stack.tied.clone()


def _load_masters(stack, snap):
    layers, tied = snap
    for st, src in zip(stack.storage, layers):
        st.master.copy_(src)
    stack.tied.copy_(tied)
    stack.refresh()


def _twin_stack(cfg, vocab, dtype=None):
    if cfg.n_heads:
        return build_xl_stack(vocab, cfg.model_dim, cfg.ffn_dim, cfg.n_blocks, cfg.seq_len, cfg.dropout_p,
                              cfg.seed_init, cfg.n_heads, cfg.mem_len, dtype=dtype or cfg.dtype, cutoffs=cfg.cutoffs,
                              activation=cfg.activation)
    return build_stack(vocab, cfg.model_dim, cfg.ffn_dim, cfg.n_blocks, cfg.seq_len, cfg.dropout_p, cfg.seed_init,
                       dtype=dtype or cfg.dtype, activation=cfg.activation)


def _sequential_loss(stack, x, y, dropout_seed, step):
    (m,) = build_modules(stack, partition(stack.num_layers, 1), dropout_seed)
    m.snapshot(step)
    loss = m.forward(x, step, 0, y, True)
    return float(loss.item())


def finite_difference_check(seed=123, coords_per_param=3, h_rel=FD_H_REL):
    """Central differences of the fp32 device loss against the analytic
    gradient of `sequential_gradients` on a tiny stack (reference
    runner.py:312-354 on its 7-token / dim-6 stack; dims here are multiples
    of 8 for the TMA row pitch).  Returns the worst relative deviation."""
    from .engine import BatchSample

    stack = build_stack(7, 8, 8, 2, 4, 0.0, seed, dtype="fp32")
    rng = SeededRng(mix64(seed, 1))
    x = (rng.uniform((2, 4)) * 7).astype(np.int64)
    y = (rng.uniform((2, 4)) * 7).astype(np.int64)
    grads, g_vi, g_vo, _ = stack_gradients(stack, BatchSample(x, y, 0), 5, 0)
    dev = stack.runtime.device
    xd, yd = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    checks = [("tied", stack.tied, g_vi + g_vo)]
    for idx, params in enumerate(stack.params):
        checks += [(f"L{idx}.{n}", v, grads[f"L{idx}.{n}"]) for n, v in params.items() if n != "tied"]
    picker = SeededRng(mix64(seed, 2))
    worst = 0.0
    for _, view, analytic in checks:
        host = view.detach().cpu().numpy()
        for _ in range(coords_per_param):
            flat = int(picker.uniform(()) * host.size)
            idx = np.unravel_index(flat, host.shape)
            old = float(host[idx])
            h = h_rel * max(1.0, abs(old))
            losses = []
            for sign in (1.0, -1.0):
                view[idx] = old + sign * h
                stack.refresh()
                losses.append(_sequential_loss(stack, xd, yd, 5, 0))
            view[idx] = old
            stack.refresh()
            fd = (losses[0] - losses[1]) / (2 * h)
            a = float(analytic[idx])
            worst = max(worst, abs(a - fd) / max(abs(a), abs(fd), 1.0))
    return worst


def dropout_replay_check(n_pairs=10, seed=77, dtype="fp32"):
    """Store-all vs recompute agreement over random stacks and steps
    (reference runner.py:357-391): the backward from the slot's stored
    intermediates must equal, bitwise, a backward that re-runs the forward
    from the slot's input with the same seeds."""
    picker = SeededRng(seed)
    mismatches = 0
    for pair in range(n_pairs):
        blocks = 1 + int(picker.uniform(()) * 3)
        stack = build_stack(7, 8, 8, blocks, 4, 0.2, mix64(seed, pair), dtype=dtype)
        (m,) = build_modules(stack, partition(stack.num_layers, 1), mix64(seed, pair, 1))
        step = int(picker.uniform(()) * 50)
        x = torch.from_numpy((picker.uniform((2, 4)) * 7).astype(np.int64)).to(stack.runtime.device)
        y = torch.from_numpy((picker.uniform((2, 4)) * 7).astype(np.int64)).to(stack.runtime.device)
        m.snapshot(step)
        m.forward(x, step, step, y, True)
        slot = m.slots[0]
        results = []
        for mode in ("snapshot", "current"):
            m.zero_grads()
            _, grads, tied, _ = m.recompute_backward(slot, None, mode, True, live_step=step)
            results.append(({k: v.clone() for k, v in grads.items()}, tied["Vi"].clone(), tied["Vo"].clone()))
        (ga, via, voa), (gb, vib, vob) = results
        mismatches += sum(not torch.equal(ga[k], gb[k]) for k in ga)
        mismatches += (not torch.equal(via, vib)) + (not torch.equal(voa, vob))
    return mismatches


def _k1_bitwise_check(cfg, steps=20):
    """The pipeline engine at K=1 against the sequential runner, bitwise
    (reference runner.py:394-421)."""
    tokens, vocab = load_corpus(cfg.data, cfg.vocab_mode)
    source = (SegmentStream(tokens, cfg.seq_len, cfg.batch_size) if cfg.n_heads
              else BatchSource(tokens, cfg.seq_len, cfg.batch_size, cfg.seed_data))
    runs = []
    for sequential in (False, True):
        stack = _twin_stack(cfg, vocab)
        part = partition(stack.num_layers, 1)
        eng = (SequentialRunner if sequential else PipelineEngine)(stack, part, cfg.seed_dropout, cfg.tied_grad)
        opt = make_optimizer(cfg.optimizer, cfg.lr_schedule(), cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps)
        runs.append((stack, eng, opt))
    for t in range(steps):
        batch = source.batch_at(t)
        losses = [eng.step(t, batch, opt)[1] for _, eng, opt in runs]
        if losses[0] != losses[1]:
            return False
    return bool(torch.equal(runs[0][0].tied, runs[1][0].tied))


def _ring_matches_snapshots(engine, snapshots, stack):
    """Every ring entry equals the compute copy of the recorded master."""
    from . import ops

    for m in engine.modules:
        for off, st in enumerate(m.storage):
            layer = m.layer_range[0] + off
            for i, s in enumerate(st.ring_step):
                if s is None:
                    continue
                if s >= len(snapshots):
                    return False
                rec = snapshots[s][0][layer]
                vec, mat, _ = st.ring[i]
                if not torch.equal(vec, rec[: st.n_vec]):
                    return False
                if st.n_mat:
                    want = torch.empty_like(mat)
                    ops.cast(rec[st.n_vec:], want)
                    if not torch.equal(mat, want):
                        return False
    return True


def verify(cfg, steps=50):
    """Replay `steps` steps, then check every delayed gradient and the mixed
    tied gradient against K=1 backprop at the recorded snapshots, plus the
    zero-padding, tie-identity, snapshot-fidelity, finite-difference,
    dropout-replay and K=1-collapse checks (reference runner.py:424-534)."""
    if steps > 200:
        raise ValueError("verify is capped at 200 steps (oracle cost)")
    cfg.validate()
    if cfg.mode == "sequential":
        raise ValueError("verify targets the pipeline modes; set mode=ouroboros-ref")
    runtime = build_runtime(cfg)
    engine, stack, K = runtime.engine, runtime.stack, runtime.part.k
    packets, batches, snapshots = [], [], []
    tie_ok = True
    emb_tied = engine.modules[0].params[0]["tied"]
    proj_tied = engine.modules[-1].params[-1]["tied"]
    try:
        for t in range(steps):
            batch = runtime.source.batch_at(t)
            snapshots.append(_masters(stack))
            batches.append(batch)
            packet, _ = engine.step(t, batch, runtime.optimizer)
            packets.append(([{k: v.clone() for k, v in g.items()} for g in packet.module_grads],
                            packet.emb_grad.clone()))
            tie_ok &= emb_tied is proj_tied and emb_tied.data_ptr() == stack.tied_store.master.data_ptr()
        # the fused optimizer already wrote w^{steps} into the rings
        ring_ok = _ring_matches_snapshots(engine, snapshots + [_masters(stack)], stack)
    finally:
        engine.close()

    twin = _twin_stack(cfg, runtime.vocab_size)
    cache = {}
    twin_module = None
    if cfg.n_heads:
        # XL: the memory of segment s is the layer input of segment s-1 at
        # w^{s-1}; a persistent K=1 twin replayed in step order carries it
        (twin_module,) = build_modules(twin, partition(twin.num_layers, 1), cfg.seed_dropout)

    def oracle(s):
        if s not in cache:
            _load_masters(twin, snapshots[s])
            cache[s] = stack_gradients(twin, batches[s], cfg.seed_dropout, s, module=twin_module)
        return cache[s]

    if twin_module is not None:
        for s in range(steps):
            oracle(s)

    deviations, emb_deviations = [], []
    zero_pad_ok = True
    for t, (module_grads, emb) in enumerate(packets):
        for k in range(1, K + 1):
            s = t - K + k
            got = module_grads[k - 1]
            if s < 0:
                zero_pad_ok &= not any(bool(g.any()) for g in got.values())
                continue
            want = oracle(s)[0]
            lo, hi = runtime.part.groups[k - 1]
            worst = 0.0
            for key, arr in want.items():
                if lo <= int(key.split(".")[0][1:]) < hi:
                    worst = max(worst, float(np.abs(got[key].double().cpu().numpy() - arr).max()))
            deviations.append((t, k, worst))
        if t - K + 1 < 0:
            zero_pad_ok &= not bool(emb.any())
            continue
        vo = torch.from_numpy(oracle(t)[2]).float()
        vi = torch.from_numpy(oracle(t - K + 1)[1]).float()
        expect = 0.5 * vo + 0.5 * vi if cfg.tied_grad == "half_avg" else vo + vi
        emb_deviations.append((t, float((emb.cpu() - expect).abs().max())))

    oracle_max = max([d for *_, d in deviations] + [d for _, d in emb_deviations] + [0.0])
    fd_worst = finite_difference_check()
    replay_mismatches = dropout_replay_check(n_pairs=10)
    k1_ok = _k1_bitwise_check(cfg)
    oracle_ok = oracle_max <= ORACLE_TOLERANCE
    informational = cfg.stale_weights == "current"
    worst_by_module = {k: 0.0 for k in range(1, K + 1)}
    for _, k, d in deviations:
        worst_by_module[k] = max(worst_by_module[k], d)
    passed = ((oracle_ok or informational) and zero_pad_ok and tie_ok and ring_ok and fd_worst < FD_TOLERANCE
              and replay_mismatches == 0 and k1_ok)
    return {
        "mode": cfg.mode, "k": K, "steps": steps, "stale_weights": cfg.stale_weights, "dtype": cfg.dtype,
        "oracle_max_abs": oracle_max, "oracle_tolerance": ORACLE_TOLERANCE, "oracle_ok": oracle_ok,
        "oracle_informational": informational, "worst_by_module": worst_by_module,
        "emb_max_abs": max([d for _, d in emb_deviations] + [0.0]), "zero_padding_ok": bool(zero_pad_ok),
        "tie_ok": bool(tie_ok), "snapshot_fidelity_ok": ring_ok, "finite_difference_worst": fd_worst,
        "finite_difference_ok": fd_worst < FD_TOLERANCE, "dropout_replay_mismatches": replay_mismatches,
        "k1_bitwise_ok": k1_ok, "passed": bool(passed),
    }


# ---------------------------------------------------------------------------
# bench


def bench(cfg, k_values, steps=30, module_cost=1.0):
    """Per K: logical-clock speed-up over sequential backprop with equal
    synthetic module costs and per-module backward utilisation (reference
    runner.py:564-620), plus the measured device milliseconds per step and
    tokens/s of the B200 engine."""
    cfg.validate()
    rows = []
    for k in k_values:
        if k > cfg.n_layers:
            raise ValueError(f"K={k} exceeds layer count {cfg.n_layers}")
        run_cfg = RunConfig(**{**cfg.to_dict(), "k": k, "steps": steps})
        run_cfg.mode = "ouroboros-concurrent" if k >= 2 else "ouroboros-ref"
        run_cfg.lr_mode = "fixed"
        runtime = build_runtime(run_cfg, synthetic_cost=module_cost)
        engine = runtime.engine
        logical, backward_logical = [], []
        warm = min(k, steps - 1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        wall0 = time.perf_counter()
        try:
            for t in range(steps):
                if t == warm:
                    ev0.record()
                engine.step(t, runtime.source.batch_at(t), runtime.optimizer)
                logical.append(engine.last_step_logical)
                backward_logical.append(engine.last_backward_logical)
            ev1.record()
            ev1.synchronize()
            wall = time.perf_counter() - wall0
            steady = [r for r in engine.trace.rows if r["step"] >= k]
            total = steps - k
            utilization = {m.index: (sum(1 for r in steady if r["module"] == m.index and r["phase"] == "backward")
                                     / total if total > 0 else 1.0) for m in engine.modules}
        finally:
            engine.close()
        synth = LogicalCostModel.synthetic(k, module_cost, cfg.relay_cost)
        seq_logical = sum(synth.fwd) + sum(synth.bwd) + 2 * (k - 1) * cfg.relay_cost
        seq_backward = k * module_cost + (k - 1) * cfg.relay_cost
        device_ms = ev0.elapsed_time(ev1) / max(steps - warm, 1)
        rows.append({
            "k": k, "wall_steps_per_sec": steps / wall,
            "logical_per_step": logical[-1], "sequential_logical_per_step": seq_logical,
            "speedup_logical": seq_logical / logical[-1],
            "backward_logical": backward_logical[-1], "sequential_backward_logical": seq_backward,
            "speedup_backward": seq_backward / backward_logical[-1], "utilization": utilization,
            "device_ms_per_step": device_ms,
            "tokens_per_sec": cfg.batch_size * cfg.seq_len / (device_ms / 1e3),
        })
    return rows
