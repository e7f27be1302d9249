"""Optimizers applied to delayed-gradient packets, plus LR schedules.

Drop-in for reference optim.py: `LrSchedule`, `SgdOptimizer`,
`AdamOptimizer`, `make_optimizer` with the same arguments, the same global
bias-correction clock (optim.py:99-112) and zero-padded early gradients fed
as literal zeros.  `apply` launches one fused update per layer buffer
(csrc/optim.cu): fp32 master, moments and gradient are read once, and the
compute-dtype copy of the new weights is written straight into the module's
next snapshot-ring slot.
"""

import math
from dataclasses import dataclass

import torch

from . import ops


@dataclass
class LrSchedule:
    """fixed | diminishing base/(1+t) | linear warm-up then cosine to zero."""

    base: float
    mode: str = "fixed"
    warmup_steps: int = 0
    total_steps: int = 0

    def __post_init__(self):
        if self.base <= 0:
            raise ValueError("base learning rate must be positive")
        if self.mode not in ("fixed", "diminishing", "warmup-cosine"):
            raise ValueError(f"unknown schedule mode {self.mode!r}")
        if self.mode == "warmup-cosine" and self.warmup_steps >= self.total_steps:
            raise ValueError("warm-up must end before total_steps in cosine mode")

    def at(self, t):
        if t < 0:
            raise ValueError("step must be >= 0")
        if self.mode == "fixed":
            return self.base
        if self.mode == "diminishing":
            return self.base / (1.0 + t)
        if t < self.warmup_steps:
            return self.base * (t + 1) / self.warmup_steps
        x = (t - self.warmup_steps) / (self.total_steps - self.warmup_steps)
        return self.base * 0.5 * (1.0 + math.cos(math.pi * x))


def _targets(module, t):
    return [st.copy_targets(t + 1) for st in module.storage]


class _Base:
    """`apply` = `apply_module` for every module + `apply_tied`.  The split
    form lets the concurrent executor update a module as soon as its own
    delayed backward is done, and the tied matrix as soon as both of its
    gradient halves are in (each parameter is still updated exactly once per
    step with the packet's gradient)."""

    def apply(self, t, packet, modules, tied):
        self.prepare(modules)
        for m in modules:
            self.apply_module(t, m)
        if tied is not None:
            self.apply_tied(t, _tied_store(modules), modules[0].runtime.flag)
        return self.schedule.at(t)

    def prepare(self, modules):
        pass

    def apply_module(self, t, module):
        flag = module.runtime.flag
        for st, (vec_dst, mat_dst) in zip(module.storage, _targets(module, t)):
            n = st.flat_master.numel()
            if n == 0:
                continue
            self._update(t, st, 0, st.n_vec, vec_dst, flag)
            self._update(t, st, st.n_vec, n, mat_dst, flag)

    def apply_tied(self, t, store, flag):
        copy = None if store.flat_compute is store.flat_master else store.flat_compute
        self._update(t, store, 0, store.flat_master.numel(), copy, flag)


class SgdOptimizer(_Base):
    name = "sgd"

    def __init__(self, schedule):
        self.schedule = schedule

    def _update(self, t, st, lo, hi, dst, flag):
        if hi > lo:
            ops.sgd_step(st.flat_master[lo:hi], st.flat_grad[lo:hi], dst, hi - lo, self.schedule.at(t), flag)

    def state_arrays(self):
        return {}

    def load_state_arrays(self, arrays):
        if arrays:
            raise ValueError("sgd carries no optimizer state")


class AdamOptimizer(_Base):
    name = "adam"

    def __init__(self, schedule, beta1=0.9, beta2=0.999, eps=1e-8):
        self.schedule = schedule
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self._mods = []
        self._pending = None

    @staticmethod
    def _moments(obj):
        if obj.m is None:
            obj.m = torch.zeros_like(obj.flat_master)
            obj.v = torch.zeros_like(obj.flat_master)
        return obj.m, obj.v

    def prepare(self, modules):
        if list(modules) != self._mods:
            self.bind(modules)

    def _update(self, t, st, lo, hi, dst, flag):
        if hi > lo:
            lr = self.schedule.at(t)
            c1 = 1.0 - self.beta1 ** (t + 1)
            c2 = 1.0 - self.beta2 ** (t + 1)
            m, v = self._moments(st)
            ops.adam_step(st.flat_master[lo:hi], st.flat_grad[lo:hi], m[lo:hi], v[lo:hi], dst, hi - lo, lr, self.beta1,
                          self.beta2, self.eps, c1, c2, flag)

    def bind(self, modules):
        """Attach the modules whose moments `state_arrays` /
        `load_state_arrays` address (`apply` binds them too)."""
        self._mods = list(modules)
        pending, self._pending = getattr(self, "_pending", None), None
        if pending:
            self.load_state_arrays(pending)
        return self

    def _moment_views(self):
        """(key, m view, v view) for every live parameter: views into the
        flat moment buffers with the parameter's own strides (wq/wk/wv are
        column blocks of the fused wqkv)."""
        out = []
        for m in self._mods:
            start = m.layer_range[0]
            for off, st in enumerate(m.storage):
                if st.master.numel() == 0:
                    continue
                mb, vb = self._moments(st)
                for name, view in st.params.items():
                    args = (view.size(), view.stride(), view.storage_offset())
                    out.append((f"L{start + off}.{name}", mb.as_strided(*args), vb.as_strided(*args)))
        store = _tied_store(self._mods)
        if store is not None:
            mb, vb = self._moments(store)
            out.append(("tied", store.rows(mb), store.rows(vb)))
        return out

    def state_arrays(self):
        """Moments keyed `adam.m.{key}` / `adam.v.{key}` like the reference
        (optim.py:128-135); device views, not copies."""
        out = {}
        for key, mv, vv in self._moment_views():
            out[f"adam.m.{key}"] = mv
            out[f"adam.v.{key}"] = vv
        return out

    def load_state_arrays(self, arrays):
        """Inverse of `state_arrays` (optim.py:137-146).  Keys the checkpoint
        lacks restart from zero moments, as the reference's lazily created
        entries do.  Before the modules are bound the arrays are held until
        `bind` / the next `apply`."""
        for name in arrays:
            if not name.startswith(("adam.m.", "adam.v.")):
                raise ValueError(f"unexpected optimizer state entry {name!r}")
        if not self._mods:
            self._pending = dict(arrays)
            return
        for key, mv, vv in self._moment_views():
            for prefix, dst in (("adam.m.", mv), ("adam.v.", vv)):
                src = arrays.get(prefix + key)
                if src is None:
                    dst.zero_()
                else:
                    dst.copy_(torch.as_tensor(src).reshape(dst.shape))


def _flag_of(modules):
    return modules[0].runtime.flag if modules else None


def _tied_store(modules):
    for m in modules:
        if m.tied is not None:
            return m.tied
    return None


def make_optimizer(kind, schedule, beta1=0.9, beta2=0.999, eps=1e-8):
    if kind == "sgd":
        return SgdOptimizer(schedule)
    if kind == "adam":
        return AdamOptimizer(schedule, beta1, beta2, eps)
    raise ValueError(f"unknown optimizer {kind!r}")
