"""Layer stack, contiguous ring partition, and device-resident Ouroboros modules.

Drop-in for reference model.py: `build_stack`, `LayerStack`, `partition`,
`ModulePartition`, `StaleSlot`, `ModuleState`, `build_modules`,
`PartitionError`, `ScheduleViolation` keep their names and argument meaning.

B200 layout:
  * every layer owns one flat fp32 master buffer [vectors | matrices] with a
    same-shaped gradient buffer; the reference-facing `params` / grads dicts
    are views into it (wq/wk/wv are column blocks of one [d, 3d] wqkv);
  * the snapshot ring (model.py:175-196) is a ring of compute-dtype copies of
    that buffer; the optimizer writes the next step's copy directly into the
    next ring slot, so `snapshot(t)` is free in steady state;
  * the tied matrix V lives once on the Ouroboros device: fp32 master, fp32
    gradient (= the packet's mixed embedding gradient) and a compute copy;
  * stale slots (model.py:162-168) keep every forward intermediate
    ("store-all"), which the reference proves bitwise equal to its recompute
    (tests/test_model.py:110-129); `stale_weights="current"` recomputes at
    the live weights.
"""

import math
import weakref
from collections import deque
from dataclasses import dataclass

import torch

from .adaptive import AdaptiveHead, HostCopy, clusters
from . import layers as LY
from . import ops
from .errors import DimensionError, PartitionError, ScheduleViolation
from .rng import mix64
from .runtime import Runtime
from .xl import XLTape, sinusoid, xl_block_backward, xl_block_forward

# ---------------------------------------------------------------------------
# layer descriptors (the reference layer kinds, layers.py:96-280)


class EmbeddingLayer:
    kind = "embedding"

    def __init__(self, vocab_size, model_dim, max_seq_len, dropout_p):
        self.vocab_size, self.model_dim = vocab_size, model_dim
        self.max_seq_len, self.dropout_p = max_seq_len, dropout_p

    def specs(self):
        return [], [("pos", (self.max_seq_len, self.model_dim))]


class TransformerBlockLayer:
    kind = "block"

    def __init__(self, model_dim, ffn_dim, dropout_p, activation="relu"):
        """activation: the FFN nonlinearity -- "relu" (the reference,
        layers.py:191) or "gelu" (exact erf form, a production option)."""
        if activation not in LY.ACTIVATIONS:
            raise ValueError(f"unknown activation {activation!r}")
        self.model_dim, self.ffn_dim, self.dropout_p = model_dim, ffn_dim, dropout_p
        self.activation = activation

    def specs(self):
        d, f = self.model_dim, self.ffn_dim
        dims = {"d": d, "f": f, "3d": 3 * d}
        vec = [(n, (dims[s],)) for n, s in LY.BLOCK_VEC]
        mat = [(n, (dims[a], dims[b])) for n, (a, b) in LY.BLOCK_MAT]
        return vec, mat


class TransformerXLBlockLayer:
    """Transformer-XL block: relative-position multi-head attention over
    [segment memory; segment] in the reference's pre-LN block (xl.py,
    oracle/xl.py).  `mem_len` <= the segment length."""

    kind = "xl_block"
    VEC = LY.BLOCK_VEC + (("r_w_bias", ("H", "dh")), ("r_r_bias", ("H", "dh")))
    MAT = LY.BLOCK_MAT + (("wr", ("d", "d")),)
    KEYS = ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "wr", "r_w_bias", "r_r_bias", "ln2_g", "ln2_b", "w1", "b1",
            "w2", "b2")

    def __init__(self, model_dim, ffn_dim, dropout_p, n_heads, mem_len, activation="relu"):
        if model_dim % n_heads:
            raise DimensionError("model_dim must be a multiple of n_heads")
        if activation not in LY.ACTIVATIONS:
            raise ValueError(f"unknown activation {activation!r}")
        self.model_dim, self.ffn_dim, self.dropout_p = model_dim, ffn_dim, dropout_p
        self.n_heads, self.mem_len = n_heads, mem_len
        self.activation = activation

    def specs(self):
        d, f, H = self.model_dim, self.ffn_dim, self.n_heads
        dims = {"d": d, "f": f, "3d": 3 * d, "H": H, "dh": d // H}
        vec = [(n, tuple(dims[x] for x in ((s,) if isinstance(s, str) else s))) for n, s in self.VEC]
        mat = [(n, (dims[a], dims[b])) for n, (a, b) in self.MAT]
        return vec, mat


class OutputProjectionLayer:
    kind = "projection"

    def __init__(self, vocab_size, model_dim, cutoffs=None):
        """cutoffs: adaptive tied softmax (adaptive.py, oracle/adaptive.py):
        the projection then owns one weight row and bias per tail cluster."""
        self.vocab_size, self.model_dim = vocab_size, model_dim
        self.cutoffs = list(cutoffs) if cutoffs else None
        self.n_clusters = len(clusters(self.cutoffs, vocab_size)) if self.cutoffs else 0

    def specs(self):
        if not self.n_clusters:
            return [], []
        return [("cluster_bias", (self.n_clusters,))], [("cluster_weight", (self.n_clusters, self.model_dim))]


# ---------------------------------------------------------------------------
# device storage


def _dtype_of(name):
    if name in ("bf16", torch.bfloat16):
        return torch.bfloat16
    if name in ("fp32", "f32", torch.float32):
        return torch.float32
    raise ValueError(f"unknown compute dtype {name!r}")


class LayerParams:
    """fp32 master + gradient + snapshot ring of one layer.

    Flat buffers: the vectors, then the matrices row-major.  A matrix whose
    compute-dtype rows would not be 16-byte multiples (bf16, cols % 8 != 0:
    BASELINE configs[3]'s d 410, d_ff 2100) keeps its rows at LY.pad_cols
    pitch in EVERY buffer (master, gradient, moments, ring), so the optimizer
    and the casts stay one flat elementwise pass; the pad columns are zero
    and stay zero (nothing writes them, and zero weight + zero gradient is a
    fixed point of SGD and Adam).  Every vector and matrix starts on a
    64-element boundary (256 bytes fp32), so each view is as aligned as a
    fresh allocation whatever the widths (d 410 vectors would otherwise leave
    the matrices 8-byte aligned)."""

    ALIGN = 64

    def __init__(self, layer, device, cdtype):
        self.layer, self.device, self.cdtype = layer, device, cdtype
        vec, mat = layer.specs()
        up = lambda n: -(-n // self.ALIGN) * self.ALIGN  # noqa: E731
        self._mat_pitch = [LY.pad_cols(s[-1], cdtype) for _, s in mat]
        self._vec_off, off = [], 0
        for _, s in vec:
            self._vec_off.append(off)
            off = up(off + math.prod(s))
        self.n_vec = off
        self._mat_off, off = [], 0
        for (_, s), pc in zip(mat, self._mat_pitch):
            self._mat_off.append(off)
            off = up(off + s[0] * pc)
        self.n_mat = off
        n = self.n_vec + self.n_mat
        self.master = torch.zeros(n, dtype=torch.float32, device=device)
        self.grad = torch.zeros(n, dtype=torch.float32, device=device)
        self.flat_master, self.flat_grad = self.master, self.grad
        self.m = self.v = None
        self._vec_specs, self._mat_specs = vec, mat
        self.P = self._carve(self.master, torch.float32, torch.float32)  # internal names
        self.G = self._carve(self.grad, torch.float32, torch.float32)
        self.params = self._public(self.P)
        self.grads = self._public(self.G)
        self.ring = []
        self.ring_step = []

    def _carve(self, flat, vec_dt, mat_dt, vec_flat=None, mat_flat=None):
        out = {}
        if vec_flat is None:
            vec_flat, mat_flat = flat[: self.n_vec], flat[self.n_vec:]
        for (name, shape), off in zip(self._vec_specs, self._vec_off):
            out[name] = vec_flat[off: off + math.prod(shape)].view(shape)
        for name, off, r, c, pc in self.mat_blocks():
            out[name] = mat_flat[off: off + r * pc].view(r, pc)[:, :c]
        return out

    def mat_blocks(self):
        """(name, offset in the matrix part, rows, cols, row pitch) per matrix."""
        return [(name, off, r, c, pc) for (name, (r, c)), pc, off in zip(self._mat_specs, self._mat_pitch,
                                                                          self._mat_off)]

    def _public(self, D):
        if self.layer.kind not in ("block", "xl_block"):
            return dict(D)
        d = self.layer.model_dim
        w = D["wqkv"]
        views = {"wq": w[:, :d], "wk": w[:, d: 2 * d], "wv": w[:, 2 * d:]}
        keys = LY.BLOCK_KEYS if self.layer.kind == "block" else self.layer.KEYS
        return {k: (views[k] if k in views else D[k]) for k in keys}

    # -- snapshot ring ----------------------------------------------------
    def configure_ring(self, capacity):
        self.ring = []
        for _ in range(capacity):
            vec = torch.empty(self.n_vec, dtype=torch.float32, device=self.device)
            mat = torch.zeros(self.n_mat, dtype=self.cdtype, device=self.device)
            self.ring.append((vec, mat, self._carve(None, None, None, vec, mat)))
        self.ring_step = [None] * capacity

    def ring_slot(self, step):
        return step % len(self.ring)

    def ensure(self, step):
        """Make the ring hold the current master weights for `step`."""
        i = self.ring_slot(step)
        if self.ring_step[i] != step:
            vec, mat, _ = self.ring[i]
            if self.n_vec:
                vec.copy_(self.master[: self.n_vec])
            if self.n_mat:
                ops.cast(self.master[self.n_vec:], mat)
            self.ring_step[i] = step

    def weights(self, step):
        i = self.ring_slot(step)
        if self.ring_step[i] != step:
            raise ScheduleViolation(f"snapshot for step {step} not in ring")
        return self.ring[i][2]

    def copy_targets(self, step):
        """(vec, mat) buffers the optimizer fills with the weights for `step`."""
        i = self.ring_slot(step)
        self.ring_step[i] = step
        vec, mat, _ = self.ring[i]
        return vec, mat

    def nbytes(self):
        return (self.master.numel() * 4 * (2 if self.m is None else 4)
                + sum(v.numel() * 4 + m.numel() * m.element_size() for v, m, _ in self.ring))


class TiedMatrix:
    """The shared input-embedding / output-projection matrix V on the
    Ouroboros device (model.py:55-59)."""

    def __init__(self, vocab, d, device, cdtype):
        self.vocab, self.d, self.device, self.cdtype = vocab, d, device, cdtype
        # rows at LY.pad_cols pitch in every buffer, as LayerParams
        self.pitch = pd = LY.pad_cols(d, cdtype)
        self.flat_master = torch.zeros(vocab * pd, dtype=torch.float32, device=device)
        self.flat_grad = torch.zeros(vocab * pd, dtype=torch.float32, device=device)
        self.flat_compute = (self.flat_master if cdtype == torch.float32
                             else torch.zeros(vocab * pd, dtype=cdtype, device=device))
        self.master, self.grad, self.compute = (self.rows(t) for t in (self.flat_master, self.flat_grad,
                                                                        self.flat_compute))
        self.m = self.v = None

    def rows(self, flat):
        """The logical [vocab, d] view of a flat buffer in this layout."""
        return flat.view(self.vocab, self.pitch)[:, : self.d]

    def refresh(self):
        if self.flat_compute is not self.flat_master:
            ops.cast(self.flat_master, self.flat_compute)


class LayerStack:
    """The unpartitioned model (model.py:36-50): `layers`, `params` (per-layer
    dicts of fp32 master views; embedding and projection dicts share the one
    `tied` tensor) and `tied`."""

    def __init__(self, layers, storage, tied, runtime, cdtype, register=True):
        self.layers = layers
        if register:
            _STACKS[id(layers)] = weakref.ref(self)
        self.storage = storage
        self.tied_store = tied
        self.tied = tied.master
        self.runtime = runtime
        self.cdtype = cdtype
        self.params = []
        for layer, st in zip(layers, storage):
            p = dict(st.params)
            if layer.kind in ("embedding", "projection"):
                p = {"tied": self.tied, **p}
            self.params.append(p)

    @property
    def num_layers(self):
        return len(self.layers)

    def twin(self):
        """A second stack of the same layers on the same device (zero weights,
        own storage), cached: the scratch model `engine.sequential_gradients`
        evaluates explicit weights on without touching the live ones."""
        tw = getattr(self, "_twin", None)
        if tw is None:
            dev = self.runtime.device
            storage = [LayerParams(layer, dev, self.cdtype) for layer in self.layers]
            tied = TiedMatrix(self.tied_store.vocab, self.tied_store.d, dev, self.cdtype)
            tw = self._twin = LayerStack(self.layers, storage, tied, self.runtime, self.cdtype, register=False)
        return tw

    def refresh(self):
        """Re-derive every compute copy from the fp32 masters after the caller
        edited `params` / `tied` in place (the reference's live arrays have no
        copies to invalidate)."""
        for st in self.storage:
            st.ring_step = [None] * len(st.ring)
        self.tied_store.refresh()


_STACKS = {}  # id(stack.layers) -> weakref(stack): `layers` lists name their stack


def stack_of(layers):
    """The LayerStack a `layers` list (or the stack itself) belongs to."""
    if isinstance(layers, LayerStack):
        return layers
    ref = _STACKS.get(id(layers))
    st = ref() if ref is not None else None
    if st is None or st.layers is not layers:
        raise ValueError("layers must be the .layers list of a stack built by build_stack / build_xl_stack")
    return st


def build_stack(vocab_size, model_dim, ffn_dim, n_blocks, seq_len, dropout_p, init_seed, *, dtype="bf16",
                device=None, activation="relu"):
    """Same draw order and scales as the reference (model.py:53-60,
    layers.py:107-112, 149-166): V ~ U(+-1/sqrt(d)) first, then per layer the
    position table and wq, wk, wv, wo, w1 (1/sqrt(d)) and w2 (1/sqrt(f));
    gains 1, biases 0.  The stream is evaluated on the device."""
    if model_dim % 8 or ffn_dim % 8:
        raise DimensionError("model_dim and ffn_dim must be multiples of 8 (TMA 16-byte rows)")
    rt = Runtime.get(device)
    cdt = _dtype_of(dtype)
    layers = [EmbeddingLayer(vocab_size, model_dim, seq_len, dropout_p)]
    layers += [TransformerBlockLayer(model_dim, ffn_dim, dropout_p, activation) for _ in range(n_blocks)]
    layers.append(OutputProjectionLayer(vocab_size, model_dim))
    storage = [LayerParams(layer, rt.device, cdt) for layer in layers]
    tied = TiedMatrix(vocab_size, model_dim, rt.device, cdt)
    with torch.cuda.device(rt.device):
        _init_params(layers, storage, tied, init_seed)
        tied.refresh()
    return LayerStack(layers, storage, tied, rt, cdt)


def build_xl_stack(vocab_size, model_dim, ffn_dim, n_blocks, seq_len, dropout_p, init_seed, n_heads, mem_len, *,
                   dtype="bf16", device=None, cutoffs=None, activation="relu"):
    """The Transformer-XL language model: the reference embedding and tied
    head around `n_blocks` XL blocks with `mem_len` memory rows each."""
    # widths that are not multiples of 8 (BASELINE configs[3]: d 410, 10 heads x 41,
    # d_ff 2100) keep every bf16 row at a 16-byte pitch (LY.pad_cols) through the
    # op-level path; the full-vocabulary head is a dense-row C-ABI composite, so
    # such widths take the adaptive head (configs[3]'s own head)
    if (model_dim % 8 or ffn_dim % 8 or (model_dim // n_heads) % 8) and not cutoffs:
        raise DimensionError("widths that are not multiples of 8 need the adaptive head (cutoffs)")
    if not 0 <= mem_len <= seq_len:
        raise DimensionError("mem_len must be in [0, seq_len]")
    rt = Runtime.get(device)
    cdt = _dtype_of(dtype)
    layers = [EmbeddingLayer(vocab_size, model_dim, seq_len, dropout_p)]
    layers += [TransformerXLBlockLayer(model_dim, ffn_dim, dropout_p, n_heads, mem_len, activation)
               for _ in range(n_blocks)]
    layers.append(OutputProjectionLayer(vocab_size, model_dim, cutoffs))
    storage = [LayerParams(layer, rt.device, cdt) for layer in layers]
    tied = TiedMatrix(vocab_size, model_dim, rt.device, cdt)
    with torch.cuda.device(rt.device):
        _init_params(layers, storage, tied, init_seed)
        tied.refresh()
    return LayerStack(layers, storage, tied, rt, cdt)


def _init_params(layers, storage, tied, init_seed):
    seed = mix64(init_seed)
    pos = 0
    d = tied.d
    sd = 1.0 / math.sqrt(d)

    def draw(dst, scale):
        nonlocal pos
        if dst.is_contiguous():
            ops.init_uniform(dst, seed, pos, scale)
        else:
            tmp = torch.empty(dst.shape, dtype=torch.float32, device=dst.device)
            ops.init_uniform(tmp, seed, pos, scale)
            dst.copy_(tmp)
        pos += dst.numel()

    draw(tied.master, sd)
    for layer, st in zip(layers, storage):
        P = st.params
        if layer.kind == "embedding":
            draw(P["pos"], sd)
        elif layer.kind == "block":
            P["ln1_g"].fill_(1.0)
            P["ln2_g"].fill_(1.0)
            for w in ("wq", "wk", "wv", "wo", "w1"):
                draw(P[w], sd)
            draw(P["w2"], 1.0 / math.sqrt(layer.ffn_dim))
        elif layer.kind == "xl_block":  # oracle/xl.py init_xl_params order
            P["ln1_g"].fill_(1.0)
            P["ln2_g"].fill_(1.0)
            for w in ("wq", "wk", "wv", "wo", "wr", "r_w_bias", "r_r_bias", "w1"):
                draw(P[w], sd)
            draw(P["w2"], 1.0 / math.sqrt(layer.ffn_dim))
        elif layer.kind == "projection" and layer.n_clusters:  # oracle/xl.py init_xl_params
            draw(P["cluster_weight"], sd)


# ---------------------------------------------------------------------------
# partition (model.py:63-141) -- pure integer logic


@dataclass
class ModulePartition:
    k: int
    groups: list
    device_of: list

    def __post_init__(self):
        if len(self.groups) != self.k or len(self.device_of) != self.k:
            raise PartitionError("group/device lists must have K entries")
        nxt = 0
        for lo, hi in self.groups:
            if lo != nxt or hi <= lo:
                raise PartitionError("groups must be contiguous, ordered, nonempty")
            nxt = hi
        if self.k >= 2 and self.device_of[0] != self.device_of[-1]:
            raise PartitionError("first and last module must share a device")

    @property
    def num_devices(self):
        return len(set(self.device_of))


def _balanced(L, K):
    q, r = divmod(L, K)
    return [q + (i < r) for i in range(K)]


def _minmax(costs, K):
    """Contiguous split of `costs` into K groups minimising the largest group
    sum; ties resolved towards the earliest cut (reference DP order)."""
    L = len(costs)
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + float(c))
    INF = float("inf")
    best = [[INF] * (L + 1) for _ in range(K + 1)]
    cut = [[0] * (L + 1) for _ in range(K + 1)]
    best[0][0] = 0.0
    for k in range(1, K + 1):
        for j in range(k, L - (K - k) + 1):
            for i in range(k - 1, j):
                if best[k - 1][i] == INF:
                    continue
                val = max(best[k - 1][i], pre[j] - pre[i])
                if val < best[k][j]:
                    best[k][j], cut[k][j] = val, i
    sizes, j = [], L
    for k in range(K, 0, -1):
        i = cut[k][j]
        sizes.append(j - i)
        j = i
    return sizes[::-1]


def partition(L, K, balance="even", costs=None):
    """K contiguous groups over L layers; modules 1 and K share device 0, so
    K modules occupy K-1 devices (ring placement, model.py:115-141)."""
    if not 1 <= K <= L:
        raise PartitionError(f"need 1 <= K <= L, got K={K}, L={L}")
    if balance == "even":
        sizes = _balanced(L, K)
    elif balance == "by_cost":
        if costs is None or len(costs) != L:
            raise PartitionError("by_cost needs one cost per layer")
        sizes = _minmax(costs, K)
    else:
        raise PartitionError(f"unknown balance mode {balance!r}")
    groups, lo = [], 0
    for s in sizes:
        groups.append((lo, lo + s))
        lo += s
    device_of = [0] if K == 1 else [0, *range(1, K - 1), 0]
    return ModulePartition(K, groups, device_of)


def measure_layer_costs(stack, batch_x, dropout_seed=0, repeats=3):
    """Device seconds of one forward + backward per layer, for the by_cost
    partition (reference model.py:144-159 times the same thing with the wall
    clock).  Each layer runs on scratch activations at the batch's shape,
    after one untimed warm-up, bracketed by CUDA events on the current stream.
    The stack's gradient buffers are used as scratch (the engines overwrite
    them every step); weights and snapshot rings are untouched."""
    rt = stack.runtime
    dev = rt.device
    tokens = torch.as_tensor(batch_x).to(device=dev, dtype=torch.int64)
    B, T = tokens.shape
    Nt = B * T
    tied = stack.tied_store
    d, cdt = tied.d, stack.cdtype
    ws = LY.Workspace(dev)
    act = LY.empty_rows(Nt, d, dtype=cdt, device=dev)
    out = LY.empty_rows(Nt, d, dtype=cdt, device=dev)
    g_out = torch.ones(Nt, d, dtype=torch.float32, device=dev)
    g_in = torch.empty_like(g_out)
    targets = torch.zeros(Nt, dtype=torch.int64, device=dev)
    tape = head = xtape = adaptive = R = ytgt = None
    act.zero_()
    costs = []
    for idx, (layer, st) in enumerate(zip(stack.layers, stack.storage)):
        mat = torch.empty(st.n_mat, dtype=cdt, device=dev)
        if st.n_mat:
            ops.cast(st.master[st.n_vec:], mat)
        W = st._carve(None, None, None, st.master[: st.n_vec], mat)
        drop = LY.Dropout.make(mix64(dropout_seed, 0, idx), getattr(layer, "dropout_p", 0.0), True)
        if layer.kind == "embedding":
            def run():
                LY.embed_forward(tied.compute, W["pos"], tokens, act, tied.vocab, drop, rt.flag)
                LY.embed_backward(g_out, tokens, layer.max_seq_len, st.G["pos"], tied.grad, 1.0, ws, drop)
        elif layer.kind == "block":
            if tape is None:
                tape = LY.BlockTape(B, T, d, layer.ffn_dim, cdt, dev, layer.activation)

            def run():
                LY.block_forward(W, W, act, out, tape, B, T, drop, ws, rt.flag)
                LY.block_backward(W, W, act, tape, g_out, g_in, st.G, B, T, drop, ws)
        elif layer.kind == "xl_block":
            # a full memory (the steady state): attention over M + T keys
            if xtape is None:
                xtape = XLTape(B, T, layer.mem_len, d, layer.ffn_dim, layer.n_heads, cdt, dev, layer.activation)
                xtape.xa.zero_()
                xtape.mem_len = layer.mem_len
                R = sinusoid(xtape.Kl, d, cdt, dev)

            def run():
                xl_block_forward(W, W, out, xtape, R, drop, ws, rt.flag)
                xl_block_backward(W, W, xtape, R, g_out, g_in, st.G, drop, ws)
        elif layer.n_clusters:
            # adaptive tied softmax: the head cluster for every row, each tail
            # for the rows whose (Zipf-distributed, model.py:144-159 has no
            # targets either) synthetic target falls in it
            if adaptive is None:
                adaptive = AdaptiveHead(layer.vocab_size, d, layer.cutoffs, dev, cdt)
                w = 1.0 / torch.arange(1, layer.vocab_size + 1, dtype=torch.float64)
                ytgt = torch.multinomial(w / w.sum(), Nt, replacement=True,
                                         generator=torch.Generator().manual_seed(0)).numpy()
            P, Gp = W, st.G

            def run():
                adaptive.forward(act, tied.compute, P["cluster_weight"], P["cluster_bias"], ytgt, rt.flag)
                adaptive.backward(g_in, tied.grad, Gp["cluster_weight"], Gp["cluster_bias"], alpha=1.0,
                                  accumulate=False)
        else:
            if head is None:
                head = LY.HeadState(Nt, dev)

            def run():
                LY.head_forward(act, tied.compute, targets, tied.vocab, head, ws, rt.flag)
                LY.head_backward(act, tied.compute, targets, tied.vocab, head, g_in, tied.grad, 1.0, ws)
        run()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(repeats):
            run()
        end.record()
        end.synchronize()
        costs.append(start.elapsed_time(end) / 1e3 / repeats)
    rt.flag.zero_()
    return costs


# ---------------------------------------------------------------------------
# modules


@dataclass
class StaleSlot:
    step: int
    sample_id: int
    inputs: object
    targets: object
    layer_seeds: list
    arena: object = None


class _Arena:
    """Device storage of one stale slot: module input, every block's tape,
    tokens (embedding module) / targets + head state (projection module)."""

    def __init__(self, module, B, T):
        dev, cdt = module.device, module.cdtype
        d, Nt = module.d, B * T
        self.B, self.T = B, T
        self.tokens = torch.empty(B, T, dtype=torch.int64, device=dev) if module.has_embedding else None
        self.targets = torch.empty(Nt, dtype=torch.int64, device=dev) if module.has_projection else None
        self.tapes = []
        self.acts = []
        for off in module.block_idx:
            layer = module.layers[off]
            if layer.kind == "xl_block":
                tp = XLTape(B, T, layer.mem_len, d, layer.ffn_dim, layer.n_heads, cdt, dev, layer.activation)
                self.acts.append(tp.x)  # the upstream writes straight into [memory; x]
            else:
                tp = LY.BlockTape(B, T, d, layer.ffn_dim, cdt, dev, layer.activation)
                self.acts.append(LY.empty_rows(Nt, d, dtype=cdt, device=dev))
            self.tapes.append(tp)
        if module.has_projection:
            self.acts.append(LY.empty_rows(Nt, d, dtype=cdt, device=dev))
        self.head = LY.HeadState(Nt, dev) if module.has_projection else None
        last = module.layers[-1]
        self.adaptive = (AdaptiveHead(last.vocab_size, d, last.cutoffs, dev, cdt)
                         if module.has_projection and last.n_clusters else None)
        self.targets_host = None  # the adaptive head buckets rows by cluster from the host targets


class ModuleState:
    """One pipeline module (model.py:199-304) resident on one device.

    Micro-batched relay (distributed.py): `forward(..., micro=(j, m),
    batch_shape=(B, T))` runs row block j of m of the batch; the slot keeps one
    arena per row block (B/m rows each) and the delayed backward runs them in
    order j = 0..m-1, summing their weight gradients in that order.  Dropout
    positions stay the flat [B, T, d] indices of the whole batch (the stream is
    shifted to the block's first row), the loss normaliser stays B*T, so the
    result is the whole-batch step up to fp32 summation order."""

    supports_micro = True

    def __init__(self, index, k_total, layer_range, layers, params, dropout_seed, *, storage=None, tied=None,
                 runtime=None, cdtype=torch.bfloat16):
        self.index, self.k_total, self.layer_range = index, k_total, layer_range
        self.layers, self.params = layers, params
        self.storage = storage
        self.tied = tied
        self.runtime = runtime
        self.device = runtime.device
        self.cdtype = cdtype
        self.dropout_seed = dropout_seed
        self.slot_capacity = k_total - index + 1
        self.slots = deque()
        self.peak_slot_floats = 0
        self.peak_slots = 0
        self.has_embedding = layers[0].kind == "embedding"
        self.has_projection = layers[-1].kind == "projection"
        self.block_idx = [i for i, l in enumerate(layers) if l.kind in ("block", "xl_block")]
        # Transformer-XL segment memory: per XL block the previous segment's
        # layer input [B*M, d], and how many of its rows are valid
        self.mem = {}
        self.mem_len = 0
        self._R = {}
        self.n_blocks = len(self.block_idx)
        ref = layers[self.block_idx[0]] if self.block_idx else layers[0]
        self.d = ref.model_dim
        self.f = layers[self.block_idx[0]].ffn_dim if self.block_idx else 8
        self.vocab = tied.vocab if tied is not None else None
        self.dropout_p = getattr(layers[0], "dropout_p", 0.0) if not self.block_idx else layers[self.block_idx[0]].dropout_p
        if self.has_embedding:
            self.dropout_p = layers[0].dropout_p
        for st in storage:
            st.configure_ring(self.slot_capacity)
        self._arenas = [None] * self.slot_capacity
        self._shape = None
        self._parts = 1
        self._loss_total = None
        self.ws_fwd = LY.Workspace(self.device)
        self.ws_bwd = LY.Workspace(self.device)
        start = layer_range[0]
        self.grad_views = {}
        for off, st in enumerate(storage):
            for name, t in st.grads.items():
                self.grad_views[f"L{start + off}.{name}"] = t
        self._standalone_tied = None
        self.last_forward_step = None
        # per-module device status word (RP_FLAG_*), polled once per step
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    # -- seeds / snapshots -------------------------------------------------
    def _layer_seed(self, step, offset):
        return mix64(self.dropout_seed, step, self.layer_range[0] + offset)

    def snapshot(self, step):
        for st in self.storage:
            st.ensure(step)

    def _arena(self, step, B, T, parts=1, part=None):
        """The slot storage of `step`: one _Arena, or with parts > 1 the list
        of row-block arenas (B / parts rows each); `part` picks one."""
        if self._shape != (B, T) or self._parts != parts:
            if self.slots:
                raise DimensionError("batch shape changed while stale slots are pending")
            if B % parts:
                raise DimensionError(f"batch of {B} rows does not split into {parts} row blocks")
            self._arenas = [None] * self.slot_capacity
            self._shape = (B, T)
            self._parts = parts
        i = step % self.slot_capacity
        if self._arenas[i] is None:
            self._arenas[i] = (_Arena(self, B, T) if parts == 1 else
                               [_Arena(self, B // parts, T) for _ in range(parts)])
        a = self._arenas[i]
        return a if part is None or parts == 1 else a[part]

    def input_buffer(self, step, B, T, micro=None):
        """Where the upstream module should write this module's input (of row
        block j when micro = (j, m))."""
        j, m = micro if micro is not None else (None, 1)
        a = self._arena(step, B, T, m, j)
        return a.acts[0] if a.acts else None

    # -- forward -----------------------------------------------------------
    def forward(self, x, step, sample_id, targets=None, train=True, out=None, micro=None, batch_shape=None):
        """Run the slice at the live weights of `step` and queue a stale slot.
        Returns the output activations [B*T, d], or for the projection module
        the mean cross-entropy as a 0-d device tensor.  micro = (j, m) with
        batch_shape = (B, T): row block j of m (see the class docstring); the
        projection module returns the whole batch's loss after the last block."""
        if micro is not None and micro[1] > 1:
            return self._forward_block(x, step, sample_id, targets, train, out, micro, batch_shape)
        if self.has_embedding:
            B, T = x.shape
        else:
            B, T = self._shape if x is None else (None, None)
            if x is not None:
                Nt = x.numel() // self.d
                B, T = (x.shape[0], x.shape[1]) if x.dim() == 3 else self._infer_bt(Nt)
        seeds = [self._layer_seed(step, i) for i in range(len(self.layers))]
        arena = self._arena(step, B, T)
        if self.has_embedding:
            arena.tokens.copy_(x if torch.is_tensor(x) else torch.as_tensor(x), non_blocking=True)
        elif x is not None and arena.acts and x.data_ptr() != arena.acts[0].data_ptr():
            arena.acts[0].copy_(x.reshape(B * T, self.d))
        if self.has_projection:
            if targets is None:
                raise ScheduleViolation("projection module slot lacks targets")
            tt = targets if torch.is_tensor(targets) else torch.as_tensor(targets)
            arena.targets.copy_(tt.reshape(-1), non_blocking=True)
            # the adaptive head buckets rows on the host: device targets leave
            # by an early side-stream copy instead of a stream sync at the head
            arena.targets_host = (HostCopy(tt) if arena.adaptive is not None and torch.is_tensor(tt) and tt.is_cuda
                                  else targets)
        slot = StaleSlot(step, sample_id, arena.acts[0] if arena.acts else arena.tokens, targets, seeds, arena)
        self.slots.append(slot)
        if len(self.slots) > self.slot_capacity:
            self.slots.pop()
            raise ScheduleViolation(f"module {self.index} slot queue exceeded {self.slot_capacity}")
        self.peak_slots = max(self.peak_slots, len(self.slots))
        stored = len(self.slots) * B * T * (1 if self.has_embedding else self.d)
        self.peak_slot_floats = max(self.peak_slot_floats, stored)
        self.last_forward_step = step
        return self._run_forward(step, arena, seeds, train, out, self.ws_fwd)

    def _forward_block(self, x, step, sample_id, targets, train, out, micro, batch_shape):
        j, m = micro
        if batch_shape is None:
            raise DimensionError("a micro-batched forward needs batch_shape=(B, T)")
        B, T = batch_shape
        if self.layers[-1].kind == "projection" and self.layers[-1].n_clusters:
            raise DimensionError("the adaptive head does not run micro-batched")
        mb = B // m
        seeds = [self._layer_seed(step, i) for i in range(len(self.layers))]
        parts = self._arena(step, B, T, m)
        arena = parts[j]
        if j == 0:
            slot = StaleSlot(step, sample_id, None, targets, seeds, parts)
            self.slots.append(slot)
            if len(self.slots) > self.slot_capacity:
                self.slots.pop()
                raise ScheduleViolation(f"module {self.index} slot queue exceeded {self.slot_capacity}")
            self.peak_slots = max(self.peak_slots, len(self.slots))
            stored = len(self.slots) * B * T * (1 if self.has_embedding else self.d)
            self.peak_slot_floats = max(self.peak_slot_floats, stored)
        elif not self.slots or self.slots[-1].step != step or self.slots[-1].arena is not parts:
            raise ScheduleViolation(f"module {self.index}: row block {j} of step {step} before block 0")
        if self.has_embedding:
            arena.tokens.copy_(x if torch.is_tensor(x) else torch.as_tensor(x), non_blocking=True)
        elif x is not None and arena.acts and x.data_ptr() != arena.acts[0].data_ptr():
            arena.acts[0].copy_(x.reshape(mb * T, self.d))
        if self.has_projection:
            if targets is None:
                raise ScheduleViolation("projection module slot lacks targets")
            tt = targets if torch.is_tensor(targets) else torch.as_tensor(targets)
            arena.targets.copy_(tt.reshape(-1), non_blocking=True)
        self.last_forward_step = step
        res = self._run_forward(step, arena, seeds, train, out, self.ws_fwd, part=(j, m))
        if self.has_projection:
            return self._combined_loss(parts) if j == m - 1 else res
        return res

    def _combined_loss(self, parts):
        """Mean cross-entropy of the whole batch from its row blocks' means
        (equal block sizes), in block order."""
        if self._loss_total is None:
            self._loss_total = torch.zeros((), dtype=torch.float32, device=self.device)
        self._loss_total.copy_(parts[0].head.loss)
        for a in parts[1:]:
            self._loss_total.add_(a.head.loss)
        self._loss_total.div_(len(parts))
        return self._loss_total

    def _infer_bt(self, Nt):
        if self._shape is not None and self._shape[0] * self._shape[1] == Nt:
            return self._shape
        raise DimensionError("pass module inputs as [B, T, d] to fix the batch shape")

    # -- Transformer-XL memory ----------------------------------------------
    def _sinusoid(self, tp):
        key = (tp.Kl, self.d, self.cdtype)
        R = self._R.get(key)
        if R is None:
            R = self._R[key] = sinusoid(tp.Kl, self.d, self.cdtype, self.device)
        return R

    def _load_memory(self, off, tp, part=(0, 1)):
        """Memory rows of this segment = the previous segment's layer input
        (rows of row block j of m)."""
        j, m = part
        rows = tp.B * tp.M * m
        buf = self.mem.get(off)
        if buf is None or buf.shape[0] != rows:
            buf = self.mem[off] = LY.empty_rows(rows, self.d, dtype=self.cdtype, device=self.device)
            buf.zero_()
        LY.copy_rows(tp.mem, buf[j * tp.B * tp.M:(j + 1) * tp.B * tp.M])
        tp.mem_len = self.mem_len

    def _store_memory(self, off, tp, part=(0, 1)):
        if tp.M:
            j = part[0]
            dst = self.mem[off][j * tp.B * tp.M:(j + 1) * tp.B * tp.M]
            LY.copy_rows(dst.view(tp.B, tp.M, self.d), tp.x.view(tp.B, tp.T, self.d)[:, tp.T - tp.M:])

    def reset_memory(self):
        self.mem_len = 0

    def _run_forward(self, wstep, arena, seeds, train, out, ws, tied_c=None, from_act0=False, live=True,
                     part=(0, 1)):
        """Forward of the slice at ring weights `wstep`.  `tied_c` overrides
        the embedding table (a snapshot of V); `from_act0` starts at the first
        block from an embedding output already in arena.acts[0] (checkpoint
        re-derivation: V is not kept in the snapshot ring).  `live` marks the
        step's own forward, which reads and advances the XL memory; replays
        (stale_weights="current", re-derivation) reuse the slot's memory."""
        B, T = arena.B, arena.T
        flag = self.flag
        nxt = 0  # next act buffer to fill
        cur = None
        xl_live = None
        j, m = part
        rows_total = B * T * m if m > 1 else 0  # token rows of the whole batch (row block j of m)
        for off, layer in enumerate(self.layers):
            st = self.storage[off]
            p = layer.dropout_p if hasattr(layer, "dropout_p") else 0.0
            drop = LY.Dropout.shift(LY.Dropout.make(seeds[off], p, train), j * B * T * self.d)
            if layer.kind == "embedding":
                if from_act0:
                    cur, nxt = arena.acts[0], 1
                    continue
                dst = arena.acts[0] if arena.acts else out
                if dst is None:  # re-derivation of an embedding-only slot
                    dst = self.ws_fwd.get("module_out", (B * T, self.d), self.cdtype)
                Wv = st.weights(wstep)
                LY.embed_forward(self.tied.compute if tied_c is None else tied_c, Wv["pos"], arena.tokens, dst,
                                 self.vocab, drop, flag)
                cur = dst
                nxt = 1
            elif layer.kind in ("block", "xl_block"):
                jb = self.block_idx.index(off)
                x_in = arena.acts[jb]
                last_act = jb + 1 >= len(arena.acts)
                dst = out if last_act else arena.acts[jb + 1]
                if dst is None:
                    dst = self.ws_fwd.get("module_out", (B * T, self.d), self.cdtype)
                W = st.weights(wstep)
                if layer.kind == "xl_block":
                    tp = arena.tapes[jb]
                    if live:
                        self._load_memory(off, tp, part)
                    xl_block_forward(W, W, dst.view(B * T, self.d), tp, self._sinusoid(tp), drop, ws, flag,
                                     rows_total=rows_total)
                    if live:
                        self._store_memory(off, tp, part)
                        xl_live = tp.M
                else:
                    LY.block_forward(W, W, x_in, dst.view(B * T, self.d), arena.tapes[jb], B, T, drop, ws, flag,
                                     rows_total=rows_total)
                cur = dst
                nxt = jb + 2
            else:  # projection + fused CE head
                h = arena.acts[-1]
                if arena.adaptive is not None:
                    P = st.weights(wstep)
                    loss = arena.adaptive.forward(h, self.tied.compute, P["cluster_weight"], P["cluster_bias"],
                                                  arena.targets_host, flag)
                    arena.head.loss.copy_(loss)
                else:
                    LY.head_forward(h, self.tied.compute, arena.targets, self.vocab, arena.head, ws, flag)
                cur = arena.head.loss
        if xl_live is not None and j == m - 1:
            self.mem_len = xl_live  # M <= T: one segment fills the memory (after its last row block)
        return cur

    # -- backward ----------------------------------------------------------
    def pop_slot(self):
        if not self.slots:
            raise ScheduleViolation(f"module {self.index} has no pending slot")
        return self.slots.popleft()

    def recompute_backward(self, slot, grad_out, stale_mode="snapshot", train=True, *, g_in=None, emb=None,
                           live_step=None, after_head=None, before_embedding=None, vo_overwrite=False):
        """Delayed backward for one slot (model.py:250-293).

        "snapshot": gradients at the weights the slot's forward used (the
        ring entry for slot.step), from the stored intermediates.
        "current": re-run the forward at the live weights, then backprop.
        `emb=(alpha, beta, grad)` fuses the tied gradient into `grad`, which
        the caller zeroed: alpha*Vo and beta*Vi are both added (in either
        order -- with two terms on a zero start fp32 addition is order-free);
        without it the two tied gradients are returned separately like the
        reference.
        Returns (g_in, grads, {"Vi", "Vo"}, loss)."""
        if isinstance(slot.arena, list):
            return self._backward_blocks(slot, grad_out, stale_mode, train, g_in, emb, live_step, after_head,
                                         before_embedding, vo_overwrite)
        arena = slot.arena
        B, T = arena.B, arena.T
        Nt, d = B * T, self.d
        if stale_mode == "snapshot":
            wstep = slot.step
            for st in self.storage:
                st.weights(wstep)  # raises ScheduleViolation when evicted
        elif stale_mode == "current":
            wstep = live_step if live_step is not None else self.last_forward_step
            self._run_forward(wstep, arena, slot.layer_seeds, train, None, self.ws_bwd, live=False)
        else:
            raise ValueError(f"unknown stale_weights mode {stale_mode!r}")
        ws = self.ws_bwd
        tied_out = {"Vi": None, "Vo": None}
        if emb is None:
            emb_alpha, emb_beta = 1.0, 1.0
            vo_buf = vi_buf = None
            if self.has_projection:
                vo_buf = self._tied_buf()
            if self.has_embedding:
                vi_buf = self._tied_buf()
            tied_out = {"Vi": vi_buf, "Vo": vo_buf}
        else:
            emb_alpha, emb_beta, emb_grad = emb
            vo_buf = emb_grad if emb_alpha else None
            vi_buf = emb_grad if emb_beta else None
        loss = None
        g = None
        if self.has_projection:
            g = ws.get("g_stream_a", (Nt, d), torch.float32)
            if arena.adaptive is not None:
                Gp = self.storage[-1].G
                arena.adaptive.backward(g, vo_buf, Gp["cluster_weight"], Gp["cluster_bias"], alpha=emb_alpha,
                                        accumulate=emb is not None and not vo_overwrite)
            else:
                LY.head_backward(arena.acts[-1], self.tied.compute, arena.targets, self.vocab, arena.head, g, vo_buf,
                                 emb_alpha, ws, vo_accumulate=emb is not None and not vo_overwrite)
            loss = arena.head.loss
            if after_head is not None:
                after_head()  # the tied gradient's output half is complete
        else:
            if grad_out is None:
                raise ScheduleViolation(f"module {self.index} missing boundary gradient")
            g = grad_out.reshape(Nt, d)
        ping = 0
        for j in range(self.n_blocks - 1, -1, -1):
            off = self.block_idx[j]
            st = self.storage[off]
            W = st.weights(wstep)
            drop = LY.Dropout.make(slot.layer_seeds[off], self.layers[off].dropout_p, train)
            first = j == 0 and not self.has_embedding
            if first and g_in is not None:
                g_next = g_in.reshape(Nt, d)
            else:
                g_next = ws.get("g_stream_b" if ping == 0 else "g_stream_a", (Nt, d), torch.float32)
                ping ^= 1
            if self.layers[off].kind == "xl_block":
                tp = arena.tapes[j]
                xl_block_backward(W, W, tp, self._sinusoid(tp), g, g_next, st.G, drop, ws)
            else:
                LY.block_backward(W, W, arena.acts[j], arena.tapes[j], g, g_next, st.G, B, T, drop, ws)
            g = g_next
        if self.has_embedding:
            if before_embedding is not None:
                before_embedding()  # e.g. order the tied-gradient scatter after the output half
            st = self.storage[0]
            drop = LY.Dropout.make(slot.layer_seeds[0], self.layers[0].dropout_p, train)
            LY.embed_backward(g, arena.tokens, self.layers[0].max_seq_len, st.G["pos"],
                              vi_buf, emb_beta, ws, drop)
            return None, self.grad_views, tied_out, loss
        if g_in is not None:
            if g.data_ptr() != g_in.data_ptr():
                g_in.reshape(Nt, d).copy_(g)
            return g_in, self.grad_views, tied_out, loss
        return g.clone().view(B, T, d), self.grad_views, tied_out, loss

    def _tied_buf(self):
        """A zeroed fp32 [vocab, d] gradient in the tied matrix's row layout."""
        return self.tied.rows(torch.zeros_like(self.tied.flat_grad))

    def zero_grads(self):
        for st in self.storage:
            st.grad.zero_()
        return self.grad_views

    def _scratch_grads(self, st):
        """A second gradient buffer of the layer (row blocks j > 0 write here,
        then it is added onto st.grad)."""
        if getattr(st, "_gscratch", None) is None or st._gscratch.numel() != st.grad.numel():
            st._gscratch = torch.zeros_like(st.grad)  # pad columns stay zero
            st._Gscratch = st._carve(st._gscratch, torch.float32, torch.float32)
        return st._Gscratch

    def _backward_blocks(self, slot, grad_out, stale_mode, train, g_in, emb, live_step, after_head,
                         before_embedding, vo_overwrite):
        """Delayed backward of a micro-batched slot: row blocks j = 0..m-1 in
        order; block 0 writes every weight gradient, later blocks add theirs
        (rp_axpy) -- a fixed summation order, so concurrent == serial stays
        bitwise.  The tied gradient's output half accumulates over the blocks'
        head backwards (cross-entropy scale 1/(B*T) of the whole batch), the
        input half over their embedding scatters."""
        parts = slot.arena
        m = len(parts)
        Bm, T = parts[0].B, parts[0].T
        Nm, d = Bm * T, self.d
        rows_total = Nm * m
        if g_in is None and not self.has_embedding:
            g_in = torch.empty(rows_total, d, dtype=torch.float32, device=self.device)
        if stale_mode == "snapshot":
            wstep = slot.step
            for st in self.storage:
                st.weights(wstep)
        elif stale_mode == "current":
            wstep = live_step if live_step is not None else self.last_forward_step
            for j, a in enumerate(parts):
                self._run_forward(wstep, a, slot.layer_seeds, train, None, self.ws_bwd, live=False, part=(j, m))
        else:
            raise ValueError(f"unknown stale_weights mode {stale_mode!r}")
        ws = self.ws_bwd
        tied_out = {"Vi": None, "Vo": None}
        if emb is None:
            emb_alpha, emb_beta = 1.0, 1.0
            vo_buf = self._tied_buf() if self.has_projection else None
            vi_buf = self._tied_buf() if self.has_embedding else None
            tied_out = {"Vi": vi_buf, "Vo": vo_buf}
        else:
            emb_alpha, emb_beta, emb_grad = emb
            vo_buf = emb_grad if emb_alpha else None
            vi_buf = emb_grad if emb_beta else None
        for j, arena in enumerate(parts):
            r0, r1 = j * Nm, (j + 1) * Nm
            if self.has_projection:
                g = ws.get("g_stream_a", (Nm, d), torch.float32)
                LY.head_backward(arena.acts[-1], self.tied.compute, arena.targets, self.vocab, arena.head, g, vo_buf,
                                 emb_alpha, ws, vo_accumulate=(emb is not None and not vo_overwrite) or j > 0,
                                 rows_total=rows_total)
                if after_head is not None and j == m - 1:
                    after_head()
            else:
                if grad_out is None:
                    raise ScheduleViolation(f"module {self.index} missing boundary gradient")
                g = grad_out.reshape(rows_total, d)[r0:r1]
            ping = 0
            for jb in range(self.n_blocks - 1, -1, -1):
                off = self.block_idx[jb]
                st = self.storage[off]
                W = st.weights(wstep)
                G = st.G if j == 0 else self._scratch_grads(st)
                drop = LY.Dropout.shift(LY.Dropout.make(slot.layer_seeds[off], self.layers[off].dropout_p, train),
                                        r0 * d)
                first = jb == 0 and not self.has_embedding
                if first and g_in is not None:
                    g_next = g_in.reshape(rows_total, d)[r0:r1]
                else:
                    g_next = ws.get("g_stream_b" if ping == 0 else "g_stream_a", (Nm, d), torch.float32)
                    ping ^= 1
                if self.layers[off].kind == "xl_block":
                    tp = arena.tapes[jb]
                    xl_block_backward(W, W, tp, self._sinusoid(tp), g, g_next, G, drop, ws, rows_total=rows_total)
                else:
                    LY.block_backward(W, W, arena.acts[jb], arena.tapes[jb], g, g_next, G, Bm, T, drop, ws,
                                      rows_total=rows_total)
                if j > 0:
                    ops.axpy(st.grad, st._gscratch)
                g = g_next
            if self.has_embedding:
                if before_embedding is not None and j == 0:
                    before_embedding()
                st = self.storage[0]
                G = st.G if j == 0 else self._scratch_grads(st)
                drop = LY.Dropout.shift(LY.Dropout.make(slot.layer_seeds[0], self.layers[0].dropout_p, train),
                                        r0 * d)
                LY.embed_backward(g, arena.tokens, self.layers[0].max_seq_len, G["pos"], vi_buf, emb_beta, ws, drop)
                if j > 0:
                    ops.axpy(st.grad, st._gscratch)
            elif g_in is not None:
                dst = g_in.reshape(rows_total, d)[r0:r1]
                if g.data_ptr() != dst.data_ptr():
                    dst.copy_(g)
        loss = self._combined_loss(parts) if self.has_projection else None
        if self.has_embedding:
            return None, self.grad_views, tied_out, loss
        return g_in, self.grad_views, tied_out, loss


def build_modules(stack, part, dropout_seed):
    modules = []
    for k, (lo, hi) in enumerate(part.groups, start=1):
        modules.append(ModuleState(k, part.k, (lo, hi), stack.layers[lo:hi], stack.params[lo:hi], dropout_seed,
                                   storage=stack.storage[lo:hi], tied=stack.tied_store, runtime=stack.runtime,
                                   cdtype=stack.cdtype))
    return modules
