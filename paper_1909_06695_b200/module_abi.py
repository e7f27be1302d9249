"""A pipeline module driven through the module-level C ABI
(`rp_module_forward` / `rp_module_backward`, include/ringpipe_b200.h), for
the reference block and the Transformer-XL block (the host keeps the XL
segment memory: it loads each block's memory rows into the slot's tapes
before the forward and stores the new memory after it, as the Python module
does around its per-block calls).

The engines use the per-layer host loop in model.py (it carries the XL
blocks and the profiling spans); this is the two-calls-per-step form a
non-Python host binds.  Both issue the same kernels in the same order, so
their results are bitwise identical (tests/test_module_abi_gpu.py).
"""

import ctypes

import torch

from . import _native as N
from . import layers as LY
from . import ops
from .rng import keep_threshold


def _arr(ctype, items):
    a = (ctype * max(1, len(items)))()
    for i, x in enumerate(items):
        a[i] = x
    return a


def _is_xl(module):
    kinds = {module.layers[off].kind for off in module.block_idx}
    if len(kinds) > 1:
        raise ValueError("the module-level C ABI takes one block kind per module")
    return kinds == {"xl_block"}


def describe(module, B, T, seeds, train, max_ctas=0, arena=None):
    """(rp_module_desc, keep-alive objects) for one call."""
    dsc = N.ModuleDesc()
    if _is_xl(module):
        from . import xl as XD

        layer = module.layers[module.block_idx[0]]
        dsc.n_heads, dsc.M = layer.n_heads, layer.mem_len
        if arena is not None and arena.tapes:
            tp = arena.tapes[0]
            dsc.mem_len, dsc.xl_fused = tp.mem_len, XD.fused_flags(tp)
        dsc.score_tile = XD.SCORE_TILE
    dsc.B, dsc.T, dsc.d, dsc.f = B, T, module.d, module.f
    dsc.vocab = module.vocab or 0
    dsc.t_max = module.layers[0].max_seq_len if module.has_embedding else 0
    dsc.n_blocks = module.n_blocks
    dsc.has_embedding, dsc.has_projection = int(module.has_embedding), int(module.has_projection)
    dsc.dtype = N.BF16 if module.cdtype == torch.bfloat16 else N.F32
    dsc.max_ctas = max_ctas
    acts = {module.layers[off].activation for off in module.block_idx}
    if len(acts) > 1:
        raise ValueError("the module-level C ABI takes one FFN activation per module")
    dsc.activation = N.ACT_GELU if acts == {"gelu"} else N.ACT_RELU
    p = module.dropout_p
    if train and p > 0.0:
        dsc.drop_enabled, dsc.drop_threshold, dsc.drop_scale = 1, keep_threshold(p), 1.0 / (1.0 - p)
    seeds_arr = _arr(ctypes.c_uint64, [int(s) for s in seeds])
    dsc.layer_seeds = ctypes.cast(seeds_arr, ctypes.POINTER(ctypes.c_uint64))
    return dsc, [seeds_arr]


def _weights(module, wstep, arena=None):
    w = N.ModuleWeights()
    keep = []
    if _is_xl(module):
        from . import xl as XD

        xb = _arr(N.XlBlockWeights, [XD.xl_weights(module.storage[off].weights(wstep)) for off in module.block_idx])
        w.xl_blocks = ctypes.cast(xb, ctypes.POINTER(N.XlBlockWeights))
        R = module._sinusoid(arena.tapes[0])
        w.R = R.data_ptr()
        keep += [xb, R]
        blocks = _arr(N.BlockWeights, [])
    else:
        blocks = _arr(N.BlockWeights, [LY._weights(module.storage[off].weights(wstep)) for off in module.block_idx])
    w.blocks = ctypes.cast(blocks, ctypes.POINTER(N.BlockWeights))
    w.tied = module.tied.compute.data_ptr() if module.tied is not None else None
    if module.has_embedding:
        w.pos = module.storage[0].weights(wstep)["pos"].data_ptr()
    return w, [blocks] + keep


def _slot(arena):
    from . import xl as XD

    acts = _arr(ctypes.c_void_p, [a.data_ptr() for a in arena.acts])
    xl = bool(arena.tapes) and isinstance(arena.tapes[0], XD.XLTape)
    tapes = _arr(N.BlockTape, [] if xl else [LY._tape(tp) for tp in arena.tapes])
    xtapes = _arr(N.XlBlockTape, [XD.xl_tape(tp) for tp in arena.tapes] if xl else [])
    s = N.ModuleSlot()
    s.xl_tapes = ctypes.cast(xtapes, ctypes.POINTER(N.XlBlockTape))
    s.tokens = arena.tokens.data_ptr() if arena.tokens is not None else None
    s.targets = arena.targets.data_ptr() if arena.targets is not None else None
    s.acts = ctypes.cast(acts, ctypes.POINTER(ctypes.c_void_p))
    s.tapes = ctypes.cast(tapes, ctypes.POINTER(N.BlockTape))
    if arena.head is not None:
        s.lse, s.loss, s.loss64 = arena.head.lse.data_ptr(), arena.head.loss.data_ptr(), arena.head.loss64.data_ptr()
    return s, [acts, tapes, xtapes]


def workspace(module, B, T, seeds, train, cache, arena=None):
    dsc, keep = describe(module, B, T, seeds, train, arena=arena)
    nbytes = N.lib().rp_module_workspace_bytes(ctypes.byref(dsc))
    buf = cache.get("module_ws", (nbytes,), torch.uint8)
    return buf, nbytes


def forward(module, arena, wstep, seeds, train, out, ws, live=False):
    """ModuleState._run_forward over the module-level entry point.  live: the
    step's own forward of an XL module (load / advance the segment memory)."""
    B, T = arena.B, arena.T
    xl = _is_xl(module)
    if xl and live:
        for j, off in enumerate(module.block_idx):
            module._load_memory(off, arena.tapes[j])
    dsc, k1 = describe(module, B, T, seeds, train, LY.CTA_BUDGET["value"], arena)
    w, k2 = _weights(module, wstep, arena)
    s, k3 = _slot(arena)
    buf, nbytes = workspace(module, B, T, seeds, train, ws, arena)
    ops._count(1)
    N.check(N.lib().rp_module_forward(ctypes.byref(dsc), ctypes.byref(w), ctypes.byref(s),
                                      out.data_ptr() if out is not None else None, buf.data_ptr(), nbytes,
                                      module.flag.data_ptr(), ops._stream()), "module_forward")
    if xl and live:
        for j, off in enumerate(module.block_idx):
            module._store_memory(off, arena.tapes[j])
        module.mem_len = arena.tapes[0].M
    return arena.head.loss if module.has_projection else out


def backward(module, arena, wstep, seeds, train, g_out, g_in, tied_grad, alpha, beta, accumulate, ws):
    """ModuleState.recompute_backward (snapshot mode) over the module-level entry point."""
    from . import xl as XD

    B, T = arena.B, arena.T
    xl = _is_xl(module)
    dsc, k1 = describe(module, B, T, seeds, train, LY.CTA_BUDGET["value"], arena)
    w, k2 = _weights(module, wstep, arena)
    s, k3 = _slot(arena)
    gs = _arr(N.BlockGrads, [] if xl else [_grads(module.storage[off].G) for off in module.block_idx])
    xgs = _arr(N.XlBlockGrads, [XD.xl_grads(module.storage[off].G) for off in module.block_idx] if xl else [])
    G = N.ModuleGrads()
    G.blocks = ctypes.cast(gs, ctypes.POINTER(N.BlockGrads))
    G.xl_blocks = ctypes.cast(xgs, ctypes.POINTER(N.XlBlockGrads))
    if module.has_embedding:
        G.pos = module.storage[0].G["pos"].data_ptr()
    G.tied = tied_grad.data_ptr() if tied_grad is not None else None
    G.tied_alpha, G.tied_beta, G.tied_accumulate = alpha, beta, int(accumulate)
    buf, nbytes = workspace(module, B, T, seeds, train, ws, arena)
    ops._count(1)
    N.check(N.lib().rp_module_backward(ctypes.byref(dsc), ctypes.byref(w), ctypes.byref(s),
                                       g_out.data_ptr() if g_out is not None else None,
                                       g_in.data_ptr() if g_in is not None else None, ctypes.byref(G),
                                       buf.data_ptr(), nbytes, ops._stream()), "module_backward")


def _grads(G):
    g = N.BlockGrads()
    for n in ("wqkv", "wo", "w1", "w2", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "b1", "b2"):
        setattr(g, n, G[n].data_ptr())
    return g
