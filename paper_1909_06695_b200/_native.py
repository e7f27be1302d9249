"""ctypes binding of libringpipe_b200.so (include/ringpipe_b200.h).

Loading is strict: there is no CPU fallback.  If the library is missing or
was built for another architecture, importing the product path raises.
"""

import ctypes
import os

from .errors import raise_for_status

_LIB_PATH = os.environ.get("RP_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                           "libringpipe_b200.so")
_lib = None

# rp_dtype / rp_math / rp_epilogue (include/ringpipe_b200.h)
F32, BF16 = 0, 1
MATH_BF16, MATH_TF32, MATH_TF32X3 = 0, 1, 2
EPI_STORE, EPI_BIAS_RELU, EPI_BIAS_DROPOUT_RESIDUAL, EPI_LSE_PARTIAL, EPI_CE_GRAD, EPI_RELU_GRAD, EPI_GELU_GRAD = range(7)
ACT_RELU, ACT_GELU = 0, 1
FLAG_NONFINITE, FLAG_DIMENSION = 1, 2


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("math", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("a_mn_major", ctypes.c_int32),
        ("b_mn_major", ctypes.c_int32),
        ("M", ctypes.c_int64),
        ("N", ctypes.c_int64),
        ("K", ctypes.c_int64),
        ("batch", ctypes.c_int64),
        ("A", ctypes.c_void_p),
        ("A_lo", ctypes.c_void_p),
        ("lda", ctypes.c_int64),
        ("stride_a", ctypes.c_int64),
        ("B", ctypes.c_void_p),
        ("B_lo", ctypes.c_void_p),
        ("ldb", ctypes.c_int64),
        ("stride_b", ctypes.c_int64),
        ("C", ctypes.c_void_p),
        ("ldc", ctypes.c_int64),
        ("stride_c", ctypes.c_int64),
        ("epilogue", ctypes.c_int32),
        ("tile_n", ctypes.c_int32),
        ("alpha", ctypes.c_float),
        ("bias", ctypes.c_void_p),
        ("residual", ctypes.c_void_p),
        ("ld_residual", ctypes.c_int64),
        ("stride_residual", ctypes.c_int64),
        ("drop_enabled", ctypes.c_int32),
        ("drop_scale", ctypes.c_float),
        ("drop_seed", ctypes.c_uint64),
        ("drop_threshold", ctypes.c_uint64),
        ("drop_pos0", ctypes.c_uint64),
        ("targets", ctypes.c_void_p),
        ("lse", ctypes.c_void_p),
        ("partial", ctypes.c_void_p),
        ("target_logit", ctypes.c_void_p),
        ("ce_scale", ctypes.c_float),
        ("k_splits", ctypes.c_int32),
        ("max_ctas", ctypes.c_int32),
        ("k_lo_sign", ctypes.c_int32),
        ("k_lo_off", ctypes.c_int64),
    ]


class BlockDesc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("T", ctypes.c_int64), ("d", ctypes.c_int64), ("f", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("drop_enabled", ctypes.c_int32), ("drop_seed", ctypes.c_uint64),
                ("drop_threshold", ctypes.c_uint64), ("drop_scale", ctypes.c_float), ("max_ctas", ctypes.c_int32),
                ("drop_rows_total", ctypes.c_int64), ("activation", ctypes.c_int32)]


class BlockWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("wqkv", "wo", "w1", "w2", "ln1_g", "ln1_b", "ln2_g", "ln2_b",
                                                 "b1", "b2")]


class BlockTape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("a", "qkv", "probs", "ctx", "x1", "m", "h1", "mean1", "rstd1",
                                                 "mean2", "rstd2", "z1")]


class BlockGrads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("wqkv", "wo", "w1", "w2", "ln1_g", "ln1_b", "ln2_g", "ln2_b",
                                                 "b1", "b2")]


class HeadDesc(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("d", ctypes.c_int64), ("vocab", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("rows_total", ctypes.c_int64)]


class ModuleDesc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("T", ctypes.c_int64), ("d", ctypes.c_int64), ("f", ctypes.c_int64),
                ("vocab", ctypes.c_int64), ("t_max", ctypes.c_int64), ("n_blocks", ctypes.c_int32),
                ("has_embedding", ctypes.c_int32), ("has_projection", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("max_ctas", ctypes.c_int32), ("drop_enabled", ctypes.c_int32), ("drop_threshold", ctypes.c_uint64),
                ("drop_scale", ctypes.c_float), ("layer_seeds", ctypes.POINTER(ctypes.c_uint64)),
                ("activation", ctypes.c_int32), ("n_heads", ctypes.c_int32), ("mem_len", ctypes.c_int32),
                ("M", ctypes.c_int64), ("xl_fused", ctypes.c_int32), ("score_tile", ctypes.c_int32)]


XL_FUSED_FWD, XL_FUSED_BWD, XL_FUSED_PV, XL_FUSED_DQ, XL_BANDED, XL_FUSED_KV = 1, 2, 4, 8, 16, 32


class XlBlockDesc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("T", ctypes.c_int64), ("M", ctypes.c_int64), ("d", ctypes.c_int64),
                ("f", ctypes.c_int64), ("H", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("drop_enabled", ctypes.c_int32), ("activation", ctypes.c_int32), ("max_ctas", ctypes.c_int32),
                ("mem_len", ctypes.c_int32), ("drop_seed", ctypes.c_uint64), ("drop_threshold", ctypes.c_uint64),
                ("drop_scale", ctypes.c_float), ("drop_rows_total", ctypes.c_int64), ("ldk", ctypes.c_int64),
                ("fused", ctypes.c_int32), ("score_tile", ctypes.c_int32)]


XL_W_MATS = ("wqkv", "wo", "w1", "w2", "wr")
XL_W_VECS = ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "b1", "b2", "r_w_bias", "r_r_bias")


class XlBlockWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in XL_W_MATS + XL_W_VECS]


XL_TAPE = ("xa", "a", "qkv", "qu", "qv", "kh", "vh", "rh", "probs", "ctx", "x1", "m", "h1", "z1", "mean1", "rstd1",
           "mean2", "rstd2")


class XlBlockTape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in XL_TAPE]


class XlBlockGrads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("wqkv", "wo", "w1", "w2", "wr", "ln1_g", "ln1_b", "ln2_g", "ln2_b",
                                                 "b1", "b2", "r_w_bias", "r_r_bias")]


class ModuleWeights(ctypes.Structure):
    _fields_ = [("blocks", ctypes.POINTER(BlockWeights)), ("tied", ctypes.c_void_p), ("pos", ctypes.c_void_p),
                ("xl_blocks", ctypes.POINTER(XlBlockWeights)), ("R", ctypes.c_void_p)]


class ModuleSlot(ctypes.Structure):
    _fields_ = [("tokens", ctypes.c_void_p), ("targets", ctypes.c_void_p), ("acts", ctypes.POINTER(ctypes.c_void_p)),
                ("tapes", ctypes.POINTER(BlockTape)), ("lse", ctypes.c_void_p), ("loss", ctypes.c_void_p),
                ("loss64", ctypes.c_void_p), ("xl_tapes", ctypes.POINTER(XlBlockTape))]


class ModuleGrads(ctypes.Structure):
    _fields_ = [("blocks", ctypes.POINTER(BlockGrads)), ("pos", ctypes.c_void_p), ("tied", ctypes.c_void_p),
                ("tied_alpha", ctypes.c_float), ("tied_beta", ctypes.c_float), ("tied_accumulate", ctypes.c_int32),
                ("xl_blocks", ctypes.POINTER(XlBlockGrads))]


def lib():
    """The loaded library; raises ImportError when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(
                f"{_LIB_PATH} not built; run `python -m paper_1909_06695_b200.build` "
                "(there is no CPU fallback)"
            )
        _lib = ctypes.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class StateEntry(ctypes.Structure):
    """rp_state_entry (include/ringpipe_b200.h)."""

    _fields_ = [("name", ctypes.c_char_p), ("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32),
                ("on_host", ctypes.c_int32), ("ndim", ctypes.c_int32), ("shape", ctypes.c_int64 * 4)]


def _declare(L):
    vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
    f32, f64 = ctypes.c_float, ctypes.c_double
    sig = {
        "rp_last_error": [ctypes.c_char_p, ctypes.c_size_t],
        "rp_gemm": [ctypes.POINTER(GemmArgs), vp],
        "rp_gemm_tile_n": [i64, i64, i64],
        "rp_gemm_choose_splits": [i64, i64, i64, i64, i64],
        "rp_splitk_reduce": [vp, i32, i64, i64, vp, i64, vp],
        "rp_tf32_split": [vp, vp, vp, i64, i64, i64, i64, vp],
        "rp_layernorm_fwd": [i32, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp],
        "rp_layernorm_bwd": [i32, vp, vp, vp, vp, vp, vp, vp, vp, u64, u64, f32, i32, vp, vp, i64, i64, i64, i64, vp],
        "rp_layernorm_bwd_blocks": [i64],
        "rp_colsum_blocks": [i64],
        "rp_mask_grad_blocks": [i64, i64],
        "rp_colsum_partial": [i32, vp, i64, i64, i64, vp, vp],
        "rp_colsum_finish": [vp, i32, i64, vp, vp],
        "rp_colsum_finish_multi": [vp, vp, vp, vp, i32, vp],
        "rp_mask_grad": [i32, vp, vp, i64, i64, u64, u64, u64, f32, i32, vp, i64, vp],
        "rp_mask_grad_blocks_ld": [i64, i64, i64],
        "rp_softmax_causal": [i32, vp, vp, i64, i64, i64, vp],
        "rp_softmax_bwd": [i32, vp, vp, vp, f32, i64, i64, i64, vp],
        "rp_embed_fwd": [i32, vp, vp, vp, vp, i64, i64, i64, i64, u64, u64, f32, i32, vp, i64, vp],
        "rp_embed_bwd": [vp, vp, i64, i64, i64, i64, i64, u64, u64, f32, i32, vp, vp, f32, vp, i64, vp],
        "rp_embed_bwd_workspace_bytes": [i64, i64],
        "rp_ce_finish": [vp, i32, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp],
        "rp_adam_step": [vp, vp, vp, vp, vp, i32, i64, f32, f32, f32, f32, f32, f32, vp, vp],
        "rp_sgd_step": [vp, vp, vp, i32, i64, f32, vp, vp],
        "rp_init_uniform": [vp, i64, u64, u64, f64, vp],
        "rp_cast": [vp, i32, vp, i32, i64, vp],
        "rp_embedding_gradient": [i64, i64, vp, vp, vp, i64, i32, vp],
        "rp_sq_norm": [vp, i64, vp, vp, i32, vp],
        "rp_xl_split_qkv": [i32, vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i32, i32, i64, i64, vp],
        "rp_xl_split_heads": [i32, vp, i64, i32, vp, i64, i32, i32, i64, vp],
        "rp_xl_merge_heads": [i32, vp, i32, vp, i64, i64, i32, i32, i64, vp],
        "rp_xl_merge_grads": [i32, vp, vp, vp, vp, vp, i64, i64, i64, i32, i32, i64, i64, i64, vp],
        "rp_xl_softmax_fwd": [i32, vp, vp, i64, vp, i64, i64, i64, i64, i64, f32, vp],
        "rp_xl_attn_fwd": [vp, vp, vp, vp, vp, i64, i64, i64, i64, i32, i32, i64, f32, vp],
        "rp_xl_attn_bwd": [vp, vp, vp, vp, vp, i64, vp, vp, i64, i64, i64, i32, i32, i64, f32, vp],
        "rp_xl_softmax_bwd": [i32, vp, i64, vp, i64, vp, vp, i64, i64, i64, i64, f32, vp],
        "rp_xl_attn_fwd_pv": [vp, vp, vp, vp, vp, vp, i64, vp, i64, i64, i64, i32, i32, i64, f32, i32, i64, vp],
        "rp_xl_attn_bwd_dq": [vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, i64, i64, i64, i32, i32, i64, f32, vp,
                              vp, vp, vp],
        "rp_xl_attn_bwd_kv": [vp, vp, vp, vp, i64, vp, vp, vp, i64, i64, i64, i32, i32, i64, f32, vp, vp],
        "rp_xl_dq_persistent": [],
        "rp_xl_dq_bias_part_bytes": [i32, i64, i64],
        "rp_xl_dq_bias_finish": [vp, vp, vp, i32, i64, i64, vp],
        "rp_xl_bias_grad_workspace_bytes": [i32, i32],
        "rp_rows_copy": [i32, vp, i64, i64, i64, vp, f32, i32, i32, vp, i64, vp],
        "rp_rows_gather": [i32, vp, i64, vp, i64, i64, vp, i64, vp],
        "rp_rows_scatter_add": [vp, i64, vp, i64, i64, vp, i64, vp],
        "rp_xl_bias_grad": [vp, vp, vp, vp, vp, i32, i64, i32, i64, vp],
        "rp_module_workspace_bytes": [ctypes.POINTER(ModuleDesc)],
        "rp_module_forward": [ctypes.POINTER(ModuleDesc), ctypes.POINTER(ModuleWeights), ctypes.POINTER(ModuleSlot),
                              vp, vp, i64, vp, vp],
        "rp_module_backward": [ctypes.POINTER(ModuleDesc), ctypes.POINTER(ModuleWeights),
                               ctypes.POINTER(ModuleSlot), vp, vp, ctypes.POINTER(ModuleGrads), vp, i64, vp],
        "rp_xl_block_workspace_bytes": [ctypes.POINTER(XlBlockDesc)],
        "rp_xl_block_forward": [ctypes.POINTER(XlBlockDesc), ctypes.POINTER(XlBlockWeights), vp, vp,
                                ctypes.POINTER(XlBlockTape), vp, i64, vp, vp],
        "rp_xl_block_backward": [ctypes.POINTER(XlBlockDesc), ctypes.POINTER(XlBlockWeights), vp,
                                 ctypes.POINTER(XlBlockTape), vp, vp, ctypes.POINTER(XlBlockGrads), vp, i64, vp],
        "rp_block_workspace_bytes": [ctypes.POINTER(BlockDesc)],
        "rp_block_forward": [ctypes.POINTER(BlockDesc), ctypes.POINTER(BlockWeights), vp, vp,
                             ctypes.POINTER(BlockTape), vp, i64, vp, vp],
        "rp_block_backward": [ctypes.POINTER(BlockDesc), ctypes.POINTER(BlockWeights), vp,
                              ctypes.POINTER(BlockTape), vp, vp, ctypes.POINTER(BlockGrads), vp, i64, vp],
        "rp_head_workspace_bytes": [ctypes.POINTER(HeadDesc)],
        "rp_head_forward": [ctypes.POINTER(HeadDesc), vp, vp, vp, vp, vp, vp, vp, i64, vp, vp],
        "rp_head_backward": [ctypes.POINTER(HeadDesc), vp, vp, vp, vp, vp, vp, f32, i32, vp, i64, vp],
        "rp_axpy": [vp, vp, f32, i64, vp],
        "rp_gelu_fwd": [i32, vp, vp, i64, vp],
        "rp_nccl_unique_id": [vp],
        "rp_ctx_create": [i32, vp, i32, i32, ctypes.POINTER(vp)],
        "rp_ctx_destroy": [vp],
        "rp_ctx_rank": [vp],
        "rp_ctx_nranks": [vp],
        "rp_send": [vp, vp, i64, i32, vp],
        "rp_recv": [vp, vp, i64, i32, vp],
        "rp_group_start": [],
        "rp_group_end": [],
        "rp_state_bytes": [ctypes.POINTER(StateEntry), i32],
        "rp_export_state": [ctypes.POINTER(StateEntry), i32, vp, i64, vp],
        "rp_import_state": [ctypes.POINTER(StateEntry), i32, vp, i64, vp],
    }
    L.rp_version.restype = ctypes.c_char_p
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int32
    L.rp_embed_bwd_workspace_bytes.restype = i64
    L.rp_xl_bias_grad_workspace_bytes.restype = i64
    L.rp_xl_dq_bias_part_bytes.restype = i64
    L.rp_block_workspace_bytes.restype = i64
    L.rp_xl_block_workspace_bytes.restype = i64
    L.rp_module_workspace_bytes.restype = i64
    L.rp_head_workspace_bytes.restype = i64
    L.rp_state_bytes.restype = i64


def last_error():
    buf = ctypes.create_string_buffer(1024)
    lib().rp_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(status, what=""):
    if status != 0:
        raise_for_status(status, f"{what}: {last_error()}")


def exported_symbols():
    """Names declared in include/ringpipe_b200.h (for the load/export test)."""
    import re

    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ringpipe_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(rp_[a-z0-9_]+)\s*\(", text)))
