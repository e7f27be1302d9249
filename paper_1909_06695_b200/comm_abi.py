"""Host wrappers of the C ABI's distributed context and state entries
(include/ringpipe_b200.h: rp_ctx_create / rp_send / rp_recv / rp_group_*,
rp_export_state / rp_import_state).

These are the calls a non-Python host binds (INTEGRATION.md shows the C and
ctypes forms); the Python engines use torch.distributed for the same
transfers (distributed.py).  `export_state` / `import_state` move named
device or host buffers to and from the reference's RPCK checkpoint container
(checkpoint.py:1-70) in memory.
"""

import ctypes

import numpy as np
import torch

from . import _native as N

I64, U64, F64 = 2, 3, 4
_DT = {torch.float32: N.F32, torch.bfloat16: N.BF16, torch.int64: I64, torch.uint64: U64, torch.float64: F64}
_NP = {np.dtype("float32"): N.F32, np.dtype("int64"): I64, np.dtype("uint64"): U64, np.dtype("float64"): F64}


def _entries(named):
    """[(name, tensor | ndarray)] -> (ctypes array of rp_state_entry, keep-alive)."""
    arr = (N.StateEntry * max(1, len(named)))()
    keep = []
    for i, (name, t) in enumerate(named):
        e = arr[i]
        key = name.encode("utf-8")
        keep.append(key)
        e.name = key
        if torch.is_tensor(t):
            if not t.is_contiguous():
                raise ValueError(f"state entry {name!r} must be contiguous")
            e.ptr, e.dtype, e.on_host = t.data_ptr(), _DT[t.dtype], int(not t.is_cuda)
            shape = tuple(t.shape)
        else:
            a = np.ascontiguousarray(t)
            keep.append(a)
            if a.dtype == np.uint16:  # raw bf16 bits on the host
                e.dtype = N.BF16
            else:
                e.dtype = _NP[a.dtype]
            e.ptr, e.on_host = a.ctypes.data, 1
            shape = a.shape
        if len(shape) > 4:
            raise ValueError(f"state entry {name!r}: at most 4 dims")
        e.ndim = len(shape)
        for k, s in enumerate(shape):
            e.shape[k] = s
    return arr, keep


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream) if torch.cuda.is_available() else None


def export_state(named):
    """Named buffers -> RPCK container bytes (rp_export_state)."""
    named = list(named.items()) if isinstance(named, dict) else list(named)
    arr, _keep = _entries(named)
    n = N.lib().rp_state_bytes(arr, len(named))
    if n < 0:
        raise ValueError(N.last_error())
    blob = ctypes.create_string_buffer(n)
    N.check(N.lib().rp_export_state(arr, len(named), blob, n, _stream()), "rp_export_state")
    return blob.raw


def import_state(named, blob):
    """RPCK container bytes -> the named buffers, in place (rp_import_state)."""
    named = list(named.items()) if isinstance(named, dict) else list(named)
    arr, _keep = _entries(named)
    buf = ctypes.create_string_buffer(bytes(blob), len(blob))
    N.check(N.lib().rp_import_state(arr, len(named), buf, len(blob), _stream()), "rp_import_state")


class NcclContext:
    """rp_ctx: one NCCL communicator over the ranks of the node."""

    @staticmethod
    def unique_id():
        buf = ctypes.create_string_buffer(128)
        N.check(N.lib().rp_nccl_unique_id(buf), "rp_nccl_unique_id")
        return buf.raw

    def __init__(self, device, uid, rank, nranks):
        self._h = ctypes.c_void_p()
        N.check(N.lib().rp_ctx_create(device, ctypes.create_string_buffer(uid, 128), rank, nranks,
                                      ctypes.byref(self._h)), "rp_ctx_create")
        self.rank, self.nranks = N.lib().rp_ctx_rank(self._h), N.lib().rp_ctx_nranks(self._h)

    def send(self, t, peer):
        N.check(N.lib().rp_send(self._h, t.data_ptr(), t.numel() * t.element_size(), peer, _stream()), "rp_send")

    def recv(self, t, peer):
        N.check(N.lib().rp_recv(self._h, t.data_ptr(), t.numel() * t.element_size(), peer, _stream()), "rp_recv")

    @staticmethod
    def group_start():
        N.check(N.lib().rp_group_start(), "rp_group_start")

    @staticmethod
    def group_end():
        N.check(N.lib().rp_group_end(), "rp_group_end")

    def close(self):
        if self._h:
            N.check(N.lib().rp_ctx_destroy(self._h), "rp_ctx_destroy")
            self._h = ctypes.c_void_p()
