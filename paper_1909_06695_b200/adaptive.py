"""Adaptive tied softmax head on the device (BASELINE
configs[3] trains WikiText-103 with it).  Restated in oracle/adaptive.py
(Grave et al. 2017 as Transformer-XL's ProjectedAdaptiveLogSoftmax with
div_val = 1 and tied output layers); the reference has no adaptive softmax,
so parity is pinned through that restatement.

Every contraction is the tcgen05 head GEMM with its fused epilogues (online
log-sum-exp partials + target logit, then the softmax-CE gradient written
once): one head problem over all N rows against [V[:c0]; W_c] -- the cluster
bias rides in as an extra K column ([h | 1] . [W | b]^T) -- and one tail
problem per cluster over the rows whose target falls in it, against the tied
rows V[c_k:c_{k+1}].  csrc/adaptive.cu gathers / scatters the cluster rows.
The cluster row lists come from the host targets (the batch the caller hands
to the step), like the data loader's bucketing; a device-only target tensor
costs one D2H copy.
"""

import numpy as np
import torch

from . import _native as N
from . import ops
from .errors import DimensionError
from . import layers as LY
from .layers import _pad8


def clusters(cutoffs, vocab):
    """Tail clusters [(c_k, c_{k+1})] for cutoffs [c_0, ..., c_{n-1}] (oracle/adaptive.clusters)."""
    edges = list(cutoffs) + [vocab]
    return [(edges[k], edges[k + 1]) for k in range(len(cutoffs)) if edges[k] < edges[k + 1]]


class HostCopy:
    """A device int64 tensor copied to pinned host memory on a side stream,
    ordered after the current stream's work so far: the adaptive head's row
    bucketing waits for this copy only, not for the whole stream (device
    batches; host batches are bucketed from the caller's array directly)."""

    _streams = {}

    def __init__(self, t):
        dev = t.device
        st = HostCopy._streams.get(dev)
        if st is None:
            st = HostCopy._streams[dev] = torch.cuda.Stream(device=dev)
        self.host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(dev))
        st.wait_event(ready)
        with torch.cuda.stream(st):
            self.host.copy_(t, non_blocking=True)
            self.done = torch.cuda.Event()
            self.done.record(st)
        t.record_stream(st)

    def numpy(self):
        self.done.synchronize()
        return self.host.numpy()


class AdaptiveHead:
    """Forward (loss) and backward (grad of the input rows, of the tied
    matrix, of the cluster weights / biases) of the adaptive tied softmax."""

    def __init__(self, vocab, d, cutoffs, device, dtype=torch.bfloat16):
        if not cutoffs or cutoffs[0] <= 0 or any(b <= a for a, b in zip(cutoffs, cutoffs[1:])) or cutoffs[-1] > vocab:
            raise DimensionError(f"adaptive softmax: bad cutoffs {cutoffs} for vocab {vocab}")
        if cutoffs[0] % 8:
            raise DimensionError("adaptive softmax: the head size c_0 must be a multiple of 8 (TMA 16-byte rows)")
        self.vocab, self.d, self.cutoffs, self.device, self.dtype = vocab, d, list(cutoffs), device, dtype
        self.tails = clusters(cutoffs, vocab)
        self.n = len(self.tails)
        self.c0 = cutoffs[0]
        self.vh = self.c0 + self.n  # head classes
        self.da = _pad8(d + 1)      # [h | 1 | 0..] width
        self.ws = {}

    def _buf(self, name, shape, dtype):
        t = self.ws.get(name)
        if t is None or t.shape != torch.Size(shape) or t.dtype != dtype:
            t = self.ws[name] = torch.empty(shape, dtype=dtype, device=self.device)
        return t

    def _lse(self, x, w, targets, vocab, tag, flag):
        rows = x.shape[0]
        nt = (vocab + ops.gemm_tile_n(vocab, rows) - 1) // ops.gemm_tile_n(vocab, rows)
        partial = self._buf(f"{tag}_partial", (rows, 2 * nt, 2), torch.float32)
        zy = self._buf(f"{tag}_zy", (rows,), torch.float32)
        lse = self._buf(f"{tag}_lse", (rows,), torch.float32)
        rloss = self._buf(f"{tag}_rows", (rows,), torch.float32)
        loss = self._buf(f"{tag}_loss", (), torch.float32)
        ops.gemm(x, w, epilogue=N.EPI_LSE_PARTIAL, targets=targets, partial=partial, target_logit=zy)
        ops.ce_finish(partial, zy, targets, vocab, lse, rloss, loss, None, flag)
        return lse, loss

    def forward(self, h, tied_c, w_c, b_c, targets, flag=None):
        """h [N, d] (compute dtype), tied_c [V, d] (compute copy), w_c [n, d],
        b_c [n] fp32 masters, targets: host int64 [N] (or a device tensor).
        Returns the mean loss as a 0-d device tensor."""
        Nr, d = h.shape
        if d != self.d or tied_c.shape != (self.vocab, d) or w_c.shape != (self.n, d) or b_c.shape != (self.n,):
            raise DimensionError("adaptive softmax: shape mismatch")
        if isinstance(targets, HostCopy):
            y = targets.numpy()
        else:
            y = targets.detach().cpu().numpy() if torch.is_tensor(targets) else np.asarray(targets)
        y = y.reshape(-1).astype(np.int64)
        if y.size != Nr or (y.size and (y.min() < 0 or y.max() >= self.vocab)):
            raise DimensionError("adaptive softmax: targets out of range")
        cdt = self.dtype
        self.h = h
        self.tied_c = tied_c
        # [h | 1] and [V[:c0] ; W_c | b_c]: the cluster bias is one more K column
        self.h_aug = self._buf("h_aug", (Nr, self.da), cdt)
        ops.rows_copy(h, self.h_aug, val_const=1.0, aug=True)
        self.w_aug = self._buf("w_aug", (self.vh, self.da), cdt)
        ops.rows_copy(tied_c[: self.c0], self.w_aug[: self.c0], aug=True, val_const=0.0)
        if self.n:
            ops.rows_copy(w_c, self.w_aug[self.c0:], val=b_c, aug=True)
        yh = y.copy()
        self.rows = []
        for k, (lo, hi) in enumerate(self.tails):
            sel = np.nonzero((y >= lo) & (y < hi))[0]
            yh[sel] = self.c0 + k
            self.rows.append(sel)
        dev = self.device
        self.y_head = torch.from_numpy(yh).to(dev, non_blocking=True)
        lse_h, loss_h = self._lse(self.h_aug, self.w_aug, self.y_head, self.vh, "head", flag)
        self.lse_h = lse_h
        total = loss_h.clone()
        self.tail_state = []
        for k, (lo, hi) in enumerate(self.tails):
            sel = self.rows[k]
            if sel.size == 0:
                self.tail_state.append(None)
                continue
            idx = torch.from_numpy(sel).to(dev, non_blocking=True)
            yk = torch.from_numpy(y[sel] - lo).to(dev, non_blocking=True)
            hk = self._buf(f"h{k}", (sel.size, LY.pad_cols(d, cdt)), cdt)[:, :d]
            ops.rows_gather(h, idx, hk)
            lse_k, loss_k = self._lse(hk, tied_c[lo:hi], yk, hi - lo, f"t{k}", flag)
            total += loss_k * (sel.size / Nr)
            self.tail_state.append((idx, yk, hk, lse_k))
        self.N = Nr
        return total

    def backward(self, g_h, g_tied, g_wc, g_bc, alpha=1.0, accumulate=False):
        """g_h [N, d] fp32 (written), g_tied [V, d] fp32: alpha x the output
        half of the tied gradient, written or (accumulate) added; g_wc [n, d],
        g_bc [n] fp32 (written).  g_tied may be None (no tied gradient)."""
        Nr, d, cdt = self.N, self.d, self.dtype
        scale = 1.0 / Nr
        dz = self._buf("dz_h", (Nr, _pad8(self.vh)), cdt)[:, : self.vh]
        ops.gemm(self.h_aug, self.w_aug, epilogue=N.EPI_CE_GRAD, targets=self.y_head, lse=self.lse_h, ce_scale=scale,
                 out=dz)
        g_aug = self._buf("gh_aug", (Nr, self.da), torch.float32)
        ops.gemm(dz, self.w_aug, b_mn=True, out=g_aug)
        ops.rows_copy(g_aug, g_h, cols=d)
        def tied_out(a, b, rows_out):
            # rows_out (+)= alpha * a^T b  (the head GEMM's fused residual add accumulates)
            if accumulate:
                ops.gemm(a, b, a_mn=True, b_mn=True, out=rows_out, alpha=alpha, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL,
                         residual=rows_out)
            else:
                ops.gemm(a, b, a_mn=True, b_mn=True, out=rows_out, alpha=alpha)

        if g_tied is not None:
            tied_out(dz[:, : self.c0], self.h, g_tied[: self.c0])
        if self.n:
            gw = self._buf("gw_aug", (self.n, self.da), torch.float32)
            ops.gemm(dz[:, self.c0:], self.h_aug, a_mn=True, b_mn=True, out=gw)
            ops.rows_copy(gw, g_wc, cols=d)
            ops.rows_copy(gw[:, d:], g_bc.view(self.n, 1), cols=1)
        for k, (lo, hi) in enumerate(self.tails):
            st = self.tail_state[k]
            if st is None:
                if g_tied is not None and not accumulate:
                    g_tied[lo:hi].zero_()
                continue
            idx, yk, hk, lse_k = st
            nk = idx.numel()
            dzk = self._buf(f"dz{k}", (nk, _pad8(hi - lo)), cdt)[:, : hi - lo]
            ops.gemm(hk, self.tied_c[lo:hi], epilogue=N.EPI_CE_GRAD, targets=yk, lse=lse_k, ce_scale=scale, out=dzk)
            ghk = self._buf(f"gh{k}", (nk, d), torch.float32)
            ops.gemm(dzk, self.tied_c[lo:hi], b_mn=True, out=ghk)
            ops.rows_scatter_add(ghk, idx, g_h)
            if g_tied is not None:
                tied_out(dzk, hk, g_tied[lo:hi])
