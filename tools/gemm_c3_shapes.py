"""Isolated timing of the 14 dense GEMMs of one Transformer-XL block at the
C3 shape (B 22, T = M = 512, d 512, d_ff 2048; bf16, CUDA-graph replay so
the host launch path is out of the measurement): which contractions hold
the block-GEMM family below the tensor peak."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import _native as N  # noqa: E402
from paper_1909_06695_b200 import ops  # noqa: E402
from paper_1909_06695_b200.rng import keep_threshold  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
if not os.environ.get("ONCE"):
    from gemm_shapes import bench  # noqa: E402

B, T, M, d, f = 22, 512, 512, 512, 2048
Nt, Nk = B * T, B * (M + T)
bf = torch.bfloat16
r = lambda *s, dt=bf: (torch.randn(*s, device="cuda") * 0.05).to(dt)  # noqa: E731
drop = (123, keep_threshold(0.1), 1 / 0.9, 0)
xa, wqkv, qkv = r(Nk, d), r(d, 3 * d), r(Nk, 3 * d)
R, wr, ctx, wo = r(M + T, d), r(d, d), r(Nt, d), r(d, d)
x, m, w1, w2, h1 = r(Nt, d), r(Nt, d), r(d, f), r(f, d), r(Nt, f)
g_h2, g_z1, g_proj, g_r, g_qkv = r(Nt, d), r(Nt, f), r(Nt, d), r(M + T, d), r(Nk, 3 * d)
b1, b2 = r(f, dt=torch.float32), r(d, dt=torch.float32)
o = {k: torch.empty(*s, device="cuda", dtype=dt) for k, s, dt in
     [("qkv", (Nk, 3 * d), bf), ("r", (M + T, d), bf), ("x1", (Nt, d), bf), ("h1", (Nt, f), bf), ("out", (Nt, d), bf),
      ("Gw2", (f, d), torch.float32), ("gz1", (Nt, f), bf), ("Gw1", (d, f), torch.float32),
      ("gm", (Nt, d), torch.float32), ("Gwo", (d, d), torch.float32), ("gctx", (Nt, d), bf),
      ("Gwr", (d, d), torch.float32), ("Gwqkv", (d, 3 * d), torch.float32), ("ga", (Nk, d), torch.float32)]}
cases = [
    ("QKV", Nk, 3 * d, d, lambda: ops.gemm(xa, wqkv, b_mn=True, out=o["qkv"])),
    ("R", M + T, d, d, lambda: ops.gemm(R, wr, b_mn=True, out=o["r"])),
    ("out-proj+drop", Nt, d, d, lambda: ops.gemm(ctx, wo, b_mn=True, out=o["x1"], epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL,
                                                 residual=x, dropout=drop)),
    ("FFN-up+relu", Nt, f, d, lambda: ops.gemm(m, w1, b_mn=True, out=o["h1"], epilogue=N.EPI_BIAS_RELU, bias=b1)),
    ("FFN-down+drop", Nt, d, f, lambda: ops.gemm(h1, w2, b_mn=True, out=o["out"], epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL,
                                                 bias=b2, residual=x, dropout=drop)),
    ("dW2 (splitK)", f, d, Nt, lambda: ops.gemm(h1, g_h2, a_mn=True, b_mn=True, out=o["Gw2"])),
    ("g_z1+relu'", Nt, f, d, lambda: ops.gemm(g_h2, w2, out=o["gz1"], epilogue=N.EPI_RELU_GRAD, residual=h1)),
    ("dW1 (splitK)", d, f, Nt, lambda: ops.gemm(m, g_z1, a_mn=True, b_mn=True, out=o["Gw1"])),
    ("g_m fp32", Nt, d, f, lambda: ops.gemm(g_z1, w1, out=o["gm"])),
    ("dWo (splitK)", d, d, Nt, lambda: ops.gemm(ctx, g_proj, a_mn=True, b_mn=True, out=o["Gwo"])),
    ("g_ctx", Nt, d, d, lambda: ops.gemm(g_proj, wo, out=o["gctx"])),
    ("dWr (splitK)", d, d, M + T, lambda: ops.gemm(R, g_r, a_mn=True, b_mn=True, out=o["Gwr"])),
    ("dWqkv (splitK)", d, 3 * d, Nk, lambda: ops.gemm(xa, g_qkv, a_mn=True, b_mn=True, out=o["Gwqkv"])),
    ("g_a fp32", Nk, d, 3 * d, lambda: ops.gemm(g_qkv, wqkv, out=o["ga"])),
]
if os.environ.get("ONCE"):  # one launch of each (for ncu --set full captures)
    for _ in range(2):
        for *_, fn in cases:
            fn()
    torch.cuda.synchronize()
    sys.exit(0)
tot_us = tot_fl = 0.0
for name, Mm, Nn, K, fn in cases:
    us = bench(fn)
    fl = 2.0 * Mm * Nn * K
    tot_us += us
    tot_fl += fl
    print(f"{name:16s} M={Mm:6d} N={Nn:5d} K={K:6d} {us:8.1f} us {fl / us / 1e6:7.1f} TFLOP/s", flush=True)
print(f"block total {tot_us:8.1f} us {tot_fl / tot_us / 1e6:7.1f} TFLOP/s (x12 blocks = {12 * tot_us / 1e3:.2f} ms)")
