"""C3-shaped (B 22, H 8, T = M = 512, dh 64) XL attention backward: the fused
softmax backward + the two head-dim-wide query-gradient GEMMs against the
backward with the query-gradient MMAs folded in (xl_attn_bwd_dq)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import ops  # noqa: E402

B, H, T, M, dh = 22, 8, 512, 512, 64
Kl = M + T
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.6).to(torch.bfloat16)  # noqa: E731
qu, qv, kh, rh, vh = mk(H, B * T, dh), mk(H, B * T, dh), mk(H, B * Kl, dh), mk(H, Kl, dh), mk(H, B * Kl, dh)
g3, gctx, ctx = mk(H, B * T, dh), mk(B * T, H * dh), mk(B * T, H * dh)
probs = torch.empty(H * B, T, Kl, device="cuda", dtype=torch.bfloat16)
gac, gbd = torch.empty_like(probs), torch.empty_like(probs)
gqu = torch.empty(H, B * T, dh, device="cuda")
gqv = torch.empty(H, B * T, dh, device="cuda")
scale = 1.0 / math.sqrt(dh)
ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, M, scale)


def unfused():
    ops.xl_attn_bwd(g3, vh, probs, gac, gbd, gctx, ctx, B, T, M, M, scale)
    ops.gemm(gac, kh.view(H * B, Kl, dh), b_mn=True, out=gqu.view(H * B, T, dh))
    ops.gemm(gbd.view(H, B * T, Kl), rh, b_mn=True, out=gqv)


def fused():
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, gac, gbd, gctx, ctx, gqu, gqv, B, T, M, M, scale)


def bwd_only():
    ops.xl_attn_bwd(g3, vh, probs, gac, gbd, gctx, ctx, B, T, M, M, scale)


which = os.environ.get("ONLY")
for name, fn in (("bwd + 2 GEMMs", unfused), ("bwd_dq", fused), ("bwd alone", bwd_only)):
    if which and which not in name:
        continue
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / n * 1e3:.1f} us")
