"""C3-shaped (B 22, H 8, T = M = 512, dh 64) fused XL attention as the step
runs it: xl_attn_fwd_pv (scores + shift + softmax + P.V) and xl_attn_bwd_dq
(dP, dS, dAC / dBD + dQu / dQv), CUDA-event timed, for ncu captures."""
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
g3 = mk(H, B * T, dh)
gctx = mk(B * T, H * dh)
ctx = torch.empty(B * T, H * dh, device="cuda", dtype=torch.bfloat16)
ldp = (Kl + 7) // 8 * 8
probs = torch.empty(H * B, T, ldp, device="cuda", dtype=torch.bfloat16)
gac, gbd = torch.empty_like(probs), torch.empty(H, B * T, ldp, device="cuda", dtype=torch.bfloat16)
gqu = torch.empty(H, B * T, dh, device="cuda")
gqv = torch.empty(H, B * T, dh, device="cuda")
scale = 1.0 / math.sqrt(dh)
reps = int(os.environ.get("REPS", "3"))


def fwd():
    ops.xl_attn_fwd_pv(qu, qv, kh, vh, rh, probs, ctx, B, T, M, M, scale)


def bwd():
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, gac, gbd, gctx, ctx, gqu, gqv, B, T, M, M, scale)


for _ in range(reps):
    fwd()
    bwd()
torch.cuda.synchronize()
if reps > 1:
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    n, ts = 20, [0.0, 0.0]
    for _ in range(n):
        ev[0].record()
        fwd()
        ev[1].record()
        bwd()
        ev[2].record()
        torch.cuda.synchronize()
        ts[0] += ev[0].elapsed_time(ev[1]) / n
        ts[1] += ev[1].elapsed_time(ev[2]) / n
    vis = (M + T / 2) / Kl  # causal + full memory: mean visible fraction of the keys
    fl_f = 2.0 * B * H * T * Kl * dh * vis * 3  # AC, BD, PV (algorithmic; BD unshifted)
    fl_b = 2.0 * B * H * T * Kl * dh * vis * 3  # dP, dQu, dQv
    print(f"xl_attn_fwd_pv {ts[0] * 1e3:.1f} us  {fl_f / ts[0] / 1e9:.1f} TFLOP/s algorithmic")
    print(f"xl_attn_bwd_dq {ts[1] * 1e3:.1f} us  {fl_b / ts[1] / 1e9:.1f} TFLOP/s algorithmic")
