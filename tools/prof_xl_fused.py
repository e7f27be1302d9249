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


d_rows = torch.empty(H * B * T, device="cuda")
gk, gv = torch.empty(H * B, Kl, dh, device="cuda", dtype=torch.bfloat16), torch.empty(H * B, Kl, dh, device="cuda",
                                                                                        dtype=torch.bfloat16)
g3h, quh, vhh = g3.view(H * B, T, dh), qu.view(H * B, T, dh), vh.view(H * B, Kl, dh)


def fwd():
    ops.xl_attn_fwd_pv(qu, qv, kh, vh, rh, probs, ctx, B, T, M, M, scale)


def bwd():
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, gac, gbd, gctx, ctx, gqu, gqv, B, T, M, M, scale)


def bwd_nodac():
    ops.xl_attn_bwd_dq(g3, vh, kh, rh, probs, None, gbd, gctx, ctx, gqu, gqv, B, T, M, M, scale, d_rows=d_rows)


def kv():
    ops.xl_attn_bwd_kv(g3h, vhh, quh, probs, d_rows, gk, gv, B, T, M, M, scale)


def gemm_dv():
    ops.gemm(probs[:, :, :Kl], g3h, a_mn=True, b_mn=True, out=gv, k_lo_off=-M)


def gemm_dk():
    ops.gemm(gac[:, :, :Kl], quh, a_mn=True, b_mn=True, out=gk, k_lo_off=-M)


fns = [fwd, bwd, bwd_nodac, kv, gemm_dv, gemm_dk]
only = os.environ.get("ONLY")
if only:
    fns = [f for f in fns if f.__name__ in only.split(",")]
for _ in range(reps):
    for f in fns:
        f()
torch.cuda.synchronize()
if reps > 1 and not os.environ.get("NOGRAPH"):
    # CUDA-graph replay of 10 back-to-back launches: no host time inside the window
    vis = (M + T / 2) / Kl  # causal + full memory: mean visible fraction of the keys
    fl = 2.0 * B * H * T * Kl * dh * vis * 3  # three MMAs of the score shape (algorithmic)
    st = torch.cuda.Stream()
    for f in fns:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            f()
            st.synchronize()
            with torch.cuda.graph(gr, stream=st):
                for _ in range(10):
                    f()
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(5):
            gr.replay()
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) / 50
        print(f"{f.__name__:12s} {t * 1e3:7.1f} us  {fl / t / 1e9:6.1f} TFLOP/s (3 score-shaped MMAs)")
