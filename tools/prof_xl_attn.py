"""One C3-shaped (Transformer-XL base: B 22, H 8, T = M = 512, dh 64) fused
attention forward + backward, for ncu captures of xl_attn_fwd / xl_attn_bwd."""
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
scale = 1.0 / math.sqrt(dh)
reps = int(os.environ.get("REPS", "3"))


def run():
    ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, M, scale)
    ops.xl_attn_bwd(g3, vh, probs, gac, gbd, gctx, ctx, B, T, M, M, scale)


for _ in range(reps):
    run()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
n = 20
ts = [0.0, 0.0]
for _ in range(n):
    ev[0].record()
    ops.xl_attn_fwd(qu, qv, kh, rh, probs, B, T, M, M, scale)
    ev[1].record()
    ops.xl_attn_bwd(g3, vh, probs, gac, gbd, gctx, ctx, B, T, M, M, scale)
    ev[2].record()
    torch.cuda.synchronize()
    ts[0] += ev[0].elapsed_time(ev[1]) / n
    ts[1] += ev[1].elapsed_time(ev[2]) / n
fl = 2 * 2.0 * B * H * T * Kl * dh  # AC + BD (algorithmic, unshifted BD)
p_bytes = B * H * T * Kl * 2
print(f"xl_attn_fwd {ts[0] * 1e3:.1f} us  {fl / ts[0] / 1e9:.1f} TFLOP/s (AC+BD)  P write {p_bytes / ts[0] / 1e6:.0f} GB/s")
print(f"xl_attn_bwd {ts[1] * 1e3:.1f} us  dP {fl / 2 / ts[1] / 1e9:.1f} TFLOP/s  "
      f"P read + dAC + dBD write {3 * p_bytes / ts[1] / 1e6:.0f} GB/s")
