"""The three head-dim-wide gradient GEMMs of the C3 XL backward (dV = P^T dO,
dK = dAC^T (q+u), dR = dBD^T (q+v); N = dh 64, K = queries, A = the 185 MB
bf16 score-shaped matrices), CUDA-event timed, for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import ops  # noqa: E402

B, H, T, M, dh = 22, 8, 512, 512, 64
Kl = M + T
ldk = (Kl + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.3).to(torch.bfloat16)  # noqa: E731
P = mk(H * B, T, ldk)[:, :, :Kl]
gac = mk(H * B, T, ldk)[:, :, :Kl]
gbd = mk(H, B * T, ldk)[:, :, :Kl]
g3, qu, qv = mk(H * B, T, dh), mk(H * B, T, dh), mk(H, B * T, dh)
gvh = torch.empty(H * B, Kl, dh, device="cuda")
gkh = torch.empty(H * B, Kl, dh, device="cuda")
grh = torch.empty(H, Kl, dh, device="cuda")
reps = int(os.environ.get("REPS", "3"))
calls = [("dV", lambda: ops.gemm(P, g3, a_mn=True, b_mn=True, out=gvh, k_lo_off=-M), 0.75 * P.numel() * 2),
         ("dK", lambda: ops.gemm(gac, qu, a_mn=True, b_mn=True, out=gkh, k_lo_off=-M), 0.75 * P.numel() * 2),
         ("dR", lambda: ops.gemm(gbd, qv, a_mn=True, b_mn=True, out=grh), gbd.numel() * 2)]
for _ in range(reps):
    for _, f, _ in calls:
        f()
torch.cuda.synchronize()
if reps > 1:
    for name, f, nbytes in calls:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 100
        print(f"{name}: {us:.1f} us  A stream {nbytes / us / 1e3:.0f} GB/s")
