"""Runs the tied-vocab head of C2 (N=8192, d=512, V=267,735, bf16) once
forward + backward: the 4 head GEMM launches, for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import layers as LY  # noqa: E402

N, d, V = 8192, 512, 267735
g = torch.Generator(device="cuda").manual_seed(0)
h = (torch.rand(N, d, device="cuda", generator=g) * 2 - 1).bfloat16()
tied = ((torch.rand(V, d, device="cuda", generator=g) * 2 - 1) * 0.044).bfloat16()
y = torch.randint(0, V, (N,), device="cuda", generator=g)
ws = LY.Workspace(h.device)
hs = LY.HeadState(N, h.device)
gh = torch.empty(N, d, device="cuda")
vo = torch.empty(V, d, device="cuda")
reps = int(os.environ.get("REPS", "2"))
for _ in range(reps):
    LY.head_forward(h, tied, y, V, hs, ws, None)
    LY.head_backward(h, tied, y, V, hs, gh, vo, 0.5, ws)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    LY.head_forward(h, tied, y, V, hs, ws, None)
    LY.head_backward(h, tied, y, V, hs, gh, vo, 0.5, ws)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"head fwd+bwd {ms:.3f} ms  -> {4 * 2 * N * d * V / ms / 1e9:.1f} TFLOP/s over 4 GEMMs, loss {hs.loss.item():.4f}")
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
f0.record()
for _ in range(5):
    LY.head_forward(h, tied, y, V, hs, ws, None)
f1.record()
torch.cuda.synchronize()
print(f"head fwd (LSE pass + CE finish) {f0.elapsed_time(f1) / 5:.3f} ms")

