"""One C2 transformer block forward + backward (bf16, B=16, T=512, d=512,
f=2048) through the native composites, for ncu captures of the block GEMMs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import layers as LY  # noqa: E402

B, T, d, f = 16, 512, 512, 2048
N = B * T
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s, sc=0.04: ((torch.rand(*s, device="cuda", generator=g) * 2 - 1) * sc)  # noqa: E731
W = {"wqkv": r(d, 3 * d).bfloat16(), "wo": r(d, d).bfloat16(), "w1": r(d, f).bfloat16(), "w2": r(f, d).bfloat16(),
     "ln1_g": 1 + r(d), "ln1_b": r(d), "ln2_g": 1 + r(d), "ln2_b": r(d), "b1": r(f), "b2": r(d)}
x = r(N, d, sc=1.0).bfloat16()
tape = LY.BlockTape(B, T, d, f, torch.bfloat16, x.device)
ws = LY.Workspace(x.device)
out = torch.empty_like(x)
g_out = r(N, d, sc=1.0).float()
g_x = torch.empty_like(g_out)
G = {k: torch.empty(v.shape, dtype=torch.float32, device="cuda") for k, v in W.items()}
drop = LY.Dropout.make(12345, 0.1, True)
reps = int(os.environ.get("REPS", "3"))
for _ in range(reps):
    LY.block_forward(W, W, x, out, tape, B, T, drop, ws, None)
    LY.block_backward(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
torch.cuda.synchronize()
import time  # noqa: E402

s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
h0 = time.perf_counter()
for _ in range(10):
    LY.block_forward(W, W, x, out, tape, B, T, drop, ws, None)
    LY.block_backward(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
host_ms = (time.perf_counter() - h0) * 1e3 / 10
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"host issue time per block fwd+bwd: {host_ms:.3f} ms")
# GPU-only time: replay the same work as a CUDA graph
gr = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    LY.block_forward(W, W, x, out, tape, B, T, drop, ws, None)
    LY.block_backward(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
    with torch.cuda.graph(gr, stream=st):
        LY.block_forward(W, W, x, out, tape, B, T, drop, ws, None)
        LY.block_backward(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
torch.cuda.synchronize()
for _ in range(3):
    gr.replay()
torch.cuda.synchronize()
s.record()
for _ in range(10):
    gr.replay()
e.record()
torch.cuda.synchronize()
print(f"graph replay block fwd+bwd {s.elapsed_time(e) / 10:.3f} ms")
fl = 3 * N * (2 * (4 * d * d + 2 * d * f) + 2 * 2 * d * T)  # fwd+bwd incl. full TxT attention
print(f"block fwd+bwd {ms:.3f} ms -> {fl / ms / 1e9:.1f} TFLOP/s")
