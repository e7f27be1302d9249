"""LayerNorm backward at the C5 shape (Transformer-XL large: 12288 rows of
d 1024; residual gradient in, fp32 dx + dropout-masked bf16 dx out), CUDA-event
timed.  RP_LN_SPLIT=1/2/4 sets the warps per row for an A/B."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import ops  # noqa: E402

rows, d = int(os.environ.get("ROWS", "12288")), int(os.environ.get("D", "1024"))
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(rows, d, device="cuda", generator=g).to(torch.bfloat16)
gain = 1 + 0.1 * torch.randn(d, device="cuda", generator=g)
bias = torch.zeros(d, device="cuda")
dy = torch.randn(rows, d, device="cuda", generator=g)
res = torch.randn(rows, d, device="cuda", generator=g)
y = torch.empty_like(x)
mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
ops.layernorm_fwd(x, gain, bias, y, mean, rstd)
nb = ops.layernorm_bwd_blocks(rows)
pg, pb = torch.empty(nb, d, device="cuda"), torch.empty(nb, d, device="cuda")
dx = torch.empty(rows, d, device="cuda")
dxm = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run():
    ops.layernorm_bwd(dy, x, mean, rstd, gain, dx, pg, pb, resid_grad=res, dx_masked=dxm, dropout=(7, int(0.1 * 2**53), 1 / 0.9))


for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    flush.zero_()  # inputs leave L2 between launches
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
us = ts[len(ts) // 2] * 1e3
nbytes = rows * d * (4 + 2 + 4 + 4 + 2)  # dy, x, resid in; dx, dx_masked out
print(f"ln_bwd rows {rows} d {d} split={os.environ.get('RP_LN_SPLIT', 'default')}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s")
