"""Unfused XL score GEMMs at the C4 shape (B 60, H 10, T = M = 150, head dim
40: AC = (q+u) k^T, BD = (q+v) r^T, and the backward dP = g_ctx v^T, fp32 out)
timed per N tile (0 = library default) with CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import ops  # noqa: E402

B, H, T, M, dh = 60, 10, 150, 150, 40
Kl = M + T
ldk = (Kl + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)  # noqa: E731
qu, qv, kh, rh = mk(H * B, T, dh), mk(H, B * T, dh), mk(H * B, Kl, dh), mk(H, Kl, dh)
ac = torch.empty(H * B, T, ldk, device="cuda")[:, :, :Kl]
bd = torch.empty(H, B * T, ldk, device="cuda")[:, :, :Kl]


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


ref_ac = ref_bd = None
for tile in (0, 64, 128, 256):
    a = t(lambda: ops.gemm(qu, kh, out=ac, tile_n=tile))
    b = t(lambda: ops.gemm(qv, rh, out=bd, tile_n=tile))
    if ref_ac is None:
        ref_ac, ref_bd = ac.clone(), bd.clone()
    same = bool(torch.equal(ac, ref_ac) and torch.equal(bd, ref_bd))
    print(f"tile {tile:3d}: AC {a:6.1f} us  BD {b:6.1f} us  bitwise-equal to default: {same}")

# P-reading GEMMs of the fused path: ctx_h = P v (C3: dh 64, C5: dh 128)
for (Bq, Hq, Tq, Mq, dq) in ((22, 8, 512, 512, 64), (16, 8, 768, 768, 128)):
    Klq = Mq + Tq
    P = mk(Hq * Bq, Tq, Klq)
    vq = mk(Hq * Bq, Klq, dq)
    o = torch.empty(Hq * Bq, Tq, dq, device="cuda", dtype=torch.bfloat16)
    ref = None
    for tile in (0, 64, 128, 256):
        us = t(lambda: ops.gemm(P, vq, b_mn=True, out=o, tile_n=tile))
        if ref is None:
            ref = o.clone()
        print(f"PV dh {dq} tile {tile:3d}: {us:6.1f} us  bitwise-equal: {bool(torch.equal(o, ref))}")
