"""Isolated timing of block-shaped GEMMs (CUDA events over 50 back-to-back
launches): where do small GEMMs lose time -- mainloop, epilogue or fixed cost?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import _native as N  # noqa: E402
from paper_1909_06695_b200 import ops  # noqa: E402
from paper_1909_06695_b200.rng import keep_threshold  # noqa: E402


def bench(fn, reps=50):
    """GPU time per launch: the launches are captured in a CUDA graph so the
    host (Python) launch path is out of the measurement."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def run(M, Nn, K, epi="store"):
    a = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(K, Nn, device="cuda").bfloat16() * 0.02
    out = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    resid = torch.randn(M, Nn, device="cuda").bfloat16()
    bias = torch.randn(Nn, device="cuda")
    kw = {}
    if epi == "dropres":
        kw = dict(epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=bias, residual=resid,
                  dropout=(123, keep_threshold(0.1), 1 / 0.9, 0))
    elif epi == "res":
        kw = dict(epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, residual=resid)
    us = bench(lambda: ops.gemm(a, w, b_mn=True, out=out, **kw))
    tf = 2 * M * Nn * K / us / 1e6
    print(f"M={M:5d} N={Nn:5d} K={K:5d} {epi:8s} {us:8.1f} us {tf:7.1f} TFLOP/s  2cta={os.environ.get('RP_2CTA', '1')}",
          flush=True)


for M, Nn, K in [(8192, 512, 2048), (8192, 512, 512), (8192, 2048, 512), (8192, 1536, 512), (8192, 512, 8192),
                 (16384, 512, 2048), (8192, 512, 4096)]:
    for epi in ("store", "res", "dropres"):
        run(M, Nn, K, epi)
