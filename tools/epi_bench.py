"""Isolates GEMM epilogue costs on the C2 Wo / FFN2 shapes: STORE vs
BIAS_DROPOUT_RESIDUAL with and without dropout / residual."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06695_b200 import _native as N  # noqa: E402
from paper_1909_06695_b200 import ops  # noqa: E402
from paper_1909_06695_b200.rng import keep_threshold  # noqa: E402

M = 8192
g = torch.Generator(device="cuda").manual_seed(0)


def r(*s):
    return ((torch.rand(*s, device="cuda", generator=g) * 2 - 1) * 0.05).bfloat16()


def timeit(fn, n=50):
    """Device time per launch: n launches replayed from a CUDA graph."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fn()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gr.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


drop = (1234, keep_threshold(0.1), 1 / 0.9, 0)
for K in (512, 2048):
    a, w = r(M, K), r(K, 512)
    res = r(M, 512)
    out = torch.empty(M, 512, dtype=torch.bfloat16, device="cuda")
    bias = torch.zeros(512, device="cuda")
    cases = {
        "store": lambda: ops.gemm(a, w, b_mn=True, out=out),
        "bias+resid": lambda: ops.gemm(a, w, b_mn=True, out=out, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=bias,
                                       residual=res),
        "bias+drop": lambda: ops.gemm(a, w, b_mn=True, out=out, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL, bias=bias,
                                      dropout=drop),
        "bias+drop+resid": lambda: ops.gemm(a, w, b_mn=True, out=out, epilogue=N.EPI_BIAS_DROPOUT_RESIDUAL,
                                            bias=bias, residual=res, dropout=drop),
    }
    for name, fn in cases.items():
        print(f"K={K:5d} {name:16s} {timeit(fn):7.1f} us")
