"""Ad-hoc numerics diagnostic for the tcgen05 GEMM (not collected by pytest)."""
import torch
from paper_1909_06695_b200 import ops, _native as N
torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
g = torch.Generator().manual_seed(0)
for K in (64, 512, 2048, 8192):
    for dt in (torch.bfloat16, torch.float32):
        a = (torch.rand(256, K, generator=g, dtype=torch.float64) * 2 - 1).to(dt).to(dev)
        b = (torch.rand(384, K, generator=g, dtype=torch.float64) * 2 - 1).to(dt).to(dev)
        ref = a.double() @ b.double().T
        rel = lambda x: ((x.double() - ref).norm() / ref.norm()).item()
        c = ops.gemm(a, b, out_dtype=torch.float32)
        line = f"K={K} {dt}: ours={rel(c):.3e}"
        if dt == torch.float32:
            c1 = ops.gemm(a, b, math=N.MATH_TF32, out_dtype=torch.float32)
            line += f" tf32x1={rel(c1):.3e} cublas_fp32={rel(a @ b.T):.3e}"
        print(line, flush=True)
