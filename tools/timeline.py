"""Kernel timeline of C2 Ouroboros steps via torch.profiler (CUPTI): GPU busy
fraction (union of kernel intervals), idle gaps, per-kernel totals."""
import collections
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1909_06695_b200 import engine as E  # noqa: E402
from paper_1909_06695_b200 import model as M  # noqa: E402
from paper_1909_06695_b200 import optim as O  # noqa: E402

c = bench.CONFIGS[os.environ.get("CFG", "c2")]
B, T = c["batch"], c["seq"]
stack = bench.make_stack(c, 1)
cls = E.PipelineEngine if os.environ.get("ENGINE") == "reference" else E.ConcurrentPipelineEngine
eng = cls(stack, M.partition(stack.num_layers, 2), 3)
opt = O.make_optimizer("adam", O.LrSchedule(2.5e-4))
rng = np.random.default_rng(0)
dev = [(torch.from_numpy(bench.zipf_tokens(rng, (B, T), c["vocab"])).cuda(),
        torch.from_numpy(bench.zipf_tokens(rng, (B, T), c["vocab"])).cuda()) for _ in range(2)]
for t in range(4):
    eng.step(t, E.BatchSample(*dev[t % 2], t), opt)
torch.cuda.synchronize()
steps = 3
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for t in range(4, 4 + steps):
        eng.step(t, E.BatchSample(*dev[t % 2], t), opt, sync="lagged")
    eng.flush_lagged()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
busy, cur_s, cur_e = 0, None, None
gaps = []
for s, e, _ in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append(s - cur_e)
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = t1 - t0
tot = collections.defaultdict(float)
for s, e, n in iv:
    tot[n.replace("(anonymous namespace)::", "").split("(")[0][:60]] += e - s
print(json.dumps({"steps": steps, "span_ms": span / 1e3, "ms_per_step": span / 1e3 / steps,
                  "gpu_busy_frac": busy / span, "gaps_over_5us": sum(1 for g in gaps if g > 5),
                  "gap_ms_total": sum(gaps) / 1e3}))
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{v / 1e3 / steps:8.3f} ms/step  {n}")
prof.export_chrome_trace(os.path.join(ROOT, "gpurun_out", "trace.json"))
