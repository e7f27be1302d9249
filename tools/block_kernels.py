"""Per-launch kernel durations (CUPTI via torch.profiler, not serialized) of
one C2 block forward + backward, in issue order."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("REPS", "3")
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_block.py")).read().split("import time")[0])

from torch.profiler import ProfilerActivity, profile  # noqa: E402

torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        LY.block_forward(W, W, x, out, tape, B, T, drop, ws, None)
        LY.block_backward(W, W, x, tape, g_out, g_x, G, B, T, drop, ws)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "rp::" in e.name]
evs.sort(key=lambda e: e.time_range.start)
half = len(evs) // 2
t0 = evs[half].time_range.start
tot = 0.0
for e in evs[half:]:
    d = e.time_range.end - e.time_range.start
    tot += d
    print(f"{(e.time_range.start - t0):8.1f} {d:7.1f}us {e.name.replace('(anonymous namespace)::', '').split('(')[0][:60]}")
span = evs[-1].time_range.end - t0
print(f"sum {tot:.1f} us, span {span:.1f} us")
