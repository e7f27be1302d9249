"""Per-stream layout of the last profiled step in gpurun_out/trace.json
(written by tools/timeline.py): busy time, first / last kernel and the long
kernels (> 0.5 ms, the head GEMMs) with their start offsets."""
import collections
import json
import os
import sys

path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "gpurun_out", "trace.json")
tr = json.load(open(path))
evs = sorted((e for e in tr["traceEvents"] if e.get("cat") == "kernel"), key=lambda e: e["ts"])
t0, t1 = evs[0]["ts"], max(e["ts"] + e["dur"] for e in evs)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
step = (t1 - t0) / steps
w0 = t0 + (steps - 1) * step
last = [e for e in evs if e["ts"] >= w0]
by = collections.defaultdict(list)
for e in last:
    by[e["args"].get("stream")].append(e)
print(f"step {step / 1e3:.3f} ms (window start = 0)")
for sid, es in sorted(by.items(), key=lambda kv: kv[1][0]["ts"]):
    busy = sum(e["dur"] for e in es)
    end = max(e["ts"] + e["dur"] for e in es) - w0
    longk = [f"{(e['ts'] - w0) / 1e3:.2f}+{e['dur'] / 1e3:.2f}" for e in es if e["dur"] > 500]
    name = lambda e: e["name"].replace("(anonymous namespace)::", "").split("(")[0].split("::")[-1][:24]  # noqa: E731
    print(f"stream {sid:>4}: n={len(es):4d} {es[0]['ts'] - w0:9.0f} .. {end:9.0f} us busy {busy:8.0f} "
          f"first={name(es[0])} last={name(es[-1])} long={longk}")
