"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main(path, step_marker="embed_fwd_kernel"):
    data = load(path)
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    us = [float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0) for d in data]
    # one full step = launches between two embedding forwards
    starts = [i for i, d in enumerate(data) if step_marker in d["Kernel Name"]]
    # the last complete window: steady state (earlier ones include warm-up allocations)
    lo, hi = (starts[-2], starts[-1]) if len(starts) >= 2 else (0, len(data))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d, t in zip(data[lo:hi], us[lo:hi]):
        name = d["Kernel Name"].split("(")[0][:60]
        agg[name][0] += 1
        agg[name][1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"one step: launches {hi - lo}, serialized kernel time {tot / 1e3:.3f} ms")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}%  n={v[0]:4d}  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
