"""Per-launch summary of an `ncu --set full` report (run here, on the CPU side):
duration, DRAM bytes read / written, tensor-pipe and SM/DRAM throughput.

  python tools/ncu_summary.py REPORT.ncu-rep [--labels "a;b;..."] [--json OUT.json] [--source NOTE]

With --json, also writes the head-GEMM traffic file bench.py reads
(bytes_per_launch = mean DRAM read + write over the launches)."""
import argparse
import csv
import io
import json
import subprocess

METRICS = {
    "ms": ("gpu__time_duration.sum", 1e-6),  # ns -> ms
    "dram_read_GB": ("dram__bytes_read.sum", 1e-9),
    "dram_write_GB": ("dram__bytes_write.sum", 1e-9),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_mem_active_pct": ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
}
UNIT = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
        "Gbyte": 1e9}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        if len(r) != len(hdr):
            continue
        d = {"kernel": r[hdr.index("Kernel Name")][:80], "grid": r[hdr.index("Grid Size")]}
        for k, (m, sc) in METRICS.items():
            cols = [c for c, h in enumerate(hdr) if h == m or h.endswith("." + m)]
            if cols:
                v = r[cols[0]].replace(",", "")
                try:
                    d[k] = round(float(v) * sc, 4)
                except ValueError:
                    d[k] = None
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--labels", default="")
    ap.add_argument("--json")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    res = load(a.report)
    labels = a.labels.split(";") if a.labels else []
    for i, d in enumerate(res):
        if i < len(labels):
            d["launch"] = labels[i]
        print(json.dumps(d))
    if a.json:
        tot = [(d.get("dram_read_GB") or 0) + (d.get("dram_write_GB") or 0) for d in res]
        with open(a.json, "w") as fh:
            json.dump({"source": a.source, "bytes_per_launch": sum(tot) / max(len(tot), 1) * 1e9, "launches": res},
                      fh, indent=1)


if __name__ == "__main__":
    main()
