"""Summarise an ncu --set full report: per-launch duration, DRAM traffic, tensor-pipe and L2 activity.

    python tools/ncu_summary.py report.ncu-rep [--flops F] [--bytes B] > summary.json

--flops / --bytes: algorithmic FLOPs and bytes of one launch (to compare with measured traffic).
"""
import argparse
import csv
import io
import json
import subprocess

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1, "": 1, "register/thread": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--flops", type=float, default=None)
    ap.add_argument("--bytes", type=float, default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, name in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                    d[name] = v * SCALE.get(units[i], 1)
                except ValueError:
                    d[name] = r[i]
        if "dram_read" in d and "dram_write" in d:
            d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
        if a.flops and d.get("duration"):
            d["tflops"] = a.flops / d["duration"] / 1e12
        if a.bytes:
            d["algorithmic_bytes"] = a.bytes
        out.append(d)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
