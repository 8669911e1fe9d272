"""Warp-stall hot spots of each kernel in an ncu --set full report (SASS source page).

    python tools/ncu_stalls.py report.ncu-rep [--top 20] [--kernel REGEX]

Prints, per kernel: total stall samples, the top instructions by samples (with the instruction
before them, which is usually the one being waited on) and the stall-reason totals.
"""
import argparse
import csv
import io
import re
import subprocess
from collections import Counter


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=20)
    ap.add_argument("--kernel", default=".")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], []
    for line in out.split("\n"):
        if line.startswith('"Kernel Name"'):
            if cur:
                blocks.append(cur)
            cur = [line]
        elif cur:
            cur.append(line)
    if cur:
        blocks.append(cur)
    seen = set()
    for b in blocks:
        rows = list(csv.reader(io.StringIO("\n".join(b))))
        name = rows[0][1]
        if name in seen or not re.search(a.kernel, name):
            continue
        seen.add(name)
        hdr = rows[1]
        data = [r for r in rows[2:] if len(r) == len(hdr)]
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_src = hdr.index("Source")
        i_ex = hdr.index("Instructions Executed")
        tot = sum(int(r[i_s] or 0) for r in data)
        print(f"=== {name[:110]}\n    samples {tot}")
        order = sorted(range(len(data)), key=lambda k: -int(data[k][i_s] or 0))[: a.top]
        for k in order:
            r = data[k]
            prev = data[k - 1][i_src].strip()[:60] if k else ""
            print(f"  {r[0][-5:]} {int(r[i_s] or 0):6d} {int(r[i_ex] or 0):9d}  {r[i_src].strip()[:58]:58s} | {prev}")
        cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
        c = Counter()
        for r in data:
            for col in cols:
                c[col] += int(r[hdr.index(col)] or 0)
        print("    reasons:", ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(8)))


if __name__ == "__main__":
    main()
