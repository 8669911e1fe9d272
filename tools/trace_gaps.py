"""Idle gaps of the compute lane in a step trace (bench.py --trace-out), with the copy-lane ops
running across each gap.

    python tools/trace_gaps.py trace.txt [--min-us 50]
"""
import argparse


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--min-us", type=float, default=50.0)
    a = ap.parse_args()
    ops = []
    for line in open(a.trace):
        f = line.split()
        if len(f) >= 7:
            ops.append((f[0], f[1], f[2], f[3], f[4], float(f[5]), float(f[6])))
    comp = sorted((o for o in ops if o[0] == "compute"), key=lambda o: o[5])
    span = max(o[6] for o in ops) - min(o[5] for o in ops)
    busy, gaps, end = 0.0, [], None
    for o in comp:
        if end is not None and o[5] - end > a.min_us:
            gaps.append((end, o[5], o))
        busy += o[6] - o[5]
        end = o[6] if end is None else max(end, o[6])
    print(f"span {span / 1000:.1f} ms, compute ops {len(comp)}, compute busy {busy / 1000:.1f} ms, "
          f"gaps > {a.min_us:.0f} us: {len(gaps)} totalling {sum(g[1] - g[0] for g in gaps) / 1000:.1f} ms")
    for g0, g1, nxt in gaps:
        across = [o for o in ops if o[0] != "compute" and o[5] < g1 and o[6] > g0]
        desc = ", ".join(f"{o[0]}:{o[1]}{o[2]}[{o[5] / 1000:.1f}-{o[6] / 1000:.1f}]" for o in across[:4])
        print(f"  gap {g0 / 1000:8.2f} -> {g1 / 1000:8.2f} ms ({(g1 - g0) / 1000:6.2f} ms) before "
              f"{nxt[1]} seg {nxt[2]} mb {nxt[3]} | {desc}")


if __name__ == "__main__":
    main()
