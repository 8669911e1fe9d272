"""Summarise an ncu gpu__time_duration.sum launch list (CSV) by kernel: python tools/launch_summary.py list.csv [header]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot = collections.defaultdict(float); cnt = collections.Counter()
for d in data:
    k = d['Kernel Name'].split('(')[0]
    v = float(d['Metric Value'].replace(',', ''))
    u = d['Metric Unit']
    v = v / 1e6 if u in ('ns', 'nsecond') else (v / 1e3 if u in ('us', 'usecond') else v)
    tot[k] += v; cnt[k] += 1
T = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"# total {T:.1f} ms over {len(data)} launches")
print("ms\tshare\tlaunches\tkernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:.2f}\t{100*v/T:.1f}%\t{cnt[k]}\t{k}")
