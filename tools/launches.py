"""Summarise an ncu --csv launch list: per-kernel count, total and mean duration."""
import csv, sys
from collections import defaultdict
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
d = defaultdict(dict)
for r in rows[1:]:
    d[int(r[ii])][r[mi]] = r[vi].replace(',', '')
    d[int(r[ii])]['name'] = r[ki]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, x in d.items():
    nm = x['name'].split('(')[0].replace('void ', '').replace('husky::', '')
    a = agg[nm]
    a[0] += 1
    a[1] += float(x.get('gpu__time_duration.sum', 0))
    a[2] += float(x.get('dram__bytes_read.sum', 0) or 0)
    a[3] += float(x.get('dram__bytes_write.sum', 0) or 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':40s} {'n':>5s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s} {'rd_MB/launch':>12s} {'wr_MB/launch':>12s}")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{nm[:40]:40s} {a[0]:5d} {a[1]/1e3:10.1f} {a[1]/a[0]/1e3:9.2f} {a[1]/tot:6.1%} {a[2]/a[0]/1e6:12.1f} {a[3]/a[0]/1e6:12.1f}")
