"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv, sys, collections, re
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = re.sub(r'\(.*', '', r[ki]).replace('void ', '')
    name = re.sub(r'cpf::', '', name)
    v = float(r[vi].replace(',', ''))
    unit = hdr[vi]
    agg[name][0] += 1
    agg[name][1] += v
    total += v
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name[:60]:60s} {n:8d} {t/1e3:12.1f} {t/n/1e3:10.2f} {t/total:7.3f}")
print(f"total {total/1e3:.1f} us")
