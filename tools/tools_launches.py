"""Aggregate an ncu --metrics gpu__time_duration.sum CSV by kernel name."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[hi]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    v *= {'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}.get(r[ui], 1.0)
    name = r[ki].split('(')[0]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / 1e6:10.2f} ms {100 * t / tot:5.1f}% {n:6d}  {k}")
print(f"total {tot / 1e6:.2f} ms")
