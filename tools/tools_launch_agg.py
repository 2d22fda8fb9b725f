"""Aggregate an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals over the last 1/k of launches."""
import csv, collections, sys
path = sys.argv[1]; frac = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
last = rows[(frac - 1) * len(rows) // frac:]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in last:
    name = r[ki].split('(')[0][:60]; agg[name][0] += 1; agg[name][1] += float(r[vi])
tot = sum(v[1] for v in agg.values())
print(f"launches {len(last)}  total {tot/1e6:.3f} ms (cold-cache, serialised)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]/1e3:9.1f} us {v[0]:4d} {100*v[1]/tot:5.1f}%  {k}")
