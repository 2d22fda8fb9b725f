"""Per-(kernel, grid) totals from an ncu CSV with gpu__time_duration.sum and launch__grid_size (last 1/k launches)."""
import csv, collections, sys
path = sys.argv[1]; frac = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, mi, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
by = collections.defaultdict(dict)
for r in rows:
    by[int(r[ii])][r[mi]] = r[vi]; by[int(r[ii])]['name'] = r[ki].split('(')[0].replace('void ', '').replace('unnamed>::', '')[:40]
ids = sorted(by); ids = ids[(frac - 1) * len(ids) // frac:]
agg = collections.defaultdict(lambda: [0, 0.0])
for i in ids:
    d = by[i]; key = (d['name'], d.get('launch__grid_size', '?'))
    agg[key][0] += 1; agg[key][1] += float(d['gpu__time_duration.sum'])
tot = sum(v[1] for v in agg.values())
print(f"launches {len(ids)} total {tot/1e6:.3f} ms")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:45]:
    print(f"{v[1]/1e3:8.1f} us {v[0]:4d} x {v[1]/1e3/v[0]:6.1f}  {100*v[1]/tot:5.1f}%  {k[0]:40s} grid={k[1]}")
