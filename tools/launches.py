"""Summarise an ncu launch list (gpu__time_duration.sum): per-kernel share of the last frame."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
data = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[hi + 1:] if len(r) > vi]
idx = [i for i, (k, v) in enumerate(data) if 'k_preprocess' in k]
frame = data[idx[-1]:] if idx else data
agg = collections.OrderedDict()
for k, v in frame:
    n = k.split('(')[0].split('<')[0].replace('void ', '').replace('cr::', '')
    agg.setdefault(n, [0, 0]); agg[n][0] += v; agg[n][1] += 1
tot = sum(a[0] for a in agg.values())
for n, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:32s} {c:4d} {v/1e6:9.3f} ms {100*v/tot:5.1f}%")
print(f"{'total':32s} {sum(a[1] for a in agg.values()):4d} {tot/1e6:9.3f} ms")
