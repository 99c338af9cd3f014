"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    agg[r[ki][:100]][0] += 1
    agg[r[ki][:100]][1] += v
    tot += v
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"# total {tot / 1e3:.1f} us over {sum(a[0] for a in agg.values())} launches (ncu: cold-cache, serialised)")
print("# share_pct  total_us  launches  avg_us  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{100 * v / tot:6.2f} {v / 1e3:10.1f} {c:6d} {v / 1e3 / c:9.2f}  {k}")
