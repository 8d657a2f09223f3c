"""Aggregate an ncu --metrics gpu__time_duration.sum CSV into a per-kernel table."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    agg[r[ik][:70]][0] += 1
    agg[r[ik][:70]][1] += v
tot = sum(v for c, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{c:5d} {v / 1e6:9.3f} ms {100 * v / tot:5.1f}% {v / c / 1e3:9.1f} us/launch  {k}")
