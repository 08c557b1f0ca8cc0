"""Per-kernel average duration from an ncu --metrics gpu__time_duration.sum CSV log:
launch_sum.py LOG.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
K, M, V, I = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[M] != "gpu__time_duration.sum":
        continue
    a = agg.setdefault(r[K][:44], [0, 0.0])
    a[0] += 1
    a[1] += float(r[V].replace(",", ""))
for n, (c, t) in agg.items():
    print(f"{n:46s} n={c:3d} avg_us={t / c / 1e3:9.1f}")
