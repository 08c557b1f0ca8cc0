#!/bin/bash
# per-kernel durations of one cold C2 step (ncu launch list): tools/launch_list.sh OUT.csv [CFG]
cfg=${2:-C2}
ncu --metrics ${METRICS:-gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct} --clock-control none --print-units base --csv --log-file "$1" \
  python -c "
import sys; sys.argv=['x','$cfg']; sys.path.insert(0,'.')
import tools.quick_time as q
" > /dev/null 2>&1
python3 - "$1" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
K = h.index("Kernel Name"); M = h.index("Metric Name"); V = h.index("Metric Value"); I = h.index("ID")
d = collections.OrderedDict()
for r in rows:
    d.setdefault(r[I], {"name": r[K][:40]})[r[M]] = r[V]
agg = collections.OrderedDict()
for k, v in d.items():
    a = agg.setdefault(v["name"], [0, 0.0, 0.0, 0.0, 0.0, 0.0])
    a[0] += 1; a[1] += float(v.get("gpu__time_duration.sum", 0)); a[2] += float(v.get("dram__bytes_read.sum", 0)); a[3] += float(v.get("dram__bytes_write.sum", 0))
    a[4] += float(v.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)); a[5] += float(v.get("lts__t_sector_hit_rate.pct", 0))
for n, a in agg.items():
    print(f"{n:42s} n={a[0]:3d} avg_us={a[1]/a[0]/1e3:9.1f} rdMB={a[2]/a[0]/1e6:8.1f} wrMB={a[3]/a[0]/1e6:8.1f} occ%={a[4]/a[0]:5.1f} l2hit%={a[5]/a[0]:5.1f}")
PY
