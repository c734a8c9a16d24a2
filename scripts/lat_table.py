"""Per-kernel durations of the last encode+decode of an ncu launch list
(scripts/gpu_lat_ncu.sh): usage python scripts/lat_table.py launches.csv [n_last]"""
import csv
import sys
from collections import OrderedDict

lines = open(sys.argv[1]).read().splitlines()
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else 14
st = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[st:]))
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
cur = OrderedDict()
for r in rows[1:]:
    cur.setdefault((r[0], r[ik][:70]), {})[r[im]] = r[iv]
tot = 0
for (i, k), m in list(cur.items())[-n_last:]:
    ns = float(m.get("gpu__time_duration.sum", 0))
    tot += ns
    print(f"{i:>4} {k:70s} {ns / 1e3:8.2f} us  grid {m.get('launch__grid_size')}")
print(f"sum {tot / 1e3:.1f} us")
