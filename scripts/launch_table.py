"""Summarise an ncu --csv launch list: last `iters`-th share of launches."""
import csv
import sys

path = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lines = open(path).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
d = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    d.setdefault(int(r[iid]), [r[ik][:48], {}])[1][r[im]] = r[iv]
ids = sorted(d)
n = len(ids) // iters
tot = 0.0
for i in ids[-n:]:
    k, m = d[i]
    t = float(m.get("gpu__time_duration.sum", 0))
    tot += t
    print(f"{k:48s} {t / 1e3:8.2f} us  grid={m.get('launch__grid_size')}")
print(f"total {tot / 1e3:.2f} us over {n} launches")
