"""Per-kernel share of the (sczip) GPU time in an ncu launch list (the
`--metrics gpu__time_duration.sum --clock-control none` pass of bench.py);
ncu times are cold-cache and serialised, so compare shares, not absolutes.

usage: python scripts/launch_shares.py launches.csv [out.txt]
"""
import csv
import sys
from collections import defaultdict

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summarize import short  # noqa: E402

path = sys.argv[1]
lines = open(path).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if len(r) < len(h) or r[im] != "gpu__time_duration.sum":
        continue
    k = short(r[ik])
    if not k.startswith("k_"):  # torch kernels of bench.py's own checks
        continue
    tot[k] += float(r[iv].replace(",", ""))
    cnt[k] += 1
all_ns = sum(tot.values())
out = [f"# kernel shares of {path.split('/')[-1]} ({sum(cnt.values())} launches, {all_ns / 1e6:.2f} ms total)",
       f"{'kernel':28s} {'share':>7s} {'launches':>9s} {'mean us':>10s}"]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    out.append(f"{k:28s} {100 * v / all_ns:6.2f}% {cnt[k]:9d} {v / cnt[k] / 1e3:10.2f}")
txt = "\n".join(out) + "\n"
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(txt)
print(txt)
