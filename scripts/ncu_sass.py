"""Per-SASS-instruction stall breakdown from an ncu report (top N by samples)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
i0 = 1 if rows[0][0] == "Kernel Name" else 0
h = rows[i0]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stalls = [(j, x) for j, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
recs = []
for r in rows[i0 + 1:]:
    if len(r) < len(h):
        continue
    try:
        s = float(r[iall] or 0)
    except ValueError:
        continue
    br = sorted(((float(r[j] or 0), x[6:]) for j, x in stalls), reverse=True)[:3]
    recs.append((s, r[ia][-5:], r[isrc].strip()[:60], br))
tot = sum(x[0] for x in recs)
order = {id(x): k for k, x in enumerate(recs)}
for s, a, src, br in sorted(recs, key=lambda x: -x[0])[:top]:
    print(f"{s:6.0f} {100 * s / tot:5.1f}% {a} {src:60s} " + " ".join(f"{n}={v:.0f}" for v, n in br if v))
