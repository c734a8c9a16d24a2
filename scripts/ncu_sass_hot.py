"""Per-kernel SASS hotspots from an ncu report: stall-sample totals by reason,
then the hottest address ranges (loops) and instructions.

usage: python scripts/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [TOP] [LAUNCH_INDEX]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"]
if len(sys.argv) > 4:
    cmd += ["--launch-skip", sys.argv[4], "--launch-count", "1"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = None
recs = []
name = None
for r in rows:
    if not r:
        continue
    if r[0] == "Kernel Name":
        if recs:
            break  # first matching launch only
        name = r[1]
        continue
    if r[0] == "Address":
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, r))
    recs.append(d)
if not recs:
    print("no records")
    sys.exit(0)


def num(v):
    try:
        return float(v)
    except (TypeError, ValueError):
        return 0.0


stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in recs)
inst = sum(num(d["Instructions Executed"]) for d in recs)
print(f"{name}\n  samples {tot:.0f}  warp-instructions {inst:.0f}")
by = {c: sum(num(d[c]) for d in recs) for c in stall_cols}
print("  stalls: " + ", ".join(f"{c[6:]} {100 * v / max(tot, 1):.1f}%" for c, v in
                               sorted(by.items(), key=lambda kv: -kv[1]) if v > 0.005 * tot))
wf = sum(num(d.get("L1 Wavefronts Shared", 0)) for d in recs)
wfi = sum(num(d.get("L1 Wavefronts Shared Ideal", 0)) for d in recs)
print(f"  shared wavefronts {wf:.0f} (ideal {wfi:.0f})")
# hottest instructions
print("  top instructions (samples, executed, shared wavefronts, top stall):")
for d in sorted(recs, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:top]:
    s = num(d["Warp Stall Sampling (All Samples)"])
    ts = max(stall_cols, key=lambda c: num(d[c]))
    print(f"  {d['Address'][-5:]} {s:6.0f} {100 * s / max(tot, 1):5.1f}% ex={num(d['Instructions Executed']):>10.0f} "
          f"wf={num(d.get('L1 Wavefronts Shared', 0)):>9.0f} {ts[6:]:14s} {d['Source'].strip()[:70]}")
# samples by 256-instruction-byte region (loops show up as dense regions)
reg = defaultdict(lambda: [0.0, 0.0])
for d in recs:
    a = int(d["Address"], 16) & 0xFFFFF
    reg[a >> 10][0] += num(d["Warp Stall Sampling (All Samples)"])
    reg[a >> 10][1] += num(d["Instructions Executed"])
print("  by 1 KB code region (offset, samples %, warp-instructions %):")
for k in sorted(reg):
    s, e = reg[k]
    if s > 0.01 * tot or e > 0.01 * inst:
        print(f"    {k << 10:06x} {100 * s / max(tot, 1):5.1f}% {100 * e / max(inst, 1):5.1f}%")
