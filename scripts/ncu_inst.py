"""Source lines of one kernel sorted by executed warp instructions (ncu report, cuda,sass view)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f = [], None
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        try:
            rows.append((int(r[7] or 0), float(r[4] or 0), f + ":" + r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows)
stall = sum(x[1] for x in rows)
print(f"total warp instructions {tot}, stall samples {stall:.0f}")
for x in sorted(rows, reverse=True)[:top]:
    print(f"{x[0]:>10d} {100 * x[0] / tot:5.1f}%  samples {100 * x[1] / max(stall, 1):5.1f}%  {x[2]:22s} {x[3]}")
