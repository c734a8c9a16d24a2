"""Top source lines by warp-stall samples from an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, out = None, []
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
            out.append([float(r[4]), int(r[7] or 0), f + ":" + r[0], r[1][:100]])
        except ValueError:
            pass
tot = sum(o[0] for o in out)
print("total samples", tot)
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0]:7.0f} {100 * o[0] / max(tot, 1):5.1f}% inst={o[1]:>9d} {o[2]:24s} {o[3]}")
