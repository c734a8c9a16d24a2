"""Per-launch durations (us) and instruction counts from an ncu report."""
import csv
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[0]
ki, ti, ii, gi = (h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
                                        "launch__grid_size"))
unit = rows[1][ti]
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1.0)
tot = 0.0
for r in rows[2:]:
    t = float(r[ti].replace(",", "")) * scale
    tot += t
    print(f"{r[ki][:48]:48s} {t:9.2f} us  grid {r[gi]:>6s}  inst {float(r[ii].replace(',', '')):>12.0f}")
print(f"total {tot:.2f} us over {len(rows) - 2} launches")
