"""Summarise a gpu_iter.sh session: tests, bench headline, shares, B=1 launches."""
import json
import subprocess
import sys

tag = sys.argv[1]
d = "gpurun_out/"
print(open(d + f"tests_{tag}.log").read()[-600:])
try:
    b = json.loads(open(d + f"bench_{tag}.json").read().strip().splitlines()[-1])
    print("value", round(b["value"], 1), "ms/step", round(b["ms_per_step"], 4), "roofline",
          {k: b["roofline"][k] for k in ("kernel", "achieved", "frac", "launch_ms")})
    lat = b.get("latency_us_p50", {})
    print("latency", {k: lat.get(k) for k in ("encode", "decode", "encode_plus_decode", "device_round_trip")})
    print("kernel_us", lat.get("kernel_us"))
    print("v1", b.get("v1_reference_format"))
except Exception as e:  # noqa: BLE001
    print("bench parse failed", e, open(d + f"bench_{tag}.err").read()[-2000:])
print(open(d + f"launch_shares_{tag}.txt").read())
print(subprocess.run([sys.executable, "scripts/launch_table.py", d + f"lat_launches_{tag}.csv"],
                     capture_output=True, text=True).stdout)
