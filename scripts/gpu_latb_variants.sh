#!/bin/bash
# A/B of the bench's B = 1 latency (L2 flushed, latency_us_p50) over variants/<name>.so
cp paper_2511_11664_b200/_lib/libsczip_b200.so /tmp/orig_latb.so
for v in "$@"; do
  cp variants/$v.so paper_2511_11664_b200/_lib/libsczip_b200.so
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-configs --no-cpu-baseline > gpurun_out/latb_$v.json 2> gpurun_out/latb_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/latb_{sys.argv[1]}.json").read().strip().splitlines()[-1])
l = d["latency_us_p50"]
print(sys.argv[1], "enc", round(l["encode"], 1), "dec", round(l["decode"], 1), "rt", round(l["device_round_trip"], 1),
      {k: v for k, v in l["kernel_us"].items() if "select" in k})
PY
done
cp /tmp/orig_latb.so paper_2511_11664_b200/_lib/libsczip_b200.so
