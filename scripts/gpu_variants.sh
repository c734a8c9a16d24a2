#!/bin/bash
# A/B builds: each variants/<name>.so replaces the in-tree library for one
# short bench run (device-resident value + per-kernel shares).
mkdir -p gpurun_out
cp paper_2511_11664_b200/_lib/libsczip_b200.so /tmp/orig.so
for v in "$@"; do
  cp variants/$v.so paper_2511_11664_b200/_lib/libsczip_b200.so
  for r in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-configs --no-cpu-baseline > gpurun_out/var_${v}_$r.json 2> gpurun_out/var_${v}_$r.err
    python - "$v" "$r" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/var_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
ms = d["ms_per_step"]
ks = {k: round(v * ms * 1000, 1) for k, v in d["kernel_share"].items()}
print(sys.argv[1], sys.argv[2], round(d["value"], 1), "GB/s", round(ms, 4), "ms", ks)
PY
  done
done
cp /tmp/orig.so paper_2511_11664_b200/_lib/libsczip_b200.so
