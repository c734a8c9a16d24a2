#!/bin/bash
# A/B of B = 1 latency (warm, scripts/latency_breakdown.py) over variants/<name>.so
cp paper_2511_11664_b200/_lib/libsczip_b200.so /tmp/orig_lat.so
for v in "$@"; do
  cp variants/$v.so paper_2511_11664_b200/_lib/libsczip_b200.so
  for r in 1 2; do
    echo "== $v $r: $(timeout 120 python scripts/latency_breakdown.py 2>&1 | grep -E 'gpu_enc|gpu_dec|wall' | awk '{print $1, $3}' | tr '\n' ' ')"
  done
done
cp /tmp/orig_lat.so paper_2511_11664_b200/_lib/libsczip_b200.so
