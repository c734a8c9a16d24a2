#!/bin/bash
# A/B of the v1 serial coders over variants/<name>.so: per-symbol times at B = 256
cp paper_2511_11664_b200/_lib/libsczip_b200.so /tmp/orig_v1.so
for v in "$@"; do
  cp variants/$v.so paper_2511_11664_b200/_lib/libsczip_b200.so
  echo "== $v $(timeout 300 python scripts/v1_probe.py vgg16 256 | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],2), d["split_ms"], d["ns_per_symbol"], d["status_ok"], d["max_err_ok"])')"
done
cp /tmp/orig_v1.so paper_2511_11664_b200/_lib/libsczip_b200.so
