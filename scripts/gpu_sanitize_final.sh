#!/bin/bash
# compute-sanitizer over the GPU parity suite on the final tree: memcheck and
# synccheck over every test except the 25 M-symbol v1 case; racecheck over the
# v2 / batch / search / quantise / row-decode tests plus the v1 coders on
# small streams (racecheck on the serial v1 streams of the full suite runs
# for hours).
mkdir -p gpurun_out
SEL="not llama and not c4"
for tool in memcheck synccheck; do
  extra=""; [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 17 --target-processes all \
      python -m pytest tests -m gpu -x -q -k "$SEL" -p no:cacheprovider > gpurun_out/final_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/final_${tool}.log
done
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 17 --target-processes all \
  python -m pytest tests -m gpu -x -q -p no:cacheprovider \
  -k "v2_containers_match_oracle or lanes_are_reference or batch_api or lazy_search or device_header_decode_matches or mixed_symbol or heterogeneous or random_round_trips or quantize or csr or test_v1_containers_bit_exact or general_alphabet_containers" \
  > gpurun_out/final_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/final_racecheck.log
for f in gpurun_out/final_*.log; do tail -n 3 "$f"; done
