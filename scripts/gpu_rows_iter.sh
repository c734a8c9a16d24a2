#!/bin/bash
# k_rows_small8 iteration: GPU parity suite, bench line, launch list of the
# bench step, memcheck + racecheck over the row-decode / corruption tests.
mkdir -p gpurun_out
TAG=${1:-rows}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/tests_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e --no-configs > /dev/null 2> gpurun_out/ncu_launch_${TAG}.err
python scripts/launch_shares.py gpurun_out/launches_${TAG}.csv > gpurun_out/launch_shares_${TAG}.txt 2>&1
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 17 --target-processes all \
    python -m pytest tests -m gpu -x -q -p no:cacheprovider \
    -k "corrupt or bench_path or batch_api or random_round_trips or csr or device_header or degenerate" \
    > gpurun_out/${tool}_${TAG}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${tool}_${TAG}.log
done
cat gpurun_out/tests_${TAG}.log gpurun_out/launch_shares_${TAG}.txt; tail -n 2 gpurun_out/memcheck_${TAG}.log gpurun_out/racecheck_${TAG}.log
