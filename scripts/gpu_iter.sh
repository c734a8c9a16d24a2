# Quick iteration session: GPU tests (or a -k subset), a short bench line
# without the host-side legs, and the ncu launch list of the bench step.
# usage: bash scripts/gpu_iter.sh TAG [pytest -k expr]
TAG=${1:-it}
mkdir -p gpurun_out
if [ -n "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$2" 2>&1 | tail -15 > gpurun_out/tests_${TAG}.log
else
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests_${TAG}.log
fi
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e --no-configs > /dev/null 2>&1
python scripts/launch_shares.py gpurun_out/launches_${TAG}.csv > gpurun_out/launch_shares_${TAG}.txt 2>&1
ITERS=3 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lat_launches_${TAG}.csv python scripts/latency_probe.py > /dev/null 2>&1
