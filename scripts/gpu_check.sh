# quick GPU check: parity suite, bench line, select-phase probe (B = 1)
set -x
mkdir -p gpurun_out
TAG=${1:-chk}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests_${TAG}.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ITERS=6 SCZ_SELECT_PROBE=1 timeout 120 python scripts/latency_probe.py > gpurun_out/selprobe_${TAG}.txt 2>&1
timeout 120 python scripts/latency_breakdown.py > gpurun_out/latbd_${TAG}.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
