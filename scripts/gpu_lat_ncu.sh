# B = 1 per-kernel durations (ncu, serialised) + the graph-replay breakdown
set -x
mkdir -p gpurun_out
TAG=${1:-l}
timeout 120 python scripts/latency_breakdown.py > gpurun_out/latbd_${TAG}.txt 2>&1
ITERS=3 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lat_launches_${TAG}.csv python scripts/latency_probe.py > /dev/null 2>&1
ls -la gpurun_out
