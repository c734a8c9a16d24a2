#!/bin/bash
# parity suite, select-phase probe (B = 1), latency breakdown, full bench line
mkdir -p gpurun_out
TAG=${1:-chk}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests_${TAG}.log
ITERS=6 SCZ_SELECT_PROBE=1 timeout 120 python scripts/latency_probe.py 2>&1 | grep "k_select" | tail -4 > gpurun_out/selprobe_${TAG}.txt
timeout 120 python scripts/latency_breakdown.py > gpurun_out/latbd_${TAG}.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
cat gpurun_out/tests_${TAG}.log gpurun_out/selprobe_${TAG}.txt gpurun_out/latbd_${TAG}.txt
