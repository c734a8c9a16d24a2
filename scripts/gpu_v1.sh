#!/bin/bash
# v1 serial kernels: GPU parity (v1 cases), per-symbol probe at B = 1 and 256
mkdir -p gpurun_out
TAG=${1:-v1}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests_${TAG}.log
timeout 300 python scripts/v1_probe.py vgg16 1 > gpurun_out/v1_probe1_${TAG}.json 2>&1
timeout 300 python scripts/v1_probe.py vgg16 256 > gpurun_out/v1_probe256_${TAG}.json 2>&1
timeout 300 python scripts/v1_probe.py mobilenetv2 256 > gpurun_out/v1_probe_mnv2_${TAG}.json 2>&1
cat gpurun_out/tests_${TAG}.log gpurun_out/v1_probe*_${TAG}.json
