#!/bin/bash
# Round-2 evidence session: GPU tests, the default bench line, the ncu launch
# list of the bench (kernel shares), and one `ncu --set full` capture of every
# kernel of a VGG16 B = 256 step (scripts/profile_step.py).  Summaries are
# written by scripts/ncu_summarize.py and scripts/launch_shares.py into
# gpurun_out/; copy them to profiles/<tag>/.
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/tests_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e --no-configs > /dev/null 2> gpurun_out/ncu_launch_${TAG}.err
[ "${SKIP_FULL:-0}" = 1 ] || timeout 1200 ncu --set full --clock-control none --import-source on \
    -s ${NCU_SKIP:-14} -c ${NCU_COUNT:-16} -o gpurun_out/prof_${TAG} -f \
    python scripts/profile_step.py vgg16 256 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
[ "${SKIP_FULL:-0}" = 1 ] || python scripts/ncu_summarize.py gpurun_out/prof_${TAG}.ncu-rep gpurun_out/ncu_full_summary_${TAG}.txt gpurun_out/ncu_traffic_${TAG}.json > /dev/null
python scripts/launch_shares.py gpurun_out/launches_${TAG}.csv > gpurun_out/launch_shares_${TAG}.txt 2>&1
ls -la gpurun_out
