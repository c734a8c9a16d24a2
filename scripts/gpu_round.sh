#!/bin/bash
# One GPU session: parity tests, the bench line, the ncu launch list and a
# full ncu capture of the heavy kernels.  Outputs land in gpurun_out/;
# summarise them into profiles/<tag>/ with scripts/ncu_summarize.py and
# scripts/launch_shares.py.
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/tests_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_launch_${TAG}.err
[ "${SKIP_FULL:-0}" = 1 ] || timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:k_(rans_enc_v2|rans_dec_v2|quantize|stats|rows_|select|rowhist|colhist|materialize|dec_prepare)" \
    -s 0 -c ${NCU_COUNT:-36} -o gpurun_out/prof_${TAG} -f \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_full_${TAG}.err
ls -la gpurun_out
