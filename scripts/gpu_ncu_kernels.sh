# ncu --set full of selected pipeline kernels in the batch bench (one launch each)
set -x
mkdir -p gpurun_out
TAG=${1:-k}
REGEX=${2:-'k_(quantize|stats|rows_small8|rans_enc_v2_u8u16)'}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$REGEX" -s 4 -c 4 \
    -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/ncu_${TAG}.err
ls -la gpurun_out
