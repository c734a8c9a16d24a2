# ncu --set full of one kernel (regex) at B = 256 (vgg16 step) and at B = 1
# (latency probe).  usage: bash scripts/gpu_ncu_one.sh REGEX TAG
K=$1; TAG=${2:-k}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/one_${TAG}_b256 -f python scripts/profile_step.py vgg16 256 4 > gpurun_out/one_${TAG}_b256.log 2>&1
ITERS=4 timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/one_${TAG}_b1 -f python scripts/latency_probe.py > gpurun_out/one_${TAG}_b1.log 2>&1
