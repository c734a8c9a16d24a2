# Round-2 profile session: B = 1 latency launch list + graph breakdown, and a
# full ncu capture (with source) of every kernel of one VGG16 B = 256 step.
set -x
mkdir -p gpurun_out
TAG=${1:-p}
bash scripts/gpu_lat_ncu.sh $TAG
timeout 1500 ncu --set full --clock-control none --import-source on \
    -s ${NCU_SKIP:-14} -c ${NCU_COUNT:-16} -o gpurun_out/prof_${TAG} -f \
    python scripts/profile_step.py vgg16 256 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
python scripts/ncu_summarize.py gpurun_out/prof_${TAG}.ncu-rep gpurun_out/ncu_full_summary_${TAG}.txt gpurun_out/ncu_traffic_${TAG}.json > /dev/null
ls -la gpurun_out
