set -x
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_lat.json 2> gpurun_out/bench_lat.err
for bs in 8192 4096 2048; do BLOCK_SYMS=$bs timeout 120 python scripts/latency_breakdown.py > gpurun_out/latbd_$bs.txt 2>&1; done
SCZ_NO_GRAPHS=1 timeout 120 python scripts/latency_breakdown.py > gpurun_out/latbd_nographs.txt 2>&1
ITERS=3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none --csv --log-file gpurun_out/lat_launches.csv python scripts/latency_probe.py > /dev/null 2>&1
ITERS=3 timeout 600 ncu --set full --clock-control none --import-source on -s 14 -c 14 -o gpurun_out/prof_lat -f python scripts/latency_probe.py > /dev/null 2>&1
ls -la gpurun_out
