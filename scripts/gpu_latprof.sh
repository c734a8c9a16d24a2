mkdir -p gpurun_out
ITERS=3 timeout 600 ncu --set full --clock-control none --import-source on -s 12 -c 12 -o gpurun_out/prof_lat_r2 -f python scripts/latency_probe.py > gpurun_out/prof_lat_r2.log 2>&1
ITERS=3 timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -s 12 -c 12 -o gpurun_out/prof_lat_r2_warm -f python scripts/latency_probe.py > gpurun_out/prof_lat_r2_warm.log 2>&1
ls -la gpurun_out
