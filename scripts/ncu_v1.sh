#!/bin/bash
# ncu --set full of the v1 serial kernels on one VGG16 tensor (B = 1)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
   -k "regex:k_rans_(enc_v1_fast|dec_v1_fast)" -c 2 -o gpurun_out/prof_v1 -f \
   python scripts/v1_probe.py vgg16 1 > gpurun_out/ncu_v1.log 2>&1
ncu -i gpurun_out/prof_v1.ncu-rep --page details --csv > gpurun_out/prof_v1_details.csv 2>&1
ncu -i gpurun_out/prof_v1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_v1_source.csv 2>&1
ls -la gpurun_out
