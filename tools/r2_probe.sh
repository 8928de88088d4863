#!/bin/bash
# round-2 probe: FP64/LDS latency microbenchmark + one full ncu capture (with
# per-instruction stall sampling) of the layered k_conv<10> on C2
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/fp64_latency.cu && /tmp/lat | tee gpurun_out/fp64_latency.txt
ncu --set full --import-source on --clock-control none -k regex:k_conv -s 1 -c 1 -o gpurun_out/r2_conv_c2 -f \
  python tools/profile_run.py --workload c2 > gpurun_out/r2_conv_c2.log 2>&1
ncu -i gpurun_out/r2_conv_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_conv_c2_sass.csv 2>/dev/null
ls -la gpurun_out/r2_conv_c2*
