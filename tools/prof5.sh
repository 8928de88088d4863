#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c3_m1 -f python tools/profile_run.py --workload c3 --m 1 > gpurun_out/prof5.log 2>&1
tail -1 gpurun_out/prof5.log
