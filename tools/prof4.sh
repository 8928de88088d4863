#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c3_m2 -f python tools/profile_run.py --workload c3 --m 2 > gpurun_out/prof4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c3_m4 -f python tools/profile_run.py --workload c3 --m 4 >> gpurun_out/prof4.log 2>&1
tail -2 gpurun_out/prof4.log; ls -la gpurun_out
