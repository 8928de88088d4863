#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --workload c2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3h.csv python tools/profile_run.py --workload c3h > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_run.py --workload c3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c3h_full -f python tools/profile_run.py --workload c3h > gpurun_out/prof3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c3_full -f python tools/profile_run.py --workload c3 >> gpurun_out/prof3.log 2>&1
ls -la gpurun_out; tail -3 gpurun_out/prof3.log
