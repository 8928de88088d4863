#!/bin/bash
# round-2 (second half) ncu evidence (one GPU): launch list of the bench
# command itself, full captures of the layered k_conv<10> (C2), the dataflow
# k_conv_flow<10> (C3'), the CTA-local layered k_conv_ctl<1> (C3 at m=1) and
# the dataflow kernel at m=2 (C3), DRAM traffic of the conv stages
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_bench_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k k_conv -s 1 -c 1 -o gpurun_out/r2b_conv_c2 -f \
  python tools/profile_run.py --workload c2 > /dev/null 2>&1; echo "conv rc=$?"
ncu --set full --import-source on --clock-control none -k k_conv_flow -c 1 -o gpurun_out/r2b_flow_c3h -f \
  python tools/profile_run.py --workload c3h > /dev/null 2>&1; echo "flow rc=$?"
ncu --set full --import-source on --clock-control none -k k_conv_ctl -c 1 -o gpurun_out/r2b_ctl_c3_m1 -f \
  python tools/profile_run.py --workload c3 --m 1 > /dev/null 2>&1; echo "ctl rc=$?"
ncu --set full --import-source on --clock-control none -k k_conv_flow -c 1 -o gpurun_out/r2b_flow_c3_m2 -f \
  python tools/profile_run.py --workload c3 --m 2 > /dev/null 2>&1; echo "flow m2 rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2b_traffic_c2.csv python tools/profile_run.py --workload c2 > /dev/null 2>&1; echo "traffic rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2b_traffic_c3_m1.csv python tools/profile_run.py --workload c3 --m 1 > /dev/null 2>&1; echo "traffic m1 rc=$?"
ls -la gpurun_out/r2b_*ncu-rep gpurun_out/r2b_*.csv
