#!/bin/bash
# round-2 ncu evidence (one GPU): the launch list of the bench command itself
# (cold-cache, serialised: compare shares), full captures of the layered
# k_conv<10> (C2), the dataflow k_conv_flow<10> (C3') and the CTA-local
# k_conv_cta<1> (C3 at m=1), and DRAM traffic of one C2 evaluation's conv stage
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k k_conv -s 1 -c 1 -o gpurun_out/r2_conv_c2 -f \
  python tools/profile_run.py --workload c2 > /dev/null 2>&1; echo "conv rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/r2_flow_c3h -f \
  python tools/profile_run.py --workload c3h > /dev/null 2>&1; echo "flow rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_conv_cta -c 1 -o gpurun_out/r2_cta_c3_m1 -f \
  python tools/profile_run.py --workload c3 --m 1 > /dev/null 2>&1; echo "cta rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_traffic_c2.csv python tools/profile_run.py --workload c2 > /dev/null 2>&1; echo "traffic rc=$?"
ls -la gpurun_out/r2_*ncu-rep gpurun_out/r2_*.csv
