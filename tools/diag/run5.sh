mkdir -p gpurun_out
./tools/fp64_latency
ncu --set full --import-source on --clock-control none -k regex:k_conv_ctl -c 1 -o gpurun_out/r2b_ctl_c3_m1 -f \
  python tools/profile_run.py --workload c3 --m 1 > /dev/null 2>&1; echo "ctl rc=$?"
