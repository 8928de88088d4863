ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/r2b_flow_c3_m2 -f \
  python tools/profile_run.py --workload c3 --m 2 > /dev/null 2>&1; echo "flow rc=$?"
python tools/diag/layers.py --workload c3 --m 2
