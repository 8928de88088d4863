ncu --set full --import-source on --clock-control none -k k_conv -s 1 -c 1 -o gpurun_out/r2b_conv_c2 -f \
  python tools/profile_run.py --workload c2 > gpurun_out/ncu16.log 2>&1; echo "conv rc=$?"; tail -5 gpurun_out/ncu16.log
