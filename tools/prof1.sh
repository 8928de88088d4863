mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3h.csv python tools/profile_run.py --workload c3h > gpurun_out/prof_c3h.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --workload c2 > gpurun_out/prof_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_conv -s 1 -c 1 -o gpurun_out/conv_c2_full python tools/profile_run.py --workload c2 > gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_conv_prod -c 1 -s 20 -o gpurun_out/prod_c3h_full python tools/profile_run.py --workload c3h >> gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_conv_accum -c 1 -s 20 -o gpurun_out/accum_c3h_full python tools/profile_run.py --workload c3h >> gpurun_out/prof_full.log 2>&1
tail -3 gpurun_out/prof_full.log
