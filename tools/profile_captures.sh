#!/bin/bash
# ncu evidence for profiles/ (run on a gpurun box, one GPU; summarise here with
# tools/ncu_summary.py). Launch lists: serialised, cold-cache per-kernel times
# (compare shares, not absolute times). Full captures: one launch each; keep at
# most two .ncu-rep per gpurun call (the merge-back limit is 64 MiB).
#   usage: tools/profile_captures.sh launches | conv_c2 | flow <workload> [m]
mkdir -p gpurun_out
case "$1" in
  launches)
    for w in c2 c3 c3h; do
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
        python tools/profile_run.py --workload $w > /dev/null 2>&1
    done
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1 ;;
  conv_c2)  # the layered k_conv (second launch: a layer-2 group)
    ncu --set full --import-source on --clock-control none -k regex:k_conv -s 1 -c 1 -o gpurun_out/conv_c2_full -f \
      python tools/profile_run.py --workload c2 ;;
  flow)     # the dataflow kernel of a workload (optionally at precision m)
    ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_$2${3:+_m$3} -f \
      python tools/profile_run.py --workload $2 ${3:+--m $3} ;;
esac
