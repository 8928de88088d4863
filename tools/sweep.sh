#!/bin/bash
# usage: tools/sweep.sh "ENV=..." workload reps  -- one timing line per config
for cfg in "$@"; do
  IFS=: read -r envs wl reps <<< "$cfg"
  echo -n "[$envs] " >> gpurun_out/sweep.log
  env $envs python tools/profile_run.py --workload $wl --reps $reps >> gpurun_out/sweep.log 2>&1
done
