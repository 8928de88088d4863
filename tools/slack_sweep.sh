#!/bin/bash
mkdir -p gpurun_out
B=paper_2101_10881_b200/pseval_b200
for sl in 1.5 2 3 5 8; do
  echo -n "slack $sl: "; PSE_FLOW_SLACK=$sl python tools/profile_run.py --workload c3h --reps 3
  echo -n "slack $sl p2: "; PSE_FLOW_SLACK=$sl timeout 300 $B bench p2 --degree 152 --precision 2 10 --csv gpurun_out/sl.csv > /dev/null 2>&1; cut -d, -f3,11 gpurun_out/sl.csv | tail -2 | tr '\n' ' '; echo
done
