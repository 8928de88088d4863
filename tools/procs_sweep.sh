#!/bin/bash
B=paper_2101_10881_b200/pseval_b200
for pr in 0.125 0.25 0.5 1 2; do for sl in 0 1; do
  echo -n "procs $pr slack $sl: "; PSE_FLOW_PROCS=$pr PSE_FLOW_SLACK=$sl timeout 300 $B bench p2 --degree 152 --precision 1 2 10 --csv gpurun_out/sw.csv > /dev/null 2>&1; cut -d, -f3,11 gpurun_out/sw.csv | tail -3 | tr '\n' ' '
  PSE_FLOW_PROCS=$pr PSE_FLOW_SLACK=$sl python tools/profile_run.py --workload c3h --reps 3
done; done
