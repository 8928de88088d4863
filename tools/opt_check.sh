#!/bin/bash
for v in "" o1 o2; do
  echo -n "variant [$v]: "; PSE_LIB_VARIANT=$v python tools/profile_run.py --workload c2 --reps 3
  echo -n "variant [$v]: "; PSE_LIB_VARIANT=$v python tools/profile_run.py --workload c3h --reps 3
done
